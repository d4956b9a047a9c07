# round check on one B200: GPU tests, smoke, default bench (+ ncu launch list of smoke)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/${TAG}_gpu_tests.log | grep -E "passed|failed|FAILED|Error" | tail -15
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; head -c 1500 gpurun_out/${TAG}_bench.json
fi
