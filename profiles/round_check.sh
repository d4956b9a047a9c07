# full round check on one B200: GPU tests, smoke, bench (ours + reference arm)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python tests/debug_tma.py > gpurun_out/debug_tma.log 2>&1; echo debug_tma_exit=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$?
grep -E "passed|failed|Error" gpurun_out/gpu_tests.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_exit=$?
timeout 900 python bench.py --workload 3 --no-e2e > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench3_exit=$?
cat gpurun_out/bench.json gpurun_out/bench3.json
