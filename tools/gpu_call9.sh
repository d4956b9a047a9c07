cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r02c_gpu_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c_gpu_tests.log
python bench.py --workload 1 --steps 5 --no-cpu > gpurun_out/r02c_bench1.json 2>&1; tail -c 600 gpurun_out/r02c_bench1.json
python bench.py --workload 3 --steps 3 --no-cpu --no-e2e > gpurun_out/r02c_bench3.json 2>&1; tail -c 400 gpurun_out/r02c_bench3.json
python bench.py --no-cpu > gpurun_out/r02c_bench4.json 2>&1; tail -c 300 gpurun_out/r02c_bench4.json
