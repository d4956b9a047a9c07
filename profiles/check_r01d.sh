# op-level parity + timings after the DMMA recombine / cross-round Jacobi / TMA CGS2 rewrite
mkdir -p gpurun_out
./tools/barrier_bench > gpurun_out/barrier.log 2>&1; echo barrier=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2 or recombine or small_svd or products or lbp" > gpurun_out/ops_tests.log 2>&1; echo ops_tests=$?
tail -3 gpurun_out/ops_tests.log
timeout 600 python tools/time_ops.py --cid 3 > gpurun_out/time_ops3.json 2>&1; echo time_ops3=$?
timeout 600 python tools/time_ops.py --cid 2 > gpurun_out/time_ops2.json 2>&1; echo time_ops2=$?
cat gpurun_out/time_ops3.json gpurun_out/time_ops2.json
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --workload 3 --no-e2e --no-cpu > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench3=$?
timeout 600 python bench.py --no-cpu > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench2=$?
cat gpurun_out/bench3.json gpurun_out/bench2.json
