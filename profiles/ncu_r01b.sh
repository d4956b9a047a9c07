set -x
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests_exit=$?
grep -E "^E  |passed|failed" gpurun_out/gpu_tests.log | head -20
timeout 300 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; echo bench_exit=$?
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_r01b.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches_exit=$?
