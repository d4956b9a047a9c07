set -x
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k forced -p no:cacheprovider 2>&1 | grep -E "assert|passed|failed" | head
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2200 --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo launches_exit=$?
$CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemv_t|k_gemv_n|k_cgs_p2|k_cgs_p1|k_cgs_p3|k_jacobi" -s 30 -c 6 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo full_exit=$?
ls -la gpurun_out
