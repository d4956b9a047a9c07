# config-3 profile: small-SVD timings, launch list, ncu --set full of the top kernels
mkdir -p gpurun_out
for p in 150 300 600; do timeout 120 python tests/prof_svd.py $p >> gpurun_out/prof_svd.log 2>&1; done
CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/plain3.log 2>&1; echo plain=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch3.log 2>&1
echo launches_exit=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_tma|k_spmv_vec|k_recombine|k_jacobi_block|k_apply_log" -s 3000 -c 8 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_full3.log 2>&1
echo full_exit=$?
ls -la gpurun_out
