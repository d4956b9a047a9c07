mkdir -p gpurun_out
CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/plain3.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_jacobi_block|k_apply_log" -c 2 -o gpurun_out/prof_jac $CMD > gpurun_out/ncu_jac.log 2>&1; echo jac=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_tma" -s 2000 -c 1 -o gpurun_out/prof_tma $CMD > gpurun_out/ncu_tma.log 2>&1; echo tma=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_bins" -s 100 -c 2 -o gpurun_out/prof_spmv $CMD > gpurun_out/ncu_spmv.log 2>&1; echo spmv=$?
