CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_vec -s 40 -c 2 -o gpurun_out/prof_spmv $CMD > gpurun_out/ncu_sp.log 2>&1
echo ncu=$?
