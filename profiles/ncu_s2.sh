mkdir -p gpurun_out
CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > gpurun_out/plain3.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs2_stream2 -s 531 -c 1 -o gpurun_out/prof_s2 $CMD > gpurun_out/ncu_s2.log 2>&1; echo s2=$?
