mkdir -p gpurun_out
CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
export SVDSC_STREAM_VARIANT=0
$CMD > gpurun_out/plain3.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs2_tma -s 530 -c 2 -o gpurun_out/prof_tma512 $CMD > gpurun_out/ncu_tma.log 2>&1; echo tma=$?
