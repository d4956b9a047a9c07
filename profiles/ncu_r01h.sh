mkdir -p gpurun_out
CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
SVDSC_STREAM_VARIANT=0 SVDSC_KTIMING=1 $CMD > gpurun_out/kt.log 2>&1; echo kt=$?; grep ktiming gpurun_out/kt.log
SVDSC_STREAM_VARIANT=0 $CMD > gpurun_out/plain3.log 2>&1; echo plain=$?
SVDSC_STREAM_VARIANT=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_tma" -s 2000 -c 1 -o gpurun_out/prof_tma32 $CMD > gpurun_out/ncu_tma.log 2>&1; echo tma=$?
