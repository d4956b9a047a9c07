set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
R="python tools/repro_smoke.py"
$R --tag plain1 > gpurun_out/c1_plain.log 2>&1; cat gpurun_out/c1_plain.log
$R --tag plain2 2>&1 | tail -1
SVDSC_JACOBI_SEPARATE=1 $R --tag jsep 2>&1 | tail -1
SVDSC_CLUSTER_CGS2=0 $R --tag nocl 2>&1 | tail -1
SVDSC_NO_FUSED=1 $R --tag nofused 2>&1 | tail -1
SVDSC_JACOBI_PULL=1 $R --tag jpull 2>&1 | tail -1
$R --tag pre_ncu > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/c1_launches.csv $R --tag ncu_default 2>&1 | grep REPRO
for v in SVDSC_JACOBI_SEPARATE=1 SVDSC_CLUSTER_CGS2=0 SVDSC_NO_FUSED=1 SVDSC_JACOBI_PULL=1; do
  env $v ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/c1_launches_$v.csv $R --tag ncu_$v 2>&1 | grep REPRO
done
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c 1000 --csv --log-file /dev/null $R --tag ncu_nocache 2>&1 | grep REPRO
