# smoke() under the driver's launch-list profiler and under serialized launches
# (round 1's parity failure appeared only under ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_smoke_launches.csv \
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke_ncu.log 2>&1; echo "smoke under ncu rc=$?"; grep "smoke ok\|Error" gpurun_out/${TAG}_smoke_ncu.log | tail -2
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke_blocking.log 2>&1; echo "smoke blocking rc=$?"; tail -1 gpurun_out/${TAG}_smoke_blocking.log
timeout 600 python tools/repro_smoke.py > gpurun_out/${TAG}_repro_plain.log 2>&1; echo "repro plain rc=$?"; tail -2 gpurun_out/${TAG}_repro_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none python tools/repro_smoke.py > gpurun_out/${TAG}_repro_ncu.log 2>&1; echo "repro ncu rc=$?"; grep -v "^==PROF==" gpurun_out/${TAG}_repro_ncu.log | tail -2
