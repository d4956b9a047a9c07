cd $GRAFT_REPO_ROOT
R="python tools/repro_smoke.py"
$R --tag plain1 2>&1 | tail -1
$R --tag plain2 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
$R --tag pre_ncu > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/c2_launches.csv $R --tag ncu_default 2>&1 | grep REPRO
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/c2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
