cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu_allbench.sh r02o
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4600 --csv --log-file gpurun_out/r02o_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ceiling > gpurun_out/r02o_ncu.log 2>&1; echo "ncu rc=$?"
