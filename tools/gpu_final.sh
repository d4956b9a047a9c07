# end-of-round evidence on one B200: GPU tests + smoke + default bench
# (tools/gpu_round.sh), all single-GPU bench lines, the ncu launch list of the
# default bench command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02}
bash tools/gpu_round.sh $TAG
bash tools/gpu_allbench.sh $TAG
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4600 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ceiling > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
