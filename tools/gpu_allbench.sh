# all single-GPU bench lines of the round (one gpurun call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02}
for w in 2 3 1 6; do
  timeout 900 python bench.py --workload $w --steps 3 --no-cpu > gpurun_out/${TAG}_bench_w$w.json 2> gpurun_out/${TAG}_bench_w$w.err; echo "w$w rc=$?"
done
timeout 900 python bench.py > gpurun_out/${TAG}_bench_w4.json 2> gpurun_out/${TAG}_bench_w4.err; echo "w4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2>&1; echo "ref rc=$?"
