# A/B of library variants (VARIANTS="libsvdsc.so libsvdsc_x.so ...") on config 3, twice each
mkdir -p gpurun_out
for i in 1 2; do
for v in ${VARIANTS:-libsvdsc.so}; do
  SVDSC_LIB_VARIANT=$v timeout 300 python bench.py --workload ${WL:-3} --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['avg_launch_us'])"
done; done
