cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "products" -p no:cacheprovider 2>&1 | tail -2
for cfg in "--workload 4 --reps 5" "--workload 3 --reps 20" "--workload 5 --scale 8 --reps 5"; do
  python tools/profile_ops.py $cfg --skip-cgs --spmv seg 2>&1 | tail -1
done
