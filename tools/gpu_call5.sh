cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "products" -p no:cacheprovider 2>&1 | tail -3
python tools/profile_ops.py --workload 4 --reps 5 --skip-cgs 2>&1 | tail -1
python tools/profile_ops.py --workload 3 --reps 20 --skip-cgs 2>&1 | tail -1
python tools/profile_ops.py --workload 5 --scale 8 --reps 5 --skip-cgs 2>&1 | tail -1
