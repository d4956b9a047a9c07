cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --gpus 2 --comm loopback --workload 4 --steps 1 --warmup 1 2>&1 | tail -3
timeout 900 python bench.py --gpus 3 --comm loopback --workload 3 --steps 1 --warmup 1 2>&1 | tail -3
timeout 600 python bench.py --gpus 2 --comm loopback --workload 2 --steps 1 --warmup 1 2>&1 | tail -3
