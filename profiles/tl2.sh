mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2 or svds_parity" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -5
python tools/timeline.py --workload 2 --out gpurun_out/tl2.json 2>&1 | grep -v -i warn | head -8
