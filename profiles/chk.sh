mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_paper_api.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
SVDSC_KTIMING=1 python tests/prof_svd.py 300 2>&1 | grep -E "p=|jtiming" | tail -2
SVDSC_KTIMING=1 python tests/prof_svd.py 150 2>&1 | grep -E "p=|jtiming" | tail -2
python tools/timeline.py --workload 2 --out gpurun_out/tl2.json 2>&1 | grep -v -i warn | head -9
