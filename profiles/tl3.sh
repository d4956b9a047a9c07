mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2 or svds" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -5
SVDSC_KTIMING=1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu 2>&1 | grep -E "qtiming"
python tools/timeline.py --workload 2 --out gpurun_out/tl2.json 2>&1 | grep -E "span|cgs2_fused"
for cfg in "SVDSC_STREAM_VARIANT=0" "SVDSC_STREAM_VARIANT=2"; do
  env $cfg python tools/timeline.py --workload 3 --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json'))
print('$cfg', round(d['span_ms'],1), 'cgs2', round(sum(v[0] for k,v in d['busy'].items() if 'cgs2' in k),1))"
done
