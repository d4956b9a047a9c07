timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "products or svds" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E |FAILED" gpurun_out/t.log | head -5
for cfg in "SVDSC_SPMV=bins" "X=1"; do
  env $cfg python tools/timeline.py --workload 3 --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('$cfg', round(d['span_ms'],1), {k: (round(v[0],1), v[2]) for k,v in b.items() if 'spmv' in k})"
done
