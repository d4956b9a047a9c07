mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "products or svds or lbp" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -5
for cfg in "SVDSC_SPMV=merge" "SVDSC_SPMV=bins"; do
 for w in 3 4; do
  env $cfg python tools/timeline.py --workload $w --out gpurun_out/tl.json > gpurun_out/tl_err.log 2>&1 || tail -3 gpurun_out/tl_err.log
  python -c "
import json; d=json.load(open('gpurun_out/tl.json'))
print('$cfg w$w', round(d['span_ms'],1), 'spmv', {k:v for k,v in d['busy'].items() if 'spmv' in k})"
 done
done
