timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2 or svds" 2>&1 | tail -1
for cfg in "SVDSC_CLUSTER_CGS2=0" "X=1" "SVDSC_CLUSTER_CGS2=40000000"; do
 for w in 1 2; do
  env $cfg python tools/timeline.py --workload $w --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('$cfg w$w', round(d['span_ms'],2), {k: (round(v[0],2), v[1], v[2]) for k,v in b.items() if 'cgs2' in k})"
 done
done
