for cfg in "X=1" "SVDSC_SPLITS_T=8" "SVDSC_SPLITS_T=16" "SVDSC_SPLITS_T=32" "SVDSC_GEMV_T_WAVES=1"; do
 for w in 2 6; do
  env $cfg python tools/timeline.py --workload $w --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('$cfg w$w', round(d['span_ms'],2), {k: v[2] for k,v in b.items() if 'gemv' in k})"
 done
done
