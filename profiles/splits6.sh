for cfg in "X=1" "SVDSC_SPLITS_T=1" "SVDSC_SPLITS_T=3" "SVDSC_SPLITS_T=4"; do
  env $cfg python tools/timeline.py --workload 6 --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('w6 $cfg', round(d['span_ms'],2), {k: v[2] for k,v in b.items() if 'gemv' in k})"
done
