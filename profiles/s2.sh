for cfg in "X=1" "SVDSC_S2_RT16=4" "SVDSC_S2_RT16=3"; do
  env $cfg python tools/timeline.py --workload 3 --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('$cfg', round(d['span_ms'],1), 'cgs2', round(sum(v[0] for k,v in b.items() if 'cgs2' in k),1), {k: v[2] for k,v in b.items() if 'stream2' in k})"
done
