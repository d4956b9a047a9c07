for cfg in "X=1"; do
  env $cfg python tools/timeline.py --workload 2 --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('$cfg', round(d['span_ms'],2), {k: v[2] for k,v in b.items() if 'gemv' in k})"
done
