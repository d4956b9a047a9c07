for v in libsvdsc.so libsvdsc_e.so libsvdsc_f.so libsvdsc_g.so; do
 for w in 3 4; do
  SVDSC_LIB_VARIANT=$v python tools/timeline.py --workload $w --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json')); b=d['busy']
print('$v w$w', round(d['span_ms'],1), {k: v[2] for k,v in b.items() if 'spmv' in k})"
 done
done
