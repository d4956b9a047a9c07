mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2_fused and tma" 2>&1 | tail -1
for cfg in "SVDSC_STREAM_VARIANT=0" "SVDSC_STREAM_VARIANT=0 SVDSC_TMA_UNIT_KB=48" "SVDSC_STREAM_VARIANT=2"; do
  env $cfg python tools/timeline.py --workload 3 --out gpurun_out/tl.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/tl.json'))
print('$cfg', round(d['span_ms'],1), 'cgs2', round(sum(v[0] for k,v in d['busy'].items() if 'cgs2' in k),1), 'spmv', d['busy'].get('k_spmv_bins'))"
done
