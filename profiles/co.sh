CMD="python bench.py --workload 3 --steps 2 --warmup 1 --no-e2e --no-cpu"
for co in "" 100 50; do
  env ${co:+SVDSC_CARVEOUT=$co} SVDSC_STREAM_VARIANT=0 SVDSC_KTIMING=1 $CMD > gpurun_out/co$co.log 2>&1; echo co=$co $?; grep ktiming gpurun_out/co$co.log | tail -1; python -c "
import json; d=json.loads(open('gpurun_out/co$co.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
done
