mkdir -p gpurun_out
CMD="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
SVDSC_STREAM_VARIANT=0 SVDSC_KTIMING=1 $CMD > gpurun_out/kt.log 2>&1; echo kt=$?; grep ktiming gpurun_out/kt.log; python -c "
import json; d=json.loads(open('gpurun_out/kt.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['breakdown_ms'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2_fused or svds_parity" > gpurun_out/ops_tests.log 2>&1; echo ops_tests=$?
tail -2 gpurun_out/ops_tests.log
SVDSC_STREAM_VARIANT=0 timeout 900 python bench.py --workload 3 --no-e2e --no-cpu --steps 3 > gpurun_out/bench3_v0.json 2> gpurun_out/bench3_v0.err; echo bench3v0=$?
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench2=$?
python - <<'PY'
import json
for f in ["bench3_v0","bench2"]:
    try:
        d=json.load(open(f"gpurun_out/{f}.json"))
        print(f, d["value"], d["ms_per_step"], d["breakdown_ms"])
    except Exception as e: print(f, e)
PY
