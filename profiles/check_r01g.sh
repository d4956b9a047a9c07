mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "cgs2 or svds_parity" > gpurun_out/ops_tests.log 2>&1; echo ops_tests=$?
tail -3 gpurun_out/ops_tests.log
timeout 600 python tools/time_ops.py --cid 3 > gpurun_out/time_ops3.json 2>&1; echo time_ops3=$?
timeout 600 python tools/time_ops.py --cid 2 > gpurun_out/time_ops2.json 2>&1; echo time_ops2=$?
cat gpurun_out/time_ops3.json gpurun_out/time_ops2.json
SVDSC_STREAM_VARIANT=0 timeout 900 python bench.py --workload 3 --no-e2e --no-cpu --steps 3 > gpurun_out/bench3_v0.json 2> gpurun_out/bench3_v0.err; echo bench3v0=$?
timeout 900 python bench.py --workload 3 --no-e2e --no-cpu --steps 3 > gpurun_out/bench3_v2.json 2> gpurun_out/bench3_v2.err; echo bench3v2=$?
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench2=$?
python - <<'PY'
import json
for f in ["bench3_v0","bench3_v2","bench2"]:
    try:
        d=json.load(open(f"gpurun_out/{f}.json"))
        print(f, d["value"], d["ms_per_step"], d["breakdown_ms"])
    except Exception as e: print(f, e)
PY
