mkdir -p gpurun_out
./tools/tma_bw 200000 300 > gpurun_out/tma_bw.log 2>&1; ./tools/tma_bw 100000 300 >> gpurun_out/tma_bw.log 2>&1
./tools/tile_bw 200000 300 > gpurun_out/tile_bw.log 2>&1
cat gpurun_out/tma_bw.log gpurun_out/tile_bw.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "small_svd or products or lbp or forced" > gpurun_out/ops_tests.log 2>&1; echo ops_tests=$?
tail -3 gpurun_out/ops_tests.log
timeout 600 python tools/time_ops.py --cid 3 > gpurun_out/time_ops3.json 2>&1; echo time_ops3=$?
timeout 600 python tools/time_ops.py --cid 2 > gpurun_out/time_ops2.json 2>&1; echo time_ops2=$?
cat gpurun_out/time_ops3.json gpurun_out/time_ops2.json
