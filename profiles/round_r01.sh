# round-1 end check on one B200: GPU tests, smoke, benches (ours + reference arm), ncu launch list + full capture
O=gpurun_out/${R01_OUT:-r01c}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $O/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > $O/host.txt; nproc >> $O/host.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo tests_exit=$?
tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_exit=$?; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_config2.json 2> $O/bench_config2.err; echo bench2=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_config2.json 2> $O/bench_ref.err; echo ref=$?
timeout 1200 python bench.py --workload 3 > $O/bench_config3.json 2> $O/bench_config3.err; echo bench3=$?
timeout 1200 python bench.py --workload 4 --steps 3 --no-e2e > $O/bench_config4.json 2> $O/bench_config4.err; echo bench4=$?
timeout 900 python bench.py --workload 6 --steps 3 > $O/bench_dense1.json 2> $O/bench_dense1.err; echo bench6=$?
timeout 900 python bench.py --workload 3 --reorth 1 --steps 3 > $O/bench_config3_pro.json 2> $O/bench_config3_pro.err; echo bench3pro=$?
C3="python bench.py --workload 3 --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_config3.csv $C3 > $O/ncu_launch3.log 2>&1; echo launches3_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cgs2_stream2|k_spmv_bins" -s 400 -c 3 -o $O/prof_config3 $C3 > $O/ncu_full3.log 2>&1; echo full3_exit=$?
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
$CMD > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_config2.csv $CMD > $O/ncu_launch.log 2>&1
echo launches_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemv_t|k_gemv_n|k_cgs2_fused|k_jacobi_block" -s 20 -c 4 -o $O/prof_config2 $CMD > $O/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_jacobi_block|k_apply_log|k_recombine_dmma" -c 3 -o $O/prof_config2_svd $CMD > $O/ncu_full_svd.log 2>&1
echo full_exit=$?
ls -la $O
