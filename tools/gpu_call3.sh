cd $GRAFT_REPO_ROOT
export SVDSC_OPCGS_FUSED=1t
python tools/profile_ops.py --workload 4 --reps 5 > gpurun_out/r02_ops_c4.json 2> gpurun_out/r02_ops_c4.err && cat gpurun_out/r02_ops_c4.json
python tools/profile_ops.py --workload 3 --reps 10 --cgs-cols 200 2>&1 | tail -1
python tools/profile_ops.py --workload 4 --reps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_spmv_merge|k_spmv_bins|k_cgs2_stream2" -c 8 -o gpurun_out/r02_c4_ops python tools/profile_ops.py --workload 4 --reps 1 > gpurun_out/r02_c4_ncu.log 2>&1; tail -3 gpurun_out/r02_c4_ncu.log
