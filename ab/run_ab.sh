# same-box A/B of two library builds (ab/libsvdsc_old.so vs ab/libsvdsc_new.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp ab/libsvdsc_new.so paper_2405_18966_b200/libsvdsc.so
timeout 900 python -m pytest tests/test_gpu_deferred.py tests/test_gpu_determinism.py tests/test_gpu_peer.py -q -m gpu -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
for v in old new old new; do
  cp ab/libsvdsc_$v.so paper_2405_18966_b200/libsvdsc.so
  echo "== $v"
  timeout 600 python tools/ab_policy.py --workload 3 --solves 3 "" 2>&1 | grep -o '"ms_per_solve": [0-9.]*\|"cgs2_fused": [0-9.]*' | tr '\n' ' '; echo
  timeout 600 python tools/ab_policy.py --workload 4 --solves 2 "" 2>&1 | grep -o '"ms_per_solve": [0-9.]*\|"cgs2_fused": [0-9.]*\|"Av": [0-9.]*' | tr '\n' ' '; echo
done
cp ab/libsvdsc_new.so paper_2405_18966_b200/libsvdsc.so
