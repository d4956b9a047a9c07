cd $GRAFT_REPO_ROOT
cp paper_2405_18966_b200/libsvdsc.so /tmp/libsvdsc_default.so
for cfg in "--workload 4 --reps 5" "--workload 3 --reps 20" "--workload 5 --scale 8 --reps 5"; do
  for v in k8f1b3 k8f0b3 k4f1b4 k4f0b5 k8f1b2; do
    cp paper_2405_18966_b200/libsvdsc_$v.so paper_2405_18966_b200/libsvdsc.so
    python tools/profile_ops.py $cfg --skip-cgs --spmv seg --tag $v 2>&1 | tail -1
  done
done
cp /tmp/libsvdsc_default.so paper_2405_18966_b200/libsvdsc.so
