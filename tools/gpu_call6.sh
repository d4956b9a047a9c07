cd $GRAFT_REPO_ROOT/paper_2405_18966_b200
cp libsvdsc.so libsvdsc_default.so
cd ..
for cfg in "--workload 4 --reps 5" "--workload 3 --reps 20" "--workload 5 --scale 8 --reps 5" "--workload 1 --reps 50"; do
  for sp in bins merge; do python tools/profile_ops.py $cfg --skip-cgs --spmv $sp --tag base 2>&1 | tail -1; done
  for v in k8p1b3 k8p0b3 k8p1b2 k4p1b4 k4p0b5 k8p0b4; do
    cp paper_2405_18966_b200/libsvdsc_$v.so paper_2405_18966_b200/libsvdsc.so
    python tools/profile_ops.py $cfg --skip-cgs --spmv seg --tag $v 2>&1 | tail -1
  done
  cp paper_2405_18966_b200/libsvdsc_default.so paper_2405_18966_b200/libsvdsc.so
done
