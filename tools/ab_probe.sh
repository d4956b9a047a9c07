mkdir -p gpurun_out
for v in libsvdsc_ve.so libsvdsc_vf.so libsvdsc_ve.so libsvdsc_vf.so; do
  SVDSC_LIB_VARIANT=$v SVDSC_KTIMING=1 timeout 120 python tools/probe_cgs2.py 200000 300 2>&1 | grep -E "median|ktiming"
done
