# A/B of library variants (libsvdsc_*.so built with SVDSC_NVCC_EXTRA / patched
# sources) on one streaming CGS2 shape, phase counters included
mkdir -p gpurun_out
for v in ${VARIANTS:-libsvdsc.so}; do
  SVDSC_LIB_VARIANT=$v SVDSC_KTIMING=1 timeout 120 python tools/probe_cgs2.py ${N:-200000} ${C:-300} 2>&1 | grep -E "median|ktiming"
done
