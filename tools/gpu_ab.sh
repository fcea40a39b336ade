# A/B of libvinp variants on the level-1 pass timings (tools/prof_kernels.py); usage: gpu_ab.sh v1 v2 ...
for i in 1 2; do
  python tools/prof_kernels.py > gpurun_out/ab_default_$i.log 2>&1
  for v in "$@"; do
    VINP_LIB_PATH=build_variants/$v.so python tools/prof_kernels.py > gpurun_out/ab_${v}_$i.log 2>&1
  done
done
