set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo rc=$?
for i in 1 2; do
python tools/prof_kernels.py > gpurun_out/prof_fm1_$i.log 2>&1
VINP_LIB_PATH=build_variants/fm0.so python tools/prof_kernels.py > gpurun_out/prof_fm0_$i.log 2>&1
done
