# round-end style check: full -m gpu suite, the bench, its ncu launch list (libvinp kernels only: the
# synthetic video generator launches ~30 K torch kernels first), ncu --set full of the level-1 kernels
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "bench rc=$?"
python bench.py --steps 1 --warmup 3 --no-extra > gpurun_out/plain_noextra.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 30000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-extra > gpurun_out/ncu_launch.log 2>&1
python tools/prof_kernels.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1025 -c 1 -o gpurun_out/prof_prop_k7 python tools/prof_kernels.py > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_random_search -s 256 -c 1 -o gpurun_out/prof_rs_k7 python tools/prof_kernels.py > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reconstruct -s 27 -c 1 -o gpurun_out/prof_rec python tools/prof_kernels.py > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_propagate -s 1000 -c 1 -o gpurun_out/prof_prop_k1 python tools/prof_kernels.py > gpurun_out/ncu4.log 2>&1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
