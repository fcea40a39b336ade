# final artefacts: bench line, ncu launch list of the bench command (libvinp kernels only: the synthetic
# video generator launches ~30 K torch kernels first), level-1 captures of the final kernels
set -x
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "bench rc=$?"
python bench.py --steps 1 --warmup 3 --no-extra > gpurun_out/plain_noextra.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 30000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-extra > gpurun_out/ncu_launch.log 2>&1
python tools/prof_kernels.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:k_prop_mark -s 110 -c 1 -o gpurun_out/prof_mark_k7 python tools/prof_kernels.py > gpurun_out/ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_evaluate -s 15 -c 1 -o gpurun_out/prof_eval python tools/prof_kernels.py > gpurun_out/ncu6.log 2>&1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
