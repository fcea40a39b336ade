# round-2 GPU check: the whole -m gpu suite, then the bench
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo rc=$?
python tools/skip_study.py > gpurun_out/skip_c5.log 2>&1
