# R42 lower bound: new tests, parity + fuzz + stale + slabs, then level-1 timings
python -m pytest tests/test_gpu_lower_bound.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_stale.py tests/test_gpu_slabs.py tests/test_gpu_edge.py -x -q -p no:cacheprovider > gpurun_out/lb_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/lb_tests.log; tail -15 gpurun_out/lb_tests.log
python tools/prof_kernels.py > gpurun_out/prof_lb.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof_lb.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print(d['summary']); print([(k['kernel'],k['ms']) for k in d['kernels'] if 'random' in k['kernel'] or k['kernel'] in ('evaluate','reconstruct')])
PY
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_lb.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_lb.log | cut -c1-900
