python -m pytest tests/test_gpu_active.py tests/test_gpu_lower_bound.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_stale.py tests/test_gpu_slabs.py tests/test_gpu_edge.py -q -x -p no:cacheprovider > gpurun_out/t14.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t14.log; tail -4 gpurun_out/t14.log
python tools/prof_kernels.py > gpurun_out/prof14.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof14.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print(d['summary'])
PY
python bench.py --steps 3 --warmup 3 > gpurun_out/bench14.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench14.log | cut -c1-330
