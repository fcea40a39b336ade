python -m pytest tests/test_gpu_active.py tests/test_gpu_lower_bound.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_stale.py tests/test_gpu_slabs.py tests/test_gpu_edge.py tests/test_bench_contract.py -q -x -p no:cacheprovider > gpurun_out/t12.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t12.log; tail -8 gpurun_out/t12.log
python tools/prof_kernels.py > gpurun_out/prof12.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof12.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print(d['summary']); print([k['ms'] for k in d['kernels'] if k['kernel'].startswith('propagate_k1_') or k['kernel'].startswith('propagate_k7_')])
PY
python bench.py --steps 3 --warmup 3 > gpurun_out/bench12.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench12.log | cut -c1-330
python __graft_entry__.py smoke 2>&1 | tail -2
