python -m pytest tests/test_gpu_lower_bound.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_stale.py -q -x -p no:cacheprovider > gpurun_out/t11.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t11.log; tail -3 gpurun_out/t11.log
python tools/prof_kernels.py > gpurun_out/prof11.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof11.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print(d['summary'])
PY
