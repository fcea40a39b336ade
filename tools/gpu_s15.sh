python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py tests/test_gpu_active.py -q -x -p no:cacheprovider > gpurun_out/t15.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t15.log; tail -3 gpurun_out/t15.log
python tools/prof_kernels.py > gpurun_out/prof15.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof15.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print(d['summary'])
PY
python bench.py --steps 3 --warmup 3 > gpurun_out/bench15.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench15.log | cut -c1-330
