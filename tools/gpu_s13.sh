python -m pytest tests/test_gpu_active.py tests/test_gpu_stale.py -q -x -p no:cacheprovider > gpurun_out/t13.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t13.log; tail -3 gpurun_out/t13.log
VINP_LIB_PATH=build_variants/rs_noeval.so python tools/prof_kernels.py > gpurun_out/prof13_noeval.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof13_noeval.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print('noeval', d['summary']['random_search'], [k['ms'] for k in d['kernels'] if k['kernel'].startswith('random')])
PY
python bench.py --steps 3 --warmup 3 > gpurun_out/bench13.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench13.log | cut -c1-330
