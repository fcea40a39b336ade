python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py -q -x -p no:cacheprovider > gpurun_out/t16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t16.log; tail -3 gpurun_out/t16.log
bash tools/gpu_ab.sh sparse32 sparse64 sparse96
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    for l in open(f):
        if l.startswith('{"config"'):
            d=json.loads(l); print(f, d['summary']['propagate']['ms'], d['summary']['reconstruct']['ms'], [k['ms'] for k in d['kernels'] if k['kernel'].startswith('propagate_k1_') or k['kernel'].startswith('propagate_k2_')])
PY
