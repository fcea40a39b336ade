bash tools/gpu_ab.sh faststale
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    for l in open(f):
        if l.startswith('{"config"'):
            d=json.loads(l); print(f, d['summary']['propagate'], [k['ms'] for k in d['kernels'] if k['kernel'].startswith('propagate_k1_') or k['kernel'].startswith('propagate_k7_')])
PY
VINP_LIB_PATH=build_variants/faststale.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_stale.py -q -p no:cacheprovider 2>&1 | tail -15
