bash tools/gpu_ab.sh chunk4 chunk4_minb4 minb4 chunk2
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    for l in open(f):
        if l.startswith('{"config"'):
            d=json.loads(l); print(f, d['summary']['propagate']['ms'], d['summary']['random_search']['ms'], [k['ms'] for k in d['kernels'] if k['kernel'].startswith('propagate_k1_') or k['kernel'].startswith('propagate_k7_')])
PY
