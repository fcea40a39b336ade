python -m pytest tests/test_gpu_lower_bound.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_stale.py tests/test_gpu_slabs.py tests/test_gpu_edge.py tests/test_gpu_abi_errors.py -q -p no:cacheprovider > gpurun_out/lb_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/lb_tests.log; tail -6 gpurun_out/lb_tests.log
bash tools/gpu_ab.sh rec_pf0 rec_pf1_m3 rec_pf1_w1 rec_pf0_w1 rec_pf1_m3_w1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    for l in open(f):
        if l.startswith('{"config"'):
            d=json.loads(l); print(f, [k['ms'] for k in d['kernels'] if k['kernel']=='reconstruct'], d['summary']['random_search']['ms'])
PY
