python -m pytest tests/test_gpu_lower_bound.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_stale.py tests/test_gpu_slabs.py tests/test_gpu_edge.py -q -x -p no:cacheprovider > gpurun_out/lb_tests2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/lb_tests2.log; tail -4 gpurun_out/lb_tests2.log
rm -f gpurun_out/ab_*.log
bash tools/gpu_ab.sh noproplb
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.log')):
    for l in open(f):
        if l.startswith('{"config"'):
            d=json.loads(l); print(f, d['summary']['propagate']['ms'], d['summary']['random_search']['ms'], [k['ms'] for k in d['kernels'] if k['kernel'].startswith('propagate_k1_') or k['kernel'].startswith('propagate_k7_')])
PY
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_lb2.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_lb2.log | cut -c1-400
VINP_LIB_PATH=build_variants/noproplb.so python bench.py --steps 3 --warmup 3 > gpurun_out/bench_lb2_noprop.log 2>&1; tail -1 gpurun_out/bench_lb2_noprop.log | cut -c1-400
