# session 3: reconstruct v2 parity + timing + ncu source counts; random-search lower-bound study
python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "reconstruct or pipeline or onion" > gpurun_out/rec_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rec_tests.log; tail -3 gpurun_out/rec_tests.log
python tools/prof_kernels.py > gpurun_out/prof_v2.log 2>&1; python - <<'PY'
import json
for l in open('gpurun_out/prof_v2.log'):
    if l.startswith('{"config"'):
        d=json.loads(l); print(d['summary']); print([k for k in d['kernels'] if k['kernel']=='reconstruct'])
PY
python tools/lb_study.py > gpurun_out/lb_study.log 2>&1; cut -c1-400 gpurun_out/lb_study.log
ncu --set full --clock-control none --import-source on -k regex:k_reconstruct -s 27 -c 1 -o gpurun_out/prof_rec_v2 python tools/prof_kernels.py > gpurun_out/ncu_rec.log 2>&1; tail -2 gpurun_out/ncu_rec.log
