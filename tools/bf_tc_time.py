"""Exact NN (a13) on the tensor cores only: vinp_brute_force_tc over all level-1 targets of the given
configs after setup, CUDA-event time and effective int8 TOPS (2 * targets * sources * 640 / t).
NOWARM=1 skips the warm-up call (so that `ncu -c 1` captures the main launch).
usage: python tools/bf_tc_time.py c1 c2 [c3]"""
import os, sys, torch, json
sys.path.insert(0, '/root/repo')
from gen.synth import CONFIGS, generate
from paper_1503_05528_b200 import Config, Inpainter, vinp as V
for name in sys.argv[1:]:
    c = CONFIGS[name]
    v, m, _ = generate(name, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, lam=c.lam, seed=c.seed), "cuda")
    ip.load(v, m)
    lv = ip.levels[0]
    x = V.NNF.alloc(lv.n_targets, "cuda")
    if not os.environ.get("NOWARM"):
        V.brute_force_tc(lv, x, ip.prm, 0, 256)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); V.brute_force_tc(lv, x, ip.prm, 0, lv.n_targets); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    macs = lv.n_targets * lv.n_sources * 640
    print(json.dumps({"config": name, "targets": lv.n_targets, "sources": lv.n_sources, "s": ms / 1e3,
                      "int8_TOPS_eff": 2 * macs / (ms / 1e3) / 1e12}))
