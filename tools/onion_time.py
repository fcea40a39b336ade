"""Onion-peel (Alg. 3) time at the coarsest level of c5 and c4, three runs each (CUDA events).
usage: python tools/onion_time.py"""
import sys, torch
sys.path.insert(0, '/root/repo')
from gen.synth import CONFIGS, generate
from paper_1503_05528_b200 import Config, Inpainter
for name in ("c5", "c4"):
    c = CONFIGS[name]
    v, m, _ = generate(name, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, pm_iters=c.pm_iters, lam=c.lam, seed=c.seed), "cuda")
    ts = []
    for r in range(3):
        ip.load(v, m)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); ip.onion_peel(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(name, "onion ms", [round(t, 2) for t in ts])
