"""Exact-NN (a13) timing: CUDA-core early-abort brute force vs the tcgen05 tensor-core form."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, Inpainter, vinp as V  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = CONFIGS[name]
v, m, _ = generate(name, device="cuda")
ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, lam=c.lam, seed=c.seed), "cuda")
ip.load(v, m)
lv = ip.levels[0]
n = lv.n_targets if len(sys.argv) < 3 else min(lv.n_targets, int(sys.argv[2]))
res = {"config": name, "targets": n, "sources": lv.n_sources}
outs = {}
for kind, fn in (("tensor_core", V.brute_force_tc), ("cuda_core", V.brute_force)):
    x = V.NNF.alloc(lv.n_targets, "cuda")
    fn(lv, x, ip.prm, 0, min(n, 256))  # warm-up
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record()
    fn(lv, x, ip.prm, 0, n)
    b.record()
    torch.cuda.synchronize()
    res[kind + "_s"] = a.elapsed_time(b) / 1000
    outs[kind] = x
pairs = n * lv.n_sources
res["pairs"] = pairs
res["equal"] = bool(torch.equal(outs["tensor_core"].e[:n], outs["cuda_core"].e[:n]))
res["tc_TOPS_int8"] = 2 * pairs * 640 / res["tensor_core_s"] / 1e12
print(json.dumps(res))
