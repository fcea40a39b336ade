"""NEXT #1 timing: realignment stages on a bench config (device time, CUDA events).

Reports, per config: affine estimate (all T-1 pairs, one CTA each), chain, warp, unwarp, the
IRLS iteration counts, and the pixel-iterations / s of the estimate (pixels of the finest level x
IRLS iterations there, + the coarser levels).  Optionally the whole aligned Alg. 4.
usage: python tools/align_bench.py [--configs c4,c5] [--full]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, inpaint, vinp as V  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps):
        ev[0].record()
        r = fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return min(ts), r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c4,c5")
    ap.add_argument("--full", action="store_true", help="also time the whole aligned Alg. 4")
    args = ap.parse_args()
    out = []
    for name in args.configs.split(","):
        c = CONFIGS[name]
        v, m, _ = generate(name, device="cuda")
        T = c.T
        ws = torch.empty(V.affine_ws_bytes(c.W, c.H, T, 3), dtype=torch.uint8, device="cuda")
        ms_est, (th, st, it) = timed(lambda: V.affine_estimate(v, m, ws=ws))
        ms_chain, (fwd, inv, err) = timed(lambda: V.affine_chain(th, T))
        ms_warp, (ar, am) = timed(lambda: V.align_warp(v, m, inv))
        ms_unwarp, _ = timed(lambda: V.unwarp(ar, v, m, fwd))
        th_h = th.cpu()
        rec = dict(config=name, dims=[c.W, c.H, T], pairs=T - 1, estimate_ms=round(ms_est, 3),
                   chain_ms=round(ms_chain, 3), warp_ms=round(ms_warp, 3), unwarp_ms=round(ms_unwarp, 3),
                   iters_total=int(it.sum().item()), iters_max=int(it.max().item()),
                   degenerate=int(st.sum().item()),
                   mean_translation=[round(float(th_h[:, 0].mean()), 4), round(float(th_h[:, 3].mean()), 4)],
                   invalid_frac=round(float((am == 2).float().mean().item()), 4))
        if args.full:
            cfg = Config(levels=c.levels, pm_iters=c.pm_iters, max_outer=c.max_outer, lam=c.lam, seed=c.seed,
                         align=True)
            inpaint(v, m, cfg)
            torch.cuda.synchronize()
            ms_full, (o, stats, ip) = timed(lambda: inpaint(v, m, cfg), reps=1)
            rec["aligned_inpaint_s"] = round(ms_full / 1e3, 3)
            rec["outer_per_level"] = [l["outer"] for l in stats.levels]
        print(json.dumps(rec), flush=True)
        out.append(rec)
    return out


if __name__ == "__main__":
    main()
