"""Per-kernel timing of the level-1 PatchMatch passes on a bench config (default c5), for ncu.

Brings level `--level` to the state of its first outer iteration in Alg. 4 (onion peel, one outer
iteration per coarser level, upsample + unweighted reconstruction; or random init + `--warm`
iterations with --random-init), then times, pass by pass with CUDA events, one evaluate, `--iters`
PatchMatch iterations (4 propagation passes with the R41 stale skip + 1 random search each) and
one weighted reconstruction, and prints per-launch ms, patch-updates, stale skips and model GB/s.
Under ncu, select one timed launch with e.g. (launch counts before it: printed first)
  ncu -k regex:k_random_search -s <rs_launches_before + 4> -c 1 python tools/prof_kernels.py
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, Inpainter, vinp as V  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--level", type=int, default=1)
    ap.add_argument("--iters", type=int, default=10, help="PatchMatch iterations timed (pass by pass)")
    ap.add_argument("--random-init", action="store_true",
                    help="start level 1 from random init + --warm iterations instead of the pipeline")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    v, m, _ = generate(args.config, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, lam=c.lam, seed=c.seed), "cuda")
    ip.load(v, m)
    if args.random_init:
        st = ip.states[args.level - 1]
        V.nnf_init_random(st.lv, st.a, ip.prm, 0)
        V.ann_search(st.lv, st.a, st.b, ip.prm, 0, args.warm)
    else:
        # Alg. 4 down to level `level`: onion peel, one outer iteration per coarser level, upsample
        # + unweighted reconstruction -> the state of the first outer iteration at that level.
        # RS launches before the timed one: (n_layers + 1 + L - level) * K.
        ip.onion_peel()
        for l in range(c.levels, args.level, -1):
            s_, f_ = ip.states[l - 1], ip.states[l - 2]
            ip.ann_search(s_, 0)
            ip.reconstruct(s_, V.WEIGHTED)
            V.nnf_upsample(s_.lv, s_.a, f_.lv, f_.a, ip.prm)
            ip.reconstruct(f_, V.UNWEIGHTED)
        args.warm = 0
    st = ip.states[args.level - 1]
    lv = st.lv
    torch.cuda.synchronize()
    if not args.random_init:
        print(json.dumps(dict(rs_launches_before=(ip.n_layers + 1 + c.levels - args.level) * 10,
                              prop_launches_before=(ip.n_layers + 1 + c.levels - args.level) * 40,
                              rec_launches_before=ip.n_layers + 2 * (c.levels - args.level))))
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")  # evaluated, stale skipped (R41)
    res = []

    def timed(name, fn, slots, per_slot=29):
        cnt.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        pu = int(cnt[0].item())
        by = 625 * pu + per_slot * slots
        res.append(dict(kernel=name, ms=round(ms, 3), patch_updates=pu, stale=int(cnt[1].item()),
                        model_GBps=round(by / ms / 1e6, 1),
                        pu_per_s=round(pu / ms * 1e3 / 1e9, 3)))

    n = lv.n_targets
    timed("evaluate", lambda: V.nnf_evaluate(lv, st.a, ip.prm, counter=cnt), n)
    clk = V.PassClock()
    for k in range(args.warm + 1, args.warm + 1 + args.iters):
        sign = 1 if k % 2 else -1
        for s in (8, 4, 2, 1):
            timed(f"propagate_k{k}_s{s}", lambda: V.propagate(lv, st.a, st.b, ip.prm, s, sign, counter=cnt,
                                                           pass_id=clk.pass_id, since=clk.since(s, sign)), n)
            clk.tick(s, sign)
            st.a, st.b = st.b, st.a
        timed(f"random_search_k{k}", lambda: V.random_search(lv, st.a, st.b, ip.prm, 0, k, counter=cnt,
                                                             pass_id=clk.pass_id), n)
        clk.tick()
        st.a, st.b = st.b, st.a
    nh = lv.n_holes
    timed("reconstruct", lambda: V.reconstruct(lv, st.a, V.WEIGHTED, st.cur_rgb, st.cur_tex), nh, 662)
    agg = {}
    for r in res:
        key = r["kernel"].split("_k")[0]
        a = agg.setdefault(key, dict(ms=0.0, launches=0, patch_updates=0))
        a["ms"] += r["ms"]
        a["launches"] += 1
        a["patch_updates"] += r["patch_updates"]
    print(json.dumps(dict(config=args.config, level=args.level, targets=n, holes=nh, kernels=res,
                          summary={k: dict(v, ms=round(v["ms"], 3)) for k, v in agg.items()})))


if __name__ == "__main__":
    main()
