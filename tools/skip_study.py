"""Study (dev): how many propagation candidates of one ANN search are *stale*, i.e. proposed by a
neighbour whose NNF entry has not changed since the previous pass with the same (step, sign) of
the same ANN search.  Such a candidate was already tested against this target (or equalled its
incumbent) and the target's D has not increased since, so it can never be accepted (strict
improvement, R25).  Prints per pass: targets changed, candidates proposed, stale candidates, and
the fraction of 32-slot warps in which every candidate is stale.

  python tools/skip_study.py [--config c5] [--level 1]
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
    ap.add_argument("--level", type=int, default=1)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    v, m, _ = generate(args.config, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, lam=c.lam, seed=c.seed), "cuda")
    ip.load(v, m)
    ip.onion_peel()
    for l in range(c.levels, args.level, -1):
        s_, f_ = ip.states[l - 1], ip.states[l - 2]
        ip.ann_search(s_, 0)
        ip.reconstruct(s_, V.WEIGHTED)
        V.nnf_upsample(s_.lv, s_.a, f_.lv, f_.a, ip.prm)
        ip.reconstruct(f_, V.UNWEIGHTED)
    st = ip.states[args.level - 1]
    lv = st.lv
    n = lv.n_targets
    W, H, T = lv.W, lv.H, lv.T
    tg = lv.targets[:n].long()
    x, y, t = tg % W, (tg // W) % H, tg // (W * H)
    flags = lv.flags
    slot = lv.slot
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    V.nnf_evaluate(lv, st.a, ip.prm, counter=cnt)
    hist = {}  # (step, sign) -> e before that pass
    rows = []
    e_prev = st.a.e[:n].clone()
    for k in range(1, 11):
        sign = 1 if k % 2 else -1
        for s in (8, 4, 2, 1):
            ein = st.a.e[:n].clone()
            q_in = (ein & 0xFFFFFFFF).long()
            prop = torch.zeros(n, dtype=torch.int32, device="cuda")
            stale = torch.zeros(n, dtype=torch.int32, device="cuda")
            old = hist.get((s, sign))
            for ax in range(3):
                ox, oy, ot = [(sign * s if a == ax else 0) for a in range(3)]
                rx, ry, rt = x + ox, y + oy, t + ot
                ok = (rx >= 0) & (rx < W) & (ry >= 0) & (ry < H) & (rt >= 0) & (rt < T)
                r = torch.where(ok, (rt * H + ry) * W + rx, torch.zeros_like(rx))
                rs = torch.where(ok, slot[r].long(), torch.full_like(rx, -1))
                ok = rs >= 0
                src = (ein[rs.clamp(min=0)] & 0xFFFFFFFF).long()
                sx, sy, stt = src % W, (src // W) % H, src // (W * H)
                qx, qy, qt = sx - ox, sy - oy, stt - ot
                inb = (qx >= 0) & (qx < W) & (qy >= 0) & (qy < H) & (qt >= 0) & (qt < T)
                q = (qt * H + qy) * W + qx
                val = ok & inb & ((flags[q.clamp(0, W * H * T - 1)] & 2) != 0) & (q != q_in)
                prop += val.int()
                if old is not None:
                    same = (old[rs.clamp(min=0)] & 0xFFFFFFFF) == (ein[rs.clamp(min=0)] & 0xFFFFFFFF)
                    stale += (val & same).int()
            hist[(s, sign)] = ein
            cnt.zero_()
            V.propagate(lv, st.a, st.b, ip.prm, s, sign, counter=cnt)
            st.a, st.b = st.b, st.a
            changed = int(((st.a.e[:n] & 0xFFFFFFFF) != (ein & 0xFFFFFFFF)).sum())
            live = prop - stale
            nw = (n + 31) // 32
            pad = torch.zeros(nw * 32, dtype=torch.int32, device="cuda")
            pad[:n] = live
            warp_idle = float((pad.view(nw, 32).amax(1) == 0).float().mean())
            padp = torch.zeros(nw * 32, dtype=torch.int32, device="cuda")
            padp[:n] = prop
            warp_idle0 = float((padp.view(nw, 32).amax(1) == 0).float().mean())
            rows.append(dict(k=k, s=s, sign=sign, counted=int(cnt.item()), proposed=int(prop.sum()),
                             stale=int(stale.sum()), changed=changed,
                             warps_all_stale=round(warp_idle, 4), warps_no_cand=round(warp_idle0, 4)))
            print(json.dumps(rows[-1]), flush=True)
        cnt.zero_()
        ein = st.a.e[:n].clone()
        V.random_search(lv, st.a, st.b, ip.prm, 0, k, counter=cnt)
        st.a, st.b = st.b, st.a
        changed = int(((st.a.e[:n] & 0xFFFFFFFF) != (ein & 0xFFFFFFFF)).sum())
        print(json.dumps(dict(k=k, rs=True, counted=int(cnt.item()), changed=changed)), flush=True)
    tot_p = sum(r["proposed"] for r in rows)
    tot_s = sum(r["stale"] for r in rows)
    print(json.dumps(dict(config=args.config, level=args.level, targets=n, proposed=tot_p, stale=tot_s,
                          stale_frac=round(tot_s / max(tot_p, 1), 4))))


if __name__ == "__main__":
    main()
