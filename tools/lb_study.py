"""Study (dev): how many random-search candidates (Eq. 3) a patch-sum lower bound would reject
before any patch row is read.

For a full target patch (n = 125) and a source q in D~, Cauchy-Schwarz over a group G of voxels
gives sum_{v in G} (a_v - b_v)^2 >= (S_G(a) - S_G(b))^2 / |G|, so
  D(p, q) = sum 4 |du|^2 + lambda |dT|^2 >= LB(p, q)
for any partition of the patch into groups, with S_G the per-channel sums over the group.  A
candidate with LB >= D_incumbent can never be accepted (strict improvement, R25), exactly like an
early abort (R35).  Variants:
  A  one group (the whole patch), 5 channel sums
  B  5 groups (frames), RGB sums per frame + one (Tx + Ty) sum over the patch
  C  5 groups (frames), all 5 channel sums per frame
Candidates are drawn like Eq. 3 (uniform in the shrinking window around the incumbent) with torch's
RNG (a study, not the Philox schedule).  Prints, per PM iteration probed, the fraction of valid
candidates that lose (D >= D_inc), and that each bound rejects.

  python tools/lb_study.py [--config c5] [--sample 200000]
"""
import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, Inpainter, vinp as V  # noqa: E402


def frame_sums(lv):
    """[5, T, H, W] float32: 5x5 in-frame box sums of R, G, B, Tx, Ty (exact: sums < 2^24)."""
    vox = lv.vox.view(lv.T, lv.H, lv.W)
    out = torch.empty((5, lv.T, lv.H, lv.W), dtype=torch.float32, device=vox.device)
    for c, sh in enumerate((0, 8, 16, 32, 40)):
        ch = ((vox >> sh) & 255).float().unsqueeze(1)  # [T,1,H,W]
        out[c] = (F.avg_pool2d(ch, 5, stride=1, padding=2, count_include_pad=True) * 25.0).round().squeeze(1)
    return out


def half_moments(lv):
    """[3 axes, 5 channels, N] float32: sum of sign(offset along the axis) * channel over the 5x5x5 patch."""
    vox = lv.vox.view(1, 1, lv.T, lv.H, lv.W)
    sgn = torch.tensor([-1.0, -1.0, 0.0, 1.0, 1.0], device=vox.device)
    one = torch.ones(5, device=vox.device)
    ks = []
    for ax in range(3):  # t, y, x kernels [5,5,5]
        w = [one, one, one]
        w[ax] = sgn
        ks.append((w[0].view(5, 1, 1) * w[1].view(1, 5, 1) * w[2].view(1, 1, 5)).view(1, 1, 5, 5, 5))
    out = torch.empty((3, 5, lv.T * lv.H * lv.W), dtype=torch.float32, device=vox.device)
    for c, sh in enumerate((0, 8, 16, 32, 40)):
        ch = ((vox >> sh) & 255).float()
        for ax in range(3):
            out[ax, c] = F.conv3d(ch, ks[ax], padding=2).round().view(-1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--level", type=int, default=1)
    ap.add_argument("--sample", type=int, default=200000)
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
    lam = c.lam
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    rows = []
    V.nnf_evaluate(lv, st.a, ip.prm)
    e0 = st.a.e.clone()
    for probe in (0, 4):  # PM iterations already run when the candidates are drawn
        if probe:
            st.a.e.copy_(e0)
            V.ann_search(lv, st.a, st.b, ip.prm, 0, probe)
        Fs = frame_sums(lv)
        Hm = half_moments(lv)
        sl = torch.arange(args.sample, device="cuda", dtype=torch.int64) * (n // args.sample)
        p = lv.targets[:n][sl].long()
        e = st.a.e[:n][sl]
        q0 = e & 0xFFFFFFFF
        Dinc = (e >> 32) & 0xFFFFFFFF
        px, py, pt = p % W, (p // W) % H, p // (W * H)
        interior = (px >= 2) & (px < W - 2) & (py >= 2) & (py < H - 2) & (pt >= 2) & (pt < T - 2)
        q0x, q0y, q0t = q0 % W, (q0 // W) % H, q0 // (W * H)
        tot = dict(valid=0, lose=0, A=0, B=0, C=0, D=0, E=0, zero=0)
        per_radius = []
        R = float(max(W, H, T))
        i = 0
        while True:
            R *= 0.5
            if R < 1.0:
                break
            i += 1
            u = torch.rand((3, p.numel()), device="cuda", generator=g, dtype=torch.float64) * 2 - 1
            qx = q0x + torch.floor(R * u[0]).long()
            qy = q0y + torch.floor(R * u[1]).long()
            qt = q0t + torch.floor(R * u[2]).long()
            inb = (qx >= 0) & (qx < W) & (qy >= 0) & (qy < H) & (qt >= 0) & (qt < T)
            q = ((qt * H + qy) * W + qx).clamp(0, W * H * T - 1)
            ok = inb & ((lv.flags[q] & 2) != 0) & (q != q0) & interior
            pp, qq, Di = p[ok], q[ok], Dinc[ok]
            D, _ = V.patch_ssd(lv, pp.int(), qq.int(), ip.prm)
            D = D.long()
            HW = H * W
            # per-frame sums of both patches: [5 channels, 5 frames, n]
            sp = torch.stack([Fs.view(5, -1)[:, pp + dt * HW] for dt in range(-2, 3)], 1).double()
            sq = torch.stack([Fs.view(5, -1)[:, qq + dt * HW] for dt in range(-2, 3)], 1).double()
            d = sp - sq
            # A: whole patch, 5 channels: 125 D >= 4 sum_c dS_c^2 + lam sum_T dS_T^2
            dA = d.sum(1)
            lbA = (4 * (dA[:3] ** 2).sum(0) + lam * (dA[3:] ** 2).sum(0)) / 125.0
            # B: per-frame RGB + one (Tx+Ty) total: 250 D >= 40 sum dS_fc^2 + lam dST^2
            dT = dA[3] + dA[4]
            lbB = (40 * (d[:3] ** 2).sum((0, 1)) + lam * dT ** 2) / 250.0
            # C: per-frame, all channels: 25 D >= 4 sum dS_fc^2 + lam sum dS_fT^2
            lbC = (4 * (d[:3] ** 2).sum((0, 1)) + lam * (d[3:] ** 2).sum((0, 1))) / 25.0
            # D: A + half-difference moments (sign(dx), sign(dy), sign(dt)) of R, G, B;  E: of T too
            dH = (Hm[:, :, pp] - Hm[:, :, qq]).double()  # [3, 5, n]
            lbD = lbA + 4 * (dH[:, :3] ** 2).sum((0, 1)) / 100.0
            lbE = lbD + lam * (dH[:, 3:] ** 2).sum((0, 1)) / 100.0
            assert bool((lbE <= D + 1e-6).all())
            assert bool((lbA <= D + 1e-6).all()) and bool((lbB <= D + 1e-6).all()) and bool((lbC <= D + 1e-6).all())
            Dd = Di.double()
            r = dict(i=i, R=R, valid=int(ok.sum()), lose=int((D >= Di).sum()), A=int((lbA >= Dd).sum()),
                     B=int((lbB >= Dd).sum()), C=int((lbC >= Dd).sum()), D=int((lbD >= Dd).sum()),
                     E=int((lbE >= Dd).sum()), zero=int((Di == 0).sum()))
            per_radius.append(r)
            for k in ("valid", "lose", "A", "B", "C", "D", "E", "zero"):
                tot[k] += r[k]
        row = dict(pm_iters_done=probe, targets=int(p.numel()), candidates=tot["valid"],
                   frac_lose=round(tot["lose"] / tot["valid"], 4),
                   reject_A=round(tot["A"] / tot["valid"], 4), reject_B=round(tot["B"] / tot["valid"], 4),
                   reject_C=round(tot["C"] / tot["valid"], 4), reject_D=round(tot["D"] / tot["valid"], 4),
                   reject_E=round(tot["E"] / tot["valid"], 4),
                   frac_incumbent_zero=round(tot["zero"] / tot["valid"], 4), per_radius=per_radius)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del Fs, Hm


if __name__ == "__main__":
    main()
