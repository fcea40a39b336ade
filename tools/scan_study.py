"""NEXT #2 study: paper-faithful sequential-scan PatchMatch (oracle, CPU) vs the Jacobi jump-flood
schedule (GPU) from the identical level-1 state (first outer iteration), against the exact NN
(tensor-core brute force).  Mean d^2 excess over the exact NN and candidate counts vs iterations K."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle.oracle as orc  # noqa: E402
import oracle_ops as OO  # noqa: E402
from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, Inpainter, vinp as V  # noqa: E402


def state(name):
    c = CONFIGS[name]
    v, m, _ = generate(name, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, pm_iters=c.pm_iters, lam=c.lam, seed=c.seed), "cuda")
    ip.load(v, m)
    ip.onion_peel()
    for l in range(c.levels, 1, -1):
        s_, f_ = ip.states[l - 1], ip.states[l - 2]
        ip.ann_search(s_, 0)
        ip.reconstruct(s_, V.WEIGHTED)
        V.nnf_upsample(s_.lv, s_.a, f_.lv, f_.a, ip.prm)
        ip.reconstruct(f_, V.UNWEIGHTED)
    return ip, c


def mean_d2(e, n):
    D = (e >> 32).double()
    return (D / (4 * n.double())).mean().item()


def main():
    out = []
    for name in sys.argv[1:] or ["c1", "c2"]:
        ip, c = state(name)
        st = ip.states[0]
        lv = st.lv
        nt = lv.n_targets
        e0, n0 = st.a.e.clone(), st.a.n.clone()
        bf = V.NNF.alloc(nt, "cuda")
        V.brute_force_tc(lv, bf, ip.prm)
        V.nnf_evaluate(lv, bf, ip.prm)
        d_bf = mean_d2(bf.e[:nt], bf.n[:nt])
        host = V.Level(lv.W, lv.H, lv.T, 1, torch.device("cpu"))
        for nm in ("vox", "flags", "slot", "targets", "holes", "sources"):
            setattr(host, nm, getattr(lv, nm).cpu())
        host.n_targets, host.n_holes, host.n_sources = lv.n_targets, lv.n_holes, lv.n_sources
        ol = OO._OLevel(host)
        for K in (1, 2, 4, 10):
            row = dict(config=name, K=K, mean_d2_exact=d_bf)
            for pol, tag in ((0, "jacobi_alternate"), (1, "jacobi_both")):
                a = V.NNF(e0.clone(), n0.clone())
                b = V.NNF.alloc(nt, "cuda", n=a.n)
                cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                V.ann_search(lv, a, b, ip.prm, 0, K, counter=cnt, sign_policy=pol)
                row[tag] = dict(excess=mean_d2(a.e[:nt], a.n[:nt]) / d_bf - 1, candidates=int(cnt.item()))
            f = OO._to_orc(host, V.NNF(e0.cpu(), n0.cpu()))
            cnt = orc.ann_search_sequential(ol, f, ip.prm.lam, ip.prm.seed, 1, 0, K)
            d = (f.D[:nt] / (4.0 * f.n[:nt])).mean()
            row["sequential_scan"] = dict(excess=d / d_bf - 1, candidates=int(cnt))
            print(json.dumps(row), flush=True)
            out.append(row)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "scan_study.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
