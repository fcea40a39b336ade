"""Study (dev): at level 1 of c5, after each outer iteration's reconstruction, how many targets have
a patch whose u8 working copy did not change (no changed hole voxel within the 5x5x5 box).  Such
targets see exactly the same distances in the next ANN search."""
import json
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, Inpainter, vinp as V  # noqa: E402
from paper_1503_05528_b200.driver import stop_now  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    c = CONFIGS[name]
    v, m, _ = generate(name, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=c.levels, lam=c.lam, seed=c.seed, graphs=False), "cuda")
    ip.load(v, m)
    ip.onion_peel()
    for l in range(c.levels, 0, -1):
        st = ip.states[l - 1]
        lv = st.lv
        k = 0
        while True:
            before = lv.vox.clone()
            st.prev_rgb.copy_(st.cur_rgb)
            ip.ann_search(st, k)
            ip.reconstruct(st, V.WEIGHTED)
            ip.change.zero_()
            V.change_l1(st.cur_rgb[:lv.n_holes], st.prev_rgb[:lv.n_holes], ip.change)
            k += 1
            ch = (lv.vox != before).view(1, 1, lv.T, lv.H, lv.W).float()
            dil = F.max_pool3d(ch, 5, stride=1, padding=2).view(-1) > 0
            tg = lv.targets[:lv.n_targets].long()
            unchanged = float((~dil[tg]).float().mean())
            print(json.dumps(dict(level=l, outer=k, changed_voxels=int(ch.sum()), holes=lv.n_holes,
                                  targets_unchanged_patch=round(unchanged, 4))), flush=True)
            if stop_now(int(ip.change.item()), lv.n_holes, k, c.max_outer):
                break
        if l > 1:
            f = ip.states[l - 2]
            V.nnf_upsample(lv, st.a, f.lv, f.a, ip.prm)
            ip.reconstruct(f, V.UNWEIGHTED)


if __name__ == "__main__":
    main()
