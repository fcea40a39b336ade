"""Seeded fuzz of the whole pipeline (Alg. 4), GPU through the C ABI vs the oracle, bit for bit:
random odd sizes, ellipsoidal holes that may cross the volume border, lambda in [0, 126], 1-3
pyramid levels, jump-step schedules and both sign policies, random-search ratios rho (so every
candidate-count instantiation of the random-search kernel runs), texture window widths, the
stopping rule or fixed outer iteration counts.  Cases whose D~ is empty must be refused by both sides."""
import numpy as np
import pytest
import torch

from gen.synth import random_holes, random_volume

pytestmark = pytest.mark.gpu

STEPS = [(8, 4, 2, 1), (4, 2, 1), (2, 1), (16, 8, 4, 2, 1), (1,)]


def _case(i):
    rng = np.random.default_rng(1000 + i)
    W, H, T = int(rng.integers(13, 66)), int(rng.integers(11, 50)), int(rng.integers(6, 15))
    levels = int(rng.integers(1, 4)) if min(W, H) >= 16 else 1
    return dict(W=W, H=H, T=T, levels=levels, lam=int(rng.choice([0, 1, 50, 126, int(rng.integers(0, 127))])),
                steps=STEPS[int(rng.integers(0, len(STEPS)))], sign_policy=int(rng.integers(0, 2)),
                pm_iters=int(rng.integers(1, 4)), fixed_outer=int(rng.choice([0, 0, 2])),
                nholes=int(rng.integers(1, 4)), seed=int(rng.integers(1, 1 << 30)),
                rho=float(rng.choice([0.5, 0.5, 0.62, 0.75, 0.85])), tex_half=int(rng.choice([-1, -1, 0, 2])))


@pytest.mark.parametrize("i", range(24))
def test_pipeline_fuzz(orc, i):
    from paper_1503_05528_b200 import Config, inpaint
    from paper_1503_05528_b200.vinp import VinpError
    c = _case(i)
    v, _, _ = random_volume(c["W"], c["H"], c["T"], seed=c["seed"] % 1000 + 1)
    m = random_holes(c["W"], c["H"], c["T"], c["seed"], c["nholes"])
    v = v.clone()
    v[m.bool()] = 0
    cfg = Config(levels=c["levels"], pm_iters=c["pm_iters"], fixed_outer=c["fixed_outer"], max_outer=4,
                 lam=c["lam"], seed=c["seed"], steps=c["steps"], sign_policy=c["sign_policy"], rho=c["rho"],
                 tex_half=c["tex_half"])
    try:
        ref, st = orc.inpaint(v.numpy(), m.numpy(), c["levels"], pm_iters=c["pm_iters"],
                              fixed_outer=c["fixed_outer"], max_outer=4, lam=c["lam"], seed=c["seed"],
                              steps=c["steps"], sign_policy=c["sign_policy"], rho=c["rho"],
                              tex_half=c["tex_half"])
    except RuntimeError:
        with pytest.raises(VinpError):
            inpaint(v, m, cfg, device="cuda")
        return
    out, stats, _ = inpaint(v, m, cfg, device="cuda")
    assert np.array_equal(out.cpu().numpy(), ref), c
    assert [l["outer"] for l in stats.levels] == st["outer_iters"], c
    assert stats.total_patch_updates + stats.total_stale_skipped == sum(st["patch_updates"]), c
    assert stats.total_stale_skipped == sum(st["stale"]), c


@pytest.mark.parametrize("i", range(6))
def test_aligned_pipeline_fuzz(orc, i):
    """realign -> inpaint (with the invalid set X) -> unwarp, random camera motion and holes"""
    from gen.synth import camera_video
    from paper_1503_05528_b200 import Config, inpaint
    rng = np.random.default_rng(2000 + i)
    W, H, T = int(rng.integers(40, 90)), int(rng.integers(32, 64)), int(rng.integers(6, 12))
    c = np.array([0.0, 1, 0, 0, 0, 1])
    cams = []
    for _ in range(T):
        cams.append(c.copy())
        a = rng.uniform(-0.01, 0.01)
        c = c + np.array([rng.uniform(-2, 2), 0, 0, rng.uniform(-1.5, 1.5), 0, 0])
        c[1], c[2], c[4], c[5] = np.cos(a), -np.sin(a), np.sin(a), np.cos(a)
    v = camera_video(W, H, T, int(rng.integers(1, 1000)), cams, noise=1.0).numpy()
    m = random_holes(W, H, T, int(rng.integers(1, 1 << 30)), 2).numpy()
    v[m.astype(bool)] = 0
    levels = int(rng.integers(1, 3))
    cfg = Config(levels=levels, pm_iters=2, max_outer=3, align=True)
    ar, am, fwd, inv, pairs, st = orc.align_pipeline(v, m)
    try:
        o_out, o_st = orc.inpaint(ar, am, levels, pm_iters=2, max_outer=3)
    except RuntimeError:
        pytest.skip("no source after realignment")
    out, stats, ip = inpaint(torch.from_numpy(v), torch.from_numpy(m), cfg, device="cuda")
    assert np.array_equal(ip.align_info["theta"].cpu().numpy(), pairs)
    assert np.array_equal(out.cpu().numpy(), orc.unwarp(o_out, v, m, fwd))
    assert [l["outer"] for l in stats.levels] == o_st["outer_iters"]
