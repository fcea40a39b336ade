"""Edge and degenerate cases of the whole pipeline (Alg. 4), GPU (C ABI) vs oracle, bit for bit:
no occlusion at all (empty H, H~ and target lists), a single-voxel hole, a volume barely larger than
one patch, whole frames occluded (temporal holes crossing every patch of those frames), and the
"no source" case that both sides must refuse (D~ empty)."""
import numpy as np
import pytest
import torch

from gen.synth import random_volume

pytestmark = pytest.mark.gpu


def _both(orc, v, m, levels, **kw):
    from paper_1503_05528_b200 import Config, inpaint
    cfg = Config(levels=levels, **kw)
    out, stats, _ = inpaint(torch.from_numpy(v), torch.from_numpy(m), cfg, device="cuda")
    ref, st = orc.inpaint(v, m, levels, pm_iters=cfg.pm_iters, fixed_outer=cfg.fixed_outer,
                          max_outer=cfg.max_outer)
    g = out.cpu().numpy()
    assert np.array_equal(g, ref)
    assert [l["outer"] for l in stats.levels] == st["outer_iters"]
    assert stats.total_patch_updates + stats.total_stale_skipped == sum(st["patch_updates"])
    assert stats.total_stale_skipped == sum(st["stale"])
    assert np.array_equal(g[m == 0], v[m == 0])
    return g, stats


def _vol(W, H, T, seed):
    v, m, _ = random_volume(W, H, T, seed=seed)
    return v.numpy(), m.numpy()


def test_no_occlusion_is_identity(orc):
    v, _ = _vol(24, 20, 8, 1)
    g, stats = _both(orc, v, np.zeros(v.shape[:3], np.uint8), 1, pm_iters=2, max_outer=2)
    assert stats.total_patch_updates == 0 and np.array_equal(g, v)


def test_single_voxel_hole(orc):
    v, _ = _vol(24, 20, 8, 1)
    m = np.zeros(v.shape[:3], np.uint8)
    m[4, 10, 12] = 1
    _both(orc, v, m, 1, pm_iters=2, max_outer=2)


def test_tiny_volume(orc):
    v, m = _vol(12, 10, 5, 2)
    _both(orc, v, m, 1, pm_iters=2, max_outer=2)


def test_whole_frames_occluded(orc):
    v, m = _vol(24, 20, 12, 1)
    m[5:7] = 1
    _both(orc, v, m, 2, pm_iters=2, max_outer=3)


def test_no_source_is_refused(orc):
    from paper_1503_05528_b200 import Config, inpaint
    from paper_1503_05528_b200.vinp import VinpError
    v, m = _vol(24, 20, 8, 1)
    m[3:5] = 1  # every 5-frame window of an 8-frame video meets frame 3 or 4: D~ is empty
    with pytest.raises(RuntimeError):
        orc.inpaint(v, m, 1, pm_iters=2, max_outer=2)
    with pytest.raises(VinpError):
        inpaint(torch.from_numpy(v), torch.from_numpy(m), Config(levels=1, pm_iters=2, max_outer=2), device="cuda")
