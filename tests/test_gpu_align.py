"""GPU parity of NEXT #1 (affine realignment, Alg. 2; S3.4 P:744-758; R36-R40) against
the oracle, through the C ABI: bit-exact theta / status / iteration counts, chain, warp (colour and
mask codes), unwarp, and the whole aligned Alg. 4 (realign -> inpaint with the invalid set X ->
unwarp) on a panning video."""
import numpy as np
import pytest
import torch

from gen.synth import CONFIGS, camera_video, generate

pytestmark = pytest.mark.gpu

ID = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 1.0])


def _moving_video(W=128, H=96, T=7, seed=3):
    rng = np.random.default_rng(seed)
    cams, c = [], ID.copy()
    for t in range(T):
        cams.append(c.copy())
        a, sc = rng.uniform(-0.01, 0.01), 1 + rng.uniform(-0.005, 0.005)
        step = np.array([rng.uniform(-3, 3), np.cos(a) * sc, -np.sin(a) * sc, rng.uniform(-2, 2),
                         np.sin(a) * sc, np.cos(a) * sc])
        M = lambda t_: np.array([[t_[1], t_[2], t_[0]], [t_[4], t_[5], t_[3]], [0, 0, 1.0]])
        P = M(c) @ M(step)
        c = np.array([P[0, 2], P[0, 0], P[0, 1], P[1, 2], P[1, 0], P[1, 1]])
    v = camera_video(W, H, T, seed, cams, noise=1.5, block=(30, 20, 40, 30, 2, -1)).numpy()
    m = np.zeros((T, H, W), np.uint8)
    yy, xx = np.mgrid[0:H, 0:W]
    for t in range(T):
        m[t] = (((xx - (70 + 2 * t)) / 14.0) ** 2 + ((yy - 50) / 10.0) ** 2 <= 1)
    v[m.astype(bool)] = 0
    return v, m


def _gpu_estimate(v, m, **kw):
    from paper_1503_05528_b200 import vinp as V
    th, st, it = V.affine_estimate(torch.from_numpy(v).cuda(), torch.from_numpy(m).cuda(), **kw)
    return th.cpu().numpy(), st.cpu().numpy(), it.cpu().numpy()


def _check_pairs(orc, v, m, pairs, th, st, it, levels=3):
    for n in pairs:
        o_th, o_st, o_it = orc.affine_estimate(v[n], v[n + 1], m[n], m[n + 1], levels)
        assert np.array_equal(th[n], o_th), (n, th[n], o_th)
        assert st[n] == o_st and it[n] == o_it, (n, st[n], o_st, it[n], o_it)


def test_estimate_bit_exact_small(orc):
    v, m = _moving_video()
    th, st, it = _gpu_estimate(v, m)
    _check_pairs(orc, v, m, range(v.shape[0] - 1), th, st, it)
    assert (st == 0).all()


@pytest.mark.parametrize("levels", [1, 2, 4])
def test_estimate_bit_exact_levels(orc, levels):
    v, m = _moving_video(T=3, seed=levels)
    th, st, it = _gpu_estimate(v, m, levels=levels)
    _check_pairs(orc, v, m, range(2), th, st, it, levels)


def test_estimate_degenerate_and_identical(orc):
    v = np.full((3, 40, 48, 3), 77, np.uint8)
    v[2] = camera_video(48, 40, 1, 2, [ID]).numpy()[0]
    m = np.zeros((3, 40, 48), np.uint8)
    th, st, it = _gpu_estimate(v, m)
    assert st[0] == 1 and np.array_equal(th[0], ID)
    _check_pairs(orc, v, m, range(2), th, st, it)


def test_estimate_c4_sampled_pairs(orc):
    """c4 (1280x720, the panning workload): bit-exact on sampled pairs of the full-size launch."""
    v, m, _ = generate("c4", device="cuda")
    from paper_1503_05528_b200 import vinp as V
    th, st, it = V.affine_estimate(v, m)
    th, st, it = th.cpu().numpy(), st.cpu().numpy(), it.cpu().numpy()
    vh, mh = v.cpu().numpy(), m.cpu().numpy()
    T = vh.shape[0]
    _check_pairs(orc, vh, mh, [0, T // 2, T - 2], th, st, it)
    # every pair recovers the pan: theta ~ translation (-2, 0)
    assert (st == 0).all()
    assert np.abs(th[:, 0] + 2).max() < 0.05 and np.abs(th[:, 3]).max() < 0.05


def test_chain_warp_unwarp_bit_exact(orc):
    from paper_1503_05528_b200 import vinp as V
    v, m = _moving_video(T=6, seed=9)
    vd, md = torch.from_numpy(v).cuda(), torch.from_numpy(m).cuda()
    th, st, it = V.affine_estimate(vd, md)
    fwd, inv, err = V.affine_chain(th, 6)
    o_fwd, o_inv = orc.affine_chain(th.cpu().numpy(), 6)
    assert int(err.item()) == 0
    assert np.array_equal(fwd.cpu().numpy(), o_fwd) and np.array_equal(inv.cpu().numpy(), o_inv)
    ar, am = V.align_warp(vd, md, inv)
    o_ar, o_am = orc.align_warp(v, m, o_inv)
    assert np.array_equal(ar.cpu().numpy(), o_ar) and np.array_equal(am.cpu().numpy(), o_am)
    assert (o_am == 2).any() and (o_am == 1).any()
    rng = np.random.default_rng(0)
    inp = rng.integers(0, 256, v.shape, dtype=np.uint8)
    out = V.unwarp(torch.from_numpy(inp).cuda(), vd, md, fwd)
    assert np.array_equal(out.cpu().numpy(), orc.unwarp(inp, v, m, o_fwd))


def test_chain_single_frame_and_pair():
    from paper_1503_05528_b200 import vinp as V
    for T in (1, 2):
        th = torch.tensor(np.tile([1.0, 1, 0, 2.0, 0, 1], (max(T - 1, 1), 1)), device="cuda")
        fwd, inv, err = V.affine_chain(th[:T - 1] if T > 1 else th[:0], T)
        assert np.array_equal(fwd.cpu().numpy()[0], ID)


def test_aligned_inpainting_end_to_end(orc):
    """Alg. 4 with realignment: GPU inpaint(cfg.align=True) == oracle (align -> or_inpaint with
    invalid codes -> unwarp), bit for bit, including per-level outer iterations and counts."""
    from paper_1503_05528_b200 import Config, inpaint
    T, W, H = 10, 96, 64
    cams = [np.array([1.5 * t, 1, 0, -0.5 * t, 0, 1]) for t in range(T)]
    v = camera_video(W, H, T, 11, cams, noise=1.0).numpy()
    m = np.zeros((T, H, W), np.uint8)
    yy, xx = np.mgrid[0:H, 0:W]
    for t in range(T):
        m[t] = (((xx - 48) / 9.0) ** 2 + ((yy - 30) / 7.0) ** 2 <= 1)
    v[m.astype(bool)] = 0
    cfg = Config(levels=2, pm_iters=3, max_outer=4, align=True)
    out, stats, ip = inpaint(torch.from_numpy(v), torch.from_numpy(m), cfg, device="cuda")
    ar, am, fwd, inv, pairs, st = orc.align_pipeline(v, m)
    assert np.array_equal(ip.align_info["theta"].cpu().numpy(), pairs)
    assert (am == 2).any()
    o_out, o_st = orc.inpaint(ar, am, 2, pm_iters=3, max_outer=4)
    ref = orc.unwarp(o_out, v, m, fwd)
    assert np.array_equal(out.cpu().numpy(), ref)
    assert [l["outer"] for l in stats.levels] == o_st["outer_iters"]
    assert stats.total_patch_updates + stats.total_stale_skipped == sum(o_st["patch_updates"])
    assert stats.total_stale_skipped == sum(o_st["stale"])
    # outside the occlusion the result is the input, bit for bit
    assert np.array_equal(out.cpu().numpy()[m == 0], v[m == 0])
