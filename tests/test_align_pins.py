"""Pins of the NEXT #1 oracle (affine realignment, Alg. 2; S3.4 P:744-758; R36-R40) against
things other than itself: homogeneous 3x3 matrix algebra (numpy), synthetic videos with a KNOWN
camera motion (gen.synth.camera_video renders a continuous world texture through per-frame affine
cameras, so the true theta_{n,n+1} = C_{n+1}^{-1} C_n is exact, not resampled), scipy's bilinear
map_coordinates, scipy morphology for the sets with the invalid set X, and the SPEC's worked
examples."""
import numpy as np
import pytest
import scipy.ndimage as ndi

from gen.synth import camera_video, random_volume

ID = np.array([0.0, 1.0, 0.0, 0.0, 0.0, 1.0])


def H3(t):
    return np.array([[t[1], t[2], t[0]], [t[4], t[5], t[3]], [0.0, 0.0, 1.0]])


def from_H3(M):
    return np.array([M[0, 2], M[0, 0], M[0, 1], M[1, 2], M[1, 0], M[1, 1]])


def true_theta(c0, c1):
    return from_H3(np.linalg.inv(H3(c1)) @ H3(c0))


def corner_err(th, ref, W, H):
    f = lambda t, x, y: np.array([t[0] + t[1] * x + t[2] * y, t[3] + t[4] * x + t[5] * y])
    return max(np.hypot(*(f(th, x, y) - f(ref, x, y))) for x in (0, W - 1) for y in (0, H - 1))


def rand_theta(rng):
    a = rng.uniform(-0.2, 0.2, 4) + np.array([1.0, 0.0, 0.0, 1.0])
    return np.array([rng.uniform(-20, 20), a[0], a[1], rng.uniform(-20, 20), a[2], a[3]])


# ---- compose / invert -----------------------------------------------------------
def test_compose_invert_algebra(orc):
    rng = np.random.default_rng(0)
    assert np.array_equal(orc.affine_compose(ID, [1, 2, 3, 4, 5, 6]), [1, 2, 3, 4, 5, 6])
    assert np.array_equal(orc.affine_compose([1, 1, 0, 2, 0, 1], [3, 1, 0, 4, 0, 1]), [4, 1, 0, 6, 0, 1])
    for _ in range(20):
        a, b = rand_theta(rng), rand_theta(rng)
        assert np.allclose(orc.affine_compose(a, b), from_H3(H3(a) @ H3(b)), rtol=0, atol=1e-12)
        assert np.allclose(orc.affine_compose(orc.affine_invert(a), a), ID, atol=1e-12)
        assert np.allclose(orc.affine_invert(a), from_H3(np.linalg.inv(H3(a))), atol=1e-12)
    with pytest.raises(ValueError):
        orc.affine_invert([0, 1, 2, 0, 2, 4])


def test_chain_matches_matrix_products(orc):
    rng = np.random.default_rng(1)
    for T in (1, 2, 5, 8):
        pairs = np.array([rand_theta(rng) for _ in range(max(T - 1, 1))])
        fwd, inv = orc.affine_chain(pairs, T)
        m = max(T // 2 - 1, 0)
        assert np.array_equal(fwd[m], ID)
        for n in range(T):
            M = np.eye(3)
            if n < m:  # theta_{m-1,m} o ... o theta_{n,n+1}
                for k in range(n, m):
                    M = H3(pairs[k]) @ M
            elif n > m:  # theta^-1_{m,m+1} o ... o theta^-1_{n-1,n}
                for k in range(m, n):
                    M = M @ np.linalg.inv(H3(pairs[k]))
            assert np.allclose(fwd[n], from_H3(M), atol=1e-9), (T, n)
            assert np.allclose(orc.affine_compose(inv[n], fwd[n]), ID, atol=1e-9)


# ---- estimation (R36-R38; SPEC S:432-441 examples) -------------------------------------------------
def test_estimate_identity_exact(orc):
    v = camera_video(96, 72, 1, 3, [ID]).numpy()
    th, st, it = orc.affine_estimate(v[0], v[0])
    assert st == 0 and np.array_equal(th, ID)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_estimate_translation_with_noise(orc, seed):
    cams = [ID, np.array([3.0, 1, 0, -2.0, 0, 1])]
    v = camera_video(128, 96, 2, seed, cams, noise=2.0).numpy()
    th, st, _ = orc.affine_estimate(v[0], v[1])
    ref = true_theta(*cams)
    assert st == 0
    assert abs(th[0] - ref[0]) < 0.1 and abs(th[3] - ref[3]) < 0.1
    assert corner_err(th, ref, 128, 96) < 0.15


def test_estimate_exact_without_noise(orc):
    cams = [ID, np.array([3.0, 1, 0, -2.0, 0, 1])]
    v = camera_video(128, 96, 2, 1, cams).numpy()
    th, st, _ = orc.affine_estimate(v[0], v[1])
    assert st == 0 and corner_err(th, true_theta(*cams), 128, 96) < 0.02


def test_estimate_general_affine(orc):
    a, sc = 0.02, 1.01
    cams = [ID, np.array([2.5, np.cos(a) * sc, -np.sin(a) * sc, -1.2, np.sin(a) * sc, np.cos(a) * sc])]
    v = camera_video(128, 96, 2, 5, cams).numpy()
    th, st, _ = orc.affine_estimate(v[0], v[1])
    assert st == 0 and corner_err(th, true_theta(*cams), 128, 96) < 0.1


def test_estimate_robust_to_moving_block(orc):
    """~30% of the pixels show an independently moving object."""
    cams = [ID, np.array([3.0, 1, 0, -2.0, 0, 1])]
    v = camera_video(128, 96, 2, 5, cams, block=(20, 20, 70, 53, -4, 3)).numpy()
    assert 0.28 <= 70 * 53 / (128 * 96) <= 0.32
    th, st, _ = orc.affine_estimate(v[0], v[1])
    ref = true_theta(*cams)
    assert st == 0 and abs(th[0] - ref[0]) < 0.25 and abs(th[3] - ref[3]) < 0.25


def test_estimate_ignores_occluded_pixels(orc):
    cams = [ID, np.array([1.5, 1, 0, 0.5, 0, 1])]
    v = camera_video(128, 96, 2, 7, cams).numpy()
    occ = np.zeros((2, 96, 128), np.uint8)
    occ[:, 30:60, 40:90] = 1
    junk = v.copy()
    junk[occ.astype(bool)] = 255 - junk[occ.astype(bool)]
    th0, _, _ = orc.affine_estimate(v[0], v[1], occ[0], occ[1])
    th1, st, _ = orc.affine_estimate(junk[0], junk[1], occ[0], occ[1])
    assert st == 0 and np.array_equal(th0, th1)  # masked pixels never vote
    assert corner_err(th1, true_theta(*cams), 128, 96) < 0.05


def test_estimate_degenerate_flat_frames(orc):
    v = np.full((64, 64, 3), 90, np.uint8)
    th, st, _ = orc.affine_estimate(v, v.copy() + 1)
    assert st == 1 and np.array_equal(th, ID)


# ---- warp / unwarp (R40) ------------------------------------------------------------
def test_warp_identity_is_exact(orc):
    v, m, _ = random_volume(40, 30, 4, seed=2, hole_frac=0.1)
    v, m = v.numpy(), m.numpy()
    inv = np.tile(ID, (4, 1))
    ar, am = orc.align_warp(v, m, inv)
    assert np.array_equal(ar, v) and np.array_equal(am, m)


def test_warp_integer_translation_and_invalid(orc):
    v, m, _ = random_volume(40, 30, 3, seed=3, hole_frac=0.1)
    v, m = v.numpy(), m.numpy()
    inv = np.tile(ID, (3, 1))
    inv[1, 0], inv[1, 3] = 5.0, -3.0  # aligned(x, y) = frame(x + 5, y - 3)
    ar, am = orc.align_warp(v, m, inv)
    assert np.array_equal(ar[1, 3:, :35], v[1, :27, 5:])
    assert np.array_equal(am[1, 3:, :35], m[1, :27, 5:])
    assert (am[1, :3, :] == 2).all() and (am[1, :, 35:] == 2).all()


def test_warp_matches_scipy_bilinear_and_mask_is_conservative(orc):
    v, m, _ = random_volume(48, 36, 2, seed=4, hole_frac=0.08)
    v, m = v.numpy(), m.numpy()
    th = np.array([1.3, 0.995, 0.02, -0.7, -0.015, 1.004])
    inv = np.stack([ID, th])
    ar, am = orc.align_warp(v, m, inv)
    yy, xx = np.mgrid[0:36, 0:48].astype(np.float64)
    xs = th[0] + th[1] * xx + th[2] * yy
    ys = th[3] + th[4] * xx + th[5] * yy
    valid = (xs >= 0) & (xs <= 47) & (ys >= 0) & (ys <= 35)
    assert np.array_equal(am[1] == 2, ~valid)
    for c in range(3):
        ref = ndi.map_coordinates(v[1, :, :, c].astype(np.float64), [ys, xs], order=1, mode="nearest")
        d = np.abs(np.floor(ref + 0.5) - ar[1, :, :, c].astype(np.float64))[valid]
        assert d.max() <= 1 and (d == 0).mean() > 0.99
    # conservativity: every valid pixel whose bilinear footprint touches H is occluded
    x0 = np.minimum(np.floor(xs), 46).astype(int)
    y0 = np.minimum(np.floor(ys), 34).astype(int)
    fx, fy = xs - x0, ys - y0
    touch = np.zeros_like(valid)
    for dx, dy, w in ((0, 0, (1 - fx) * (1 - fy)), (1, 0, fx * (1 - fy)), (0, 1, (1 - fx) * fy), (1, 1, fx * fy)):
        yi, xi = np.clip(y0 + dy, 0, 35), np.clip(x0 + dx, 0, 47)
        touch |= (w > 0) & (m[1][yi, xi] == 1)
    assert np.array_equal(am[1] == 1, touch & valid)


def test_unwarp_preserves_known_and_identity_pastes(orc):
    v, m, _ = random_volume(40, 30, 5, seed=5, hole_frac=0.1)
    v, m = v.numpy(), m.numpy()
    rng = np.random.default_rng(0)
    inp = rng.integers(0, 256, v.shape, dtype=np.uint8)
    fwd = np.array([rand_theta(rng) * [0.1, 1, 1, 0.1, 1, 1] for _ in range(5)])
    out = orc.unwarp(inp, v, m, fwd)
    known = m == 0
    assert np.array_equal(out[known], v[known])
    out2 = orc.unwarp(inp, v, m, np.tile(ID, (5, 1)))
    assert np.array_equal(out2[~known], inp[~known])


def test_unwarp_roundtrip_translation(orc):
    """pure translation: warp then unwarp of a smooth image is within 1 grey level"""
    cams = [ID] * 3
    v = camera_video(64, 48, 3, 2, cams, cell=128.0).numpy()
    m = np.ones((3, 48, 64), np.uint8)
    fwd = np.tile(ID, (3, 1))
    fwd[0, 0], fwd[0, 3] = 0.5, 0.25
    inv = np.stack([orc.affine_invert(f) for f in fwd])
    ar, _ = orc.align_warp(v, m, inv)
    back = orc.unwarp(ar, v, m, fwd)
    inner = (slice(None), slice(2, -2), slice(2, -2))
    assert np.abs(back[inner].astype(int) - v[inner].astype(int)).max() <= 2
    assert np.abs(back[inner].astype(int) - v[inner].astype(int)).mean() < 0.6


def test_align_static_video_is_identity(orc):
    """a static video is returned unchanged with identity warps."""
    v = camera_video(64, 48, 4, 3, [ID] * 4).numpy()
    m = np.zeros((4, 48, 64), np.uint8)
    m[:, 20:30, 20:30] = 1
    ar, am, fwd, inv, pairs, st = orc.align_pipeline(v, m)
    assert st == [0, 0, 0] and np.array_equal(pairs, np.tile(ID, (3, 1)))
    assert np.array_equal(ar, v) and np.array_equal(am, m)


def test_align_pan_agrees_with_reference_frame(orc):
    """a globally translating video aligns to the reference within interpolation error"""
    T = 5
    cams = [np.array([1.7 * t, 1, 0, -0.6 * t, 0, 1]) for t in range(T)]
    v = camera_video(96, 72, T, 4, cams).numpy()
    m = np.zeros((T, 72, 96), np.uint8)
    ar, am, fwd, inv, pairs, st = orc.align_pipeline(v, m)
    ref = T // 2 - 1
    for n in range(T):
        ok = am[n] == 0
        d = np.abs(ar[n].astype(int) - ar[ref].astype(int))[ok]
        assert d.mean() < 2.0, n


# ---- sets with X (R40) ------------------------------------------------------------------------------
def test_sets_x_vs_scipy(orc):
    rng = np.random.default_rng(3)
    occ = (rng.random((9, 20, 24)) < 0.01).astype(np.uint8)
    inv = np.zeros_like(occ)
    inv[:, :, :4] = 1
    src, tgt = orc.sets_x(occ, inv)
    box = np.ones((5, 5, 5), bool)
    ok = ndi.binary_erosion((occ == 0) & (inv == 0), box, border_value=0)
    assert np.array_equal(src.astype(bool), ok)
    assert np.array_equal(tgt.astype(bool), ndi.binary_dilation(occ.astype(bool), box))
    s0, t0 = orc.sets(occ)
    assert np.array_equal(orc.sets_x(occ, None)[0], s0)


def test_inpaint_with_invalid_codes_keeps_known_voxels(orc):
    v, m, _ = random_volume(40, 32, 10, seed=6, hole_frac=0.05)
    v, m = v.numpy(), m.numpy().copy()
    m[:, :, :5][m[:, :, :5] == 0] = 2
    out, _ = orc.inpaint(v, m, 2, pm_iters=2, max_outer=2)
    assert np.array_equal(out[m != 1], v[m != 1])
