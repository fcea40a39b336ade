"""Pins of the CPU oracle against things other than itself (CPU only, `-m "not gpu"`).

Each test names what fixes the expected value: a closed form, a SPEC.md/PAPER.md example,
a library routine (scipy.ndimage, numpy, cuRAND's host Philox), brute force on tiny inputs,
or an invariant of the method.  Citations: P:n = PAPER.md line, S:n = SPEC.md line.
"""
import os
import subprocess

import numpy as np
import pytest
import scipy.ndimage as ndi

from gen.synth import generate, random_volume

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _vol(T, H, W, seed=0, lo=0, hi=256):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi, size=(T, H, W, 3), dtype=np.uint8)


# ----------------------------------------------------------------------------- Philox
def test_philox_matches_curand_host(orc, tmp_path):
    """Philox4x32-10 (Salmon et al. SC'11) == cuRAND's curand_Philox4x32_10 run on the host."""
    exe = tmp_path / "kat"
    src = os.path.join(ROOT, "tests", "tools", "curand_kat.cu")
    r = subprocess.run(["nvcc", "-O1", "-Wno-deprecated-gpu-targets", "-o", str(exe), src],
                       capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip("nvcc host build failed: " + r.stderr[-300:])
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    n = 0
    for line in out.strip().splitlines():
        v = [int(x) for x in line.split()]
        ctr, k0, k1, ref = v[:4], v[4], v[5], v[6:]
        got = orc.philox(ctr, (k1 << 32) | k0)
        assert list(got) == ref, (ctr, k0, k1)
        n += 1
    assert n == 192


# ----------------------------------------------------------------------------- pyramid (a1)
def test_pyramid_constant_and_dims(orc):
    rgb = np.full((4, 17, 23, 3), 77, np.uint8)
    occ = np.zeros((4, 17, 23), np.uint8)
    rc, oc = orc.pyramid_down(rgb, occ)
    assert rc.shape == (4, 9, 12, 3)  # ceil(W/2)
    assert (rc == 77).all() and (oc == 0).all()


def test_pyramid_ramp_is_reproduced(orc):
    """A symmetric normalised kernel reproduces an affine ramp at interior samples."""
    T, H, W = 2, 12, 40
    x = np.arange(W)
    rgb = np.zeros((T, H, W, 3), np.uint8)
    rgb[..., 0] = (3 * x)[None, None, :]
    rgb[..., 1] = (100 + 2 * np.arange(H))[None, :, None]
    occ = np.zeros((T, H, W), np.uint8)
    rc, _ = orc.pyramid_down(rgb, occ)
    X = np.arange(1, rc.shape[2] - 1)
    assert np.array_equal(rc[:, :, 1:-1, 0], np.broadcast_to(6 * X, rc[:, :, 1:-1, 0].shape))
    Y = np.arange(1, rc.shape[1] - 1)
    assert np.array_equal(rc[:, 1:-1, :, 1], np.broadcast_to((100 + 4 * Y)[:, None], rc[:, 1:-1, :, 1].shape))


@pytest.mark.parametrize("with_hole", [False, True])
def test_pyramid_vs_scipy_masked_binomial(orc, with_hole):
    """Masked binomial low-pass == scipy.ndimage.correlate(u*m)/correlate(m), mirror (reflect-101)."""
    T, H, W = 3, 21, 30
    rgb = _vol(T, H, W, seed=3)
    occ = np.zeros((T, H, W), np.uint8)
    if with_hole:
        occ[:, 5:12, 8:19] = 1
        occ[1, 0:3, 0:4] = 1
    rc, oc = orc.pyramid_down(rgb, occ)
    k1 = np.array([1, 4, 6, 4, 1], np.float64)
    k = np.outer(k1, k1)
    m = 1.0 - occ.astype(np.float64)
    for c in range(3):
        for t in range(T):
            num = ndi.correlate(rgb[t, :, :, c] * m[t], k, mode="mirror")
            den = ndi.correlate(m[t], k, mode="mirror")
            num, den = num[::2, ::2], den[::2, ::2]
            ref = np.where(den > 0, np.floor(num / np.maximum(den, 1) + 0.5), 0)
            # exact integers: compare with the half-up rule on integers
            ref = np.where(den > 0, (2 * num + den) // (2 * np.maximum(den, 1)), 0)
            assert np.array_equal(rc[t, :, :, c], ref.astype(np.uint8))
    # any-of-2x2 occlusion rule (R18), via block max
    pad = np.zeros((T, 2 * oc.shape[1], 2 * oc.shape[2]), np.uint8)
    pad[:, :H, :W] = occ
    ref = pad.reshape(T, oc.shape[1], 2, oc.shape[2], 2).max(axis=(2, 4))
    assert np.array_equal(oc, ref)


def test_pyramid_ignores_hole_content(orc):
    rgb = _vol(2, 20, 20, seed=5)
    occ = np.zeros((2, 20, 20), np.uint8)
    occ[:, 6:14, 6:14] = 1
    rgb2 = rgb.copy()
    rgb2[occ.astype(bool)] = 255 - rgb2[occ.astype(bool)]
    assert np.array_equal(orc.pyramid_down(rgb, occ)[0], orc.pyramid_down(rgb2, occ)[0])


# ----------------------------------------------------------------------------- sets (a2)
def test_sets_spec_counts(orc):
    occ = np.zeros((10, 10, 10), np.uint8)
    src, tgt = orc.sets(occ)
    assert src.sum() == 6 * 6 * 6 and src[2:8, 2:8, 2:8].all()
    assert tgt.sum() == 0
    occ[5, 5, 5] = 1
    src, tgt = orc.sets(occ)
    assert tgt.sum() == 125  # 5x5x5 dilation of one voxel (S:66 with a 5^3 patch)
    occ[:] = 0
    occ[0, 0, 0] = 1
    assert orc.sets(occ)[1].sum() == 27  # corner: clipped
    occ[:] = 1
    assert orc.sets(occ)[0].sum() == 0


def test_sets_vs_scipy_morphology(orc):
    rng = np.random.default_rng(7)
    occ = (rng.random((9, 14, 17)) < 0.03).astype(np.uint8)
    src, tgt = orc.sets(occ)
    st = np.ones((5, 5, 5), bool)
    ref_tgt = ndi.binary_dilation(occ.astype(bool), structure=st)
    # D~: erosion of D with out-of-bounds treated as not-D
    ref_src = ndi.binary_erosion(~occ.astype(bool), structure=st, border_value=0)
    assert np.array_equal(tgt.astype(bool), ref_tgt)
    assert np.array_equal(src.astype(bool), ref_src)
    assert not (src.astype(bool) & tgt.astype(bool)).any()  # D~ and H~ disjoint


@pytest.mark.parametrize("name,n_h,n_t,n_s", [("c1", 1440, 3584, 38656)])
def test_sets_match_survey_appendix(orc, name, n_h, n_t, n_s):
    """|H|, |H~|, |D~| computed independently (NumPy/SciPy) in SURVEY.md Appendix A."""
    _, m, _ = generate(name)
    src, tgt = orc.sets(m.numpy())
    assert int(m.sum()) == n_h and int(tgt.sum()) == n_t and int(src.sum()) == n_s


# ----------------------------------------------------------------------------- texture (a3)
def test_texture_constant_is_zero(orc):
    rgb = np.full((2, 9, 11, 3), 130, np.uint8)
    tex = orc.texture(rgb, np.zeros((2, 9, 11), np.uint8), 2)
    assert (tex == 0).all()


def test_texture_step_spec_example(orc):
    """vertical step of 10 grey levels, nu_half = 0 -> T_x = 5 at the two adjacent columns."""
    rgb = np.zeros((1, 6, 10, 3), np.uint8)
    rgb[:, :, 5:, :] = 10  # grey step of 10 between columns 4 and 5
    tex = orc.texture(rgb, np.zeros((1, 6, 10), np.uint8), 0)
    tx = tex[0, :, :, 0]
    assert (tx[:, 4] == 10).all() and (tx[:, 5] == 10).all()  # half units: T_q = 2 T = 10
    assert tx[:, [0, 1, 2, 3, 6, 7, 8, 9]].sum() == 0
    assert (tex[..., 1] == 0).all()


def test_texture_vs_scipy(orc):
    """Eq. 8 via scipy box sums of masked |central differences| (independent formulation)."""
    T, H, W, h = 2, 13, 19, 2
    rgb = _vol(T, H, W, seed=11)
    occ = np.zeros((T, H, W), np.uint8)
    occ[:, 4:8, 5:11] = 1
    tex = orc.texture(rgb, occ, h)
    Y = rgb[..., 0].astype(np.int64) * 299 + rgb[..., 1].astype(np.int64) * 587 + rgb[..., 2].astype(np.int64) * 114
    for axis, ch in ((2, 0), (1, 1)):
        n = Y.shape[axis]
        idx = np.arange(n)
        im = np.abs(idx - 1)
        ip = np.where(idx + 1 >= n, 2 * (n - 1) - (idx + 1), idx + 1)
        dY = np.abs(np.take(Y, ip, axis=axis) - np.take(Y, im, axis=axis))
        ok = (np.take(occ, ip, axis=axis) == 0) & (np.take(occ, im, axis=axis) == 0)
        ones = np.ones((1, 2 * h + 1, 2 * h + 1))
        s = ndi.correlate((dY * ok).astype(np.float64), ones, mode="constant")
        c = ndi.correlate(ok.astype(np.float64), ones, mode="constant")
        s, c = np.rint(s).astype(np.int64), np.rint(c).astype(np.int64)
        ref = np.where(c > 0, (s + 500 * c) // (1000 * np.maximum(c, 1)), 0)
        assert np.array_equal(tex[..., ch], ref.astype(np.uint8))


def test_texture_decimation_impulse(orc):
    """impulse at (8,8,t0), L=4 -> nonzero only at (1,1,t0) at level 4."""
    tex1 = np.zeros((3, 20, 20, 2), np.uint8)
    tex1[1, 8, 8, :] = (7, 9)
    t4 = orc.texture_decimate(tex1, 4, 3, 3)
    nz = np.argwhere(t4.any(-1))
    assert nz.tolist() == [[1, 1, 1]] and tuple(t4[1, 1, 1]) == (7, 9)


# ----------------------------------------------------------------------------- layers (Alg. 3)
def test_layers_erosion_examples(orc):
    occ = np.zeros((9, 9, 9), np.uint8)
    occ[3:6, 3:6, 3:6] = 1  # 3^3 block -> 1 layer shell + centre
    lay, n = orc.layers(occ)
    assert n == 2 and (lay == 2).sum() == 1 and lay[4, 4, 4] == 2
    occ[:] = 0
    occ[2:7, 2:7, 2:7] = 1  # 5^3 -> inner 3^3 after one erosion
    lay, n = orc.layers(occ)
    assert (lay >= 2).sum() == 27 and n == 3
    occ = np.zeros((11, 30, 30), np.uint8)
    occ[:, 10:20, 10:20] = 1  # half-thickness 5 box (all frames, out-of-bounds = occluded): 5 layers
    assert orc.layers(occ)[1] == 5


def test_layers_vs_scipy_chessboard(orc):
    rng = np.random.default_rng(3)
    occ = np.zeros((8, 20, 24), np.uint8)
    occ[1:7, 3:15, 4:20] = 1
    occ |= (rng.random(occ.shape) < 0.02).astype(np.uint8)
    lay, n = orc.layers(occ)
    # L_inf distance to D with out-of-bounds treated as occluded (R22): pad with ones
    pad = np.pad(occ, 1, constant_values=1)
    # distance from each voxel to the nearest zero in the padded volume, padding can't be D
    d = ndi.distance_transform_cdt(pad, metric="chessboard")[1:-1, 1:-1, 1:-1]
    assert np.array_equal(lay.astype(np.int64), np.where(occ > 0, d, 0))
    assert n == lay.max()


# ----------------------------------------------------------------------------- distance (a4)
def _level(orc, rgb, occ, tex=None, layers=False):
    if tex is None:
        tex = np.zeros(rgb.shape[:3] + (2,), np.uint8)
    return orc.Level(rgb, tex, occ, with_layers=layers)


def test_distance_examples(orc):
    T, H, W = 9, 9, 9
    rgb = np.full((T, H, W, 3), 50, np.uint8)
    occ = np.zeros((T, H, W), np.uint8)
    occ[0, 0, 0] = 1
    lv = _level(orc, rgb, occ)
    p = (4 * H + 4) * W + 4
    assert orc.patch_ssd(lv, p, p, 50) == (0, 125)  # p = q -> 0
    lv.rgb[5, 5, 5, 1] = 60  # one voxel differs by 10 in one channel (S:187 at N = 125)
    q = (4 * H + 4) * W + 3  # q patch covers (5,5,5) at offset (+1): r = q+(2,1,1)... use p vs q
    D, n = orc.patch_ssd(lv, p, q, 0)
    # N_p contains (5,5,5) and (5,5,6)->source; count the differing terms directly
    ref = 0
    for dt in range(-2, 3):
        for dy in range(-2, 3):
            for dx in range(-2, 3):
                a = lv.rgb[4 + dt, 4 + dy, 4 + dx].astype(int)
                b = lv.rgb[4 + dt, 4 + dy, 3 + dx].astype(int)
                ref += 4 * int(((a - b) ** 2).sum())
    assert (D, n) == (ref, 125) and ref == 2 * 400


def test_distance_single_voxel_diff(orc):
    rgb = np.full((12, 12, 12, 3), 50, np.uint8)
    rgb[3, 3, 3, 0] = 60
    lv = _level(orc, rgb, np.zeros((12, 12, 12), np.uint8))
    p = (3 * 12 + 3) * 12 + 3
    q = (8 * 12 + 8) * 12 + 8
    D, n = orc.patch_ssd(lv, p, q, 0)
    assert D == 400 and n == 125  # d^2 = D/(4n) = 100/125 (S:187 with N = 125)


def test_partial_distance_one_known_voxel(orc):
    """exactly one known voxel with colour diff 6 in one channel -> d^2 = 36."""
    T, H, W = 12, 12, 24
    rgb = np.full((T, H, W, 3), 100, np.uint8)
    occ = np.zeros((T, H, W), np.uint8)
    occ[3:8, 3:8, 3:8] = 1
    occ[3, 3, 3] = 0  # the single known voxel of N_p for p = (5,5,5)
    lv = _level(orc, rgb, occ, layers=True)
    lv.rgb[3, 3, 3, 2] = 106
    p = (5 * H + 5) * W + 5
    q = int(lv.sources[0])
    D, n = orc.patch_ssd(lv, p, q, 50, kb=1)  # K = D
    assert n == 1 and D / (4 * n) == 36.0


def test_distance_vs_numpy_eq9(orc):
    """Eq. 9 (and Eq. 2 at lambda = 0) via numpy slicing; symmetry; lambda-monotone."""
    T, H, W = 8, 11, 13
    rgb = _vol(T, H, W, seed=21)
    tex = np.random.default_rng(2).integers(0, 60, (T, H, W, 2), dtype=np.uint8)
    lv = _level(orc, rgb, np.zeros((T, H, W), np.uint8), tex)
    rng = np.random.default_rng(5)
    for _ in range(40):
        p = (int(rng.integers(2, T - 2)), int(rng.integers(2, H - 2)), int(rng.integers(2, W - 2)))
        q = (int(rng.integers(2, T - 2)), int(rng.integers(2, H - 2)), int(rng.integers(2, W - 2)))
        lp = (p[0] * H + p[1]) * W + p[2]
        lq = (q[0] * H + q[1]) * W + q[2]
        sl = lambda c: (slice(c[0] - 2, c[0] + 3), slice(c[1] - 2, c[1] + 3), slice(c[2] - 2, c[2] + 3))
        dc = ((rgb[sl(p)].astype(np.int64) - rgb[sl(q)]) ** 2).sum()
        dtx = ((tex[sl(p)].astype(np.int64) - tex[sl(q)]) ** 2).sum()
        for lam in (0, 1, 50):
            D, n = orc.patch_ssd(lv, lp, lq, lam)
            assert n == 125 and D == 4 * dc + lam * dtx
            assert D / (4 * n) == pytest.approx((dc + lam * dtx / 4) / 125, rel=0, abs=1e-9)
        assert orc.patch_ssd(lv, lq, lp, 50) == orc.patch_ssd(lv, lp, lq, 50)


def test_distance_border_clip(orc):
    """R23: a target at the volume corner is clipped to Omega: n = 27."""
    rgb = _vol(8, 8, 8, seed=1)
    lv = _level(orc, rgb, np.zeros((8, 8, 8), np.uint8))
    q = (4 * 8 + 4) * 8 + 4
    D, n = orc.patch_ssd(lv, 0, q, 50)
    ref = 0
    for t in range(3):
        for y in range(3):
            for x in range(3):
                ref += 4 * int(((rgb[t, y, x].astype(int) - rgb[4 + t, 4 + y, 4 + x]) ** 2).sum())
    assert (D, n) == (ref, 27)


# ----------------------------------------------------------------------------- NNF (a5-a8)
def _c1_level(orc, lam_tex=True):
    v, m, _ = generate("c1")
    rgb, occ = v.numpy(), m.numpy()
    tex = orc.texture(rgb, occ, 1) if lam_tex else None
    return _level(orc, rgb, occ, tex)


def _check_nnf(orc, lv, nnf, lam, kb=-1):
    for s, p in enumerate(lv.targets):
        t, y, x = p // (lv.H * lv.W), (p // lv.W) % lv.H, p % lv.W
        qx, qy, qt = x + nnf.dx[s], y + nnf.dy[s], t + nnf.dt[s]
        assert 0 <= qx < lv.W and 0 <= qy < lv.H and 0 <= qt < lv.T
        q = (qt * lv.H + qy) * lv.W + qx
        assert lv.src.ravel()[q] == 1
        assert orc.patch_ssd(lv, p, q, lam, kb) == (int(nnf.D[s]), int(nnf.n[s]))


def test_random_init_forced_and_deterministic(orc):
    T = H = W = 9
    occ = np.ones((T, H, W), np.uint8)
    occ[2:7, 2:7, 2:7] = 0  # D~ = the single centre voxel
    lv = _level(orc, _vol(T, H, W), occ)
    assert len(lv.sources) == 1
    nnf = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, nnf, 9, 1, 0)
    for s, p in enumerate(lv.targets):
        t, y, x = p // 81, (p // 9) % 9, p % 9
        assert (x + nnf.dx[s], y + nnf.dy[s], t + nnf.dt[s]) == (4, 4, 4)


def test_random_init_uniform(orc):
    lv = _c1_level(orc)
    a, b = orc.NNF.empty(len(lv.targets)), orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 123, 1, 0)
    orc.init_random(lv, b, 123, 1, 0)
    assert np.array_equal(a.dx, b.dx) and np.array_equal(a.dt, b.dt)
    # chi-square over 16 buckets of the D~ list index
    idx = []
    pos = {int(q): i for i, q in enumerate(lv.sources)}
    for s, p in enumerate(lv.targets):
        t, y, x = p // (lv.H * lv.W), (p // lv.W) % lv.H, p % lv.W
        q = ((t + a.dt[s]) * lv.H + y + a.dy[s]) * lv.W + x + a.dx[s]
        idx.append(pos[int(q)])
    hist = np.bincount(np.array(idx) * 16 // len(lv.sources), minlength=16)
    exp = len(idx) / 16
    chi2 = ((hist - exp) ** 2 / exp).sum()
    assert chi2 < 45  # 15 dof; p ~ 1e-4


def test_patchmatch_invariants_and_monotone(orc):
    lv = _c1_level(orc)
    lam = 50
    a = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 5, 1, 0)
    orc.evaluate(lv, a, lam)
    _check_nnf(orc, lv, a, lam)
    b = a.copy()
    for k in (1, 2):
        sign = 1 if k % 2 else -1
        for st in (8, 4, 2, 1):
            orc.propagate(lv, a, b, lam, st, sign)
            assert (b.D <= a.D).all()
            _check_nnf(orc, lv, b, lam)
            a, b = b, a
        orc.random_search(lv, a, b, lam, 5, 0.5, lv.rmax, 1, 0, k)
        assert (b.D <= a.D).all()
        _check_nnf(orc, lv, b, lam)
        a, b = b, a


def test_random_search_radius_property(orc):
    """Eq. 3 with rmax = 2, rho = 0.5: one radius R_1 = 1, offsets floor(delta) in {-1, 0}."""
    lv = _c1_level(orc)
    a = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 3, 1, 0)
    orc.evaluate(lv, a, 50)
    b = a.copy()
    cnt = orc.random_search(lv, a, b, 50, 3, 0.5, 2, 1, 0, 1)
    assert cnt > 0
    for arr in ("dx", "dy", "dt"):
        d = getattr(b, arr) - getattr(a, arr)
        assert set(np.unique(d)) <= {-1, 0}
    # rmax = 1: R_1 = 0.5 < 1, no candidate at all
    assert orc.random_search(lv, a, b, 50, 3, 0.5, 1, 1, 0, 1) == 0


def test_exact_copy_reaches_zero(orc):
    """an exact unoccluded copy of every target patch exists -> PatchMatch finds D = 0."""
    T, H, W = 6, 16, 40
    base = _vol(T, H, 20, seed=8)
    rgb = np.concatenate([base, base], axis=2)  # right half is a copy of the left half
    occ = np.zeros((T, H, W), np.uint8)
    occ[2:4, 6:9, 8:11] = 1
    lv = _level(orc, rgb, occ)
    a = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 1, 1, 0)
    # make the hole content equal to the copy so that exact matches exist
    lv.rgb[2:4, 6:9, 8:11] = rgb[2:4, 6:9, 28:31]
    a, cnt = orc.ann_search(lv, a, 0, 1, 1, 0, 10)
    interior = [s for s, p in enumerate(lv.targets)
                if 2 <= p // (H * W) < T - 2 and 2 <= (p // W) % H < H - 2]
    assert np.mean(a.D[interior] == 0) > 0.9


def test_brute_force_definition_and_ties(orc):
    T, H, W = 5, 7, 14
    rgb = _vol(T, H, W, seed=4)
    occ = np.zeros((T, H, W), np.uint8)
    occ[2, 3, 2] = 1
    lv = _level(orc, rgb, occ)
    nnf = orc.NNF.empty(len(lv.targets))
    orc.brute_force(lv, nnf, 0)
    for s, p in enumerate(lv.targets):
        Ds = [orc.patch_ssd(lv, p, q, 0)[0] for q in lv.sources]
        j = int(np.argmin(Ds))  # numpy argmin returns the first minimum = smallest q
        q = int(lv.sources[j])
        t, y, x = p // (H * W), (p // W) % H, p % W
        assert ((t + nnf.dt[s]) * H + y + nnf.dy[s]) * W + x + nnf.dx[s] == q
        assert nnf.D[s] == Ds[j]
    # two equidistant sources: constant volume -> every source ties -> the first source
    lv2 = _level(orc, np.full((T, H, W, 3), 9, np.uint8), occ)
    nnf2 = orc.NNF.empty(len(lv2.targets))
    orc.brute_force(lv2, nnf2, 50)
    s0 = int(lv2.sources[0])
    for s, p in enumerate(lv2.targets):
        t, y, x = p // (H * W), (p // W) % H, p % W
        assert ((t + nnf2.dt[s]) * H + y + nnf2.dy[s]) * W + x + nnf2.dx[s] == s0


def test_brute_force_dominates_patchmatch_and_quality(orc):
    """D(PatchMatch) >= D(brute force) per target; mean d^2 ratio reported (north_star 5%)."""
    v, m, _ = random_volume(24, 20, 8, seed=3, hole_frac=0.04)
    rgb, occ = v.numpy(), m.numpy()
    lv = _level(orc, rgb, occ, orc.texture(rgb, occ, 1))
    bf = orc.NNF.empty(len(lv.targets))
    orc.brute_force(lv, bf, 50)
    a = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 2, 1, 0)
    a, _ = orc.ann_search(lv, a, 50, 2, 1, 0, 10)
    assert (a.D >= bf.D).all()
    d_pm = (a.D / (4.0 * a.n)).mean()
    d_bf = (bf.D / (4.0 * bf.n)).mean()
    assert d_pm <= 1.5 * d_bf  # S:266 quality invariant


# ----------------------------------------------------------------------------- reconstruction
def _recon_fixture(orc, colour_fn, D_fn=None):
    """Level with a 1-voxel hole; every contributor's shift points at a chosen source."""
    T = H = W = 11
    rgb = np.zeros((T, H, W, 3), np.uint8)
    occ = np.zeros((T, H, W), np.uint8)
    occ[5, 5, 5] = 1
    lv = _level(orc, rgb, occ)
    nnf = orc.NNF.empty(len(lv.targets))
    return lv, nnf


def test_reconstruct_examples(orc):
    T = H = W = 13
    rng = np.random.default_rng(0)
    rgb = rng.integers(0, 256, (T, H, W, 3), dtype=np.uint8)
    occ = np.zeros((T, H, W), np.uint8)
    occ[6, 6, 6] = 1
    lv = _level(orc, rgb, occ)
    nt = len(lv.targets)
    assert nt == 125
    # all contributors map to sources of identical colour c -> c in every mode
    lv.rgb[:] = 0
    lv.rgb[6, 6, 6] = 0
    lv.rgb[..., :] = (10, 20, 30)
    lv.rgb[6, 6, 6] = 0
    nnf = orc.NNF.empty(nt)
    nnf.dx[:] = 3 if True else 0  # p + phi(q) lands at x + 3: stays inside the constant region
    nnf.dx[:] = 0
    nnf.dt[:] = 0
    nnf.dy[:] = 0
    for s, p in enumerate(lv.targets):
        nnf.dx[s] = -4  # q + phi(q) = q - 4 in x; valid sources exist for these
        nnf.D[s] = 100 + s
        nnf.n[s] = 125
    for mode in (orc.WEIGHTED, orc.UNWEIGHTED, orc.BEST_PATCH):
        out, tex = orc.reconstruct(lv, nnf, mode)
        assert np.array_equal(out[0], [10, 20, 30])


def _one_hole(orc, seed=0):
    T = H = W = 13
    rng = np.random.default_rng(seed)
    rgb = rng.integers(0, 256, (T, H, W, 3), dtype=np.uint8)
    occ = np.zeros((T, H, W), np.uint8)
    occ[6, 6, 6] = 1
    lv = _level(orc, rgb, occ)
    nnf = orc.NNF.empty(len(lv.targets))
    return lv, nnf


def test_reconstruct_unweighted_two_values(orc):
    """unweighted mean of {100, 200} -> 150 (here 62 contributors each)."""
    lv, nnf = _one_hole(orc)
    # contributors q (in N_p order) alternate between two shifts pointing at 100 and 200
    lv.rgb[6, 6, 1] = (100, 100, 100)  # p + (0,0,-5)
    lv.rgb[6, 6, 11] = (200, 200, 200)  # p + (0,0,+5)
    for s in range(125):
        nnf.dx[s] = -5 if s % 2 == 0 else 5
        nnf.D[s] = 7
        nnf.n[s] = 125
    out, _ = orc.reconstruct(lv, nnf, orc.UNWEIGHTED)
    assert out[0, 0] == pytest.approx((63 * 100 + 62 * 200) / 125, abs=1e-4)
    for s in range(125):
        nnf.dx[s] = -5 if s < 62 else 5
    nnf.dx[124] = -5
    nnf.dx[0] = 5  # 62 vs 63 -> shuffle to 62/63 balance
    nnf.dx[:] = np.where(np.arange(125) < 62, -5, 5)
    out, _ = orc.reconstruct(lv, nnf, orc.UNWEIGHTED)
    assert out[0, 0] == pytest.approx((62 * 100 + 63 * 200) / 125, abs=1e-4)


def test_reconstruct_weighted_vs_numpy(orc):
    """Eqs. 4-5 evaluated with numpy (percentile method 'inverted_cdf' = nearest rank, np.exp,
    fp64 sums in another order) agree to 1e-6 on random instances."""
    rng = np.random.default_rng(4)
    for trial in range(10):
        lv, nnf = _one_hole(orc, seed=trial)
        dxs = rng.integers(-5, 6, 125)
        nnf.dx[:] = np.where(np.abs(dxs) < 4, 5, dxs)  # keep p + phi(q) off the hole
        nnf.dy[:] = rng.integers(-4, 5, 125)
        nnf.D[:] = rng.integers(0, 400000, 125)
        nnf.D[rng.integers(0, 125, 3)] = 0
        nnf.n[:] = 125
        out, _ = orc.reconstruct(lv, nnf, orc.WEIGHTED)
        d2 = nnf.D / (4.0 * nnf.n)
        sig2 = np.percentile(d2, 75, method="inverted_cdf")
        w = np.exp(-d2 / (2 * sig2))
        vals = np.array([lv.rgb[6, 6 + nnf.dy[s], 6 + nnf.dx[s]] for s in range(125)], np.float64)
        ref = (w[:, None] * vals).sum(0) / w.sum()
        assert np.allclose(out[0], ref, atol=2e-5, rtol=0)  # fp32 output + 2^-36 weights
        assert (out[0] >= vals.min(0) - 1e-6).all() and (out[0] <= vals.max(0) + 1e-6).all()


def test_reconstruct_sigma_zero_and_best_patch(orc):
    lv, nnf = _one_hole(orc, seed=3)
    nnf.dx[:] = 5
    nnf.dy[:] = np.arange(125) % 5 - 2
    nnf.D[:] = 0  # sigma = 0 -> mean over zero-distance contributors
    nnf.D[100:] = 50
    nnf.n[:] = 125
    out, _ = orc.reconstruct(lv, nnf, orc.WEIGHTED)
    vals = np.array([lv.rgb[6, 6 + nnf.dy[s], 11] for s in range(125)], np.float64)
    assert np.allclose(out[0], vals[:100].mean(0), atol=1e-4)
    # best patch: unique minimum -> exact copy; ties -> smallest q
    nnf.D[:] = 9
    nnf.D[37] = 1
    out, _ = orc.reconstruct(lv, nnf, orc.BEST_PATCH)
    assert np.array_equal(out[0], vals[37])
    nnf.D[:] = 4
    out, _ = orc.reconstruct(lv, nnf, orc.BEST_PATCH)
    assert np.array_equal(out[0], vals[0])


def test_change_l1_constructed(orc):
    a = np.array([1.0, 2.5, 100.0, 0.25], np.float32)
    b = np.array([0.5, 3.0, 100.0, 1.0], np.float32)
    assert orc.change_l1(a, b) == int((0.5 + 0.5 + 0 + 0.75) * 2 ** 20)


def test_energy_is_sum_of_distances(orc):
    lv = _c1_level(orc)
    a = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 1, 1, 0)
    orc.evaluate(lv, a, 50)
    E = orc.energy(lv, a)
    ref = 0.0
    for p in lv.holes:
        s = lv.slot[p]
        ref += a.D[s] / (4.0 * a.n[s])
    assert E == pytest.approx(ref, rel=1e-12)


# ----------------------------------------------------------------------------- pipeline
def test_pipeline_preserves_outside_and_ignores_hole_content(orc):
    v, m, _ = generate("c1")
    rgb, occ = v.numpy(), m.numpy()
    out1, st = orc.inpaint(rgb, occ, 1, pm_iters=4, fixed_outer=3)
    mm = occ.astype(bool)
    assert np.array_equal(out1[~mm], rgb[~mm])
    rgb2 = rgb.copy()
    rgb2[mm] = 200
    out2, _ = orc.inpaint(rgb2, occ, 1, pm_iters=4, fixed_outer=3)
    assert np.array_equal(out1, out2)
    out3, _ = orc.inpaint(rgb, occ, 1, pm_iters=4, fixed_outer=3)
    assert np.array_equal(out1, out3)  # determinism
    assert st["outer_iters"] == [3] and st["onion_layers"] == 5


def test_pipeline_periodic_texture_psnr(orc):
    """SPEC acceptance 4 analogue: translating periodic texture, 12x12 box -> PSNR in H > 28 dB."""
    T, H, W = 16, 64, 64
    t, y, x = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    rgb = np.stack([128 + 60 * np.sin(2 * np.pi * (x - t) / 8) + 40 * np.cos(2 * np.pi * y / 6),
                    128 + 50 * np.cos(2 * np.pi * (x + y - t) / 10),
                    100 + 30 * np.sin(2 * np.pi * y / 7)], -1)
    rgb = np.clip(np.floor(rgb + 0.5), 0, 255).astype(np.uint8)
    occ = np.zeros((T, H, W), np.uint8)
    occ[:, 26:38, 26:38] = 1
    v = rgb.copy()
    v[occ.astype(bool)] = 0
    out, st = orc.inpaint(v, occ, 2, pm_iters=10)
    d = out.astype(float) - rgb
    psnr = 10 * np.log10(255 ** 2 / np.mean(d[occ.astype(bool)] ** 2))
    assert psnr > 28


# ----------------------------------------------------------------------------- directed pins
def _copy_world(orc):
    """Exact-copy volume: the right half repeats the left half, so shift (+20, 0, 0) is perfect."""
    T, H, W = 9, 12, 40
    base = _vol(T, H, 20, seed=31)
    rgb = np.concatenate([base, base], axis=2)
    occ = np.zeros((T, H, W), np.uint8)
    occ[4, 6, 6] = 1  # one hole voxel -> a 5x5x5 block of targets around (6, 6, 4)
    lv = _level(orc, rgb, occ)
    lv.rgb[4, 6, 6] = rgb[4, 6, 26]  # hole content equals its copy
    return lv


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("sign", [1, -1])
def test_propagation_direction_and_axis(orc, axis, sign):
    """P:377-386 / Alg. 1: the candidate of target p is phi(p + sign*step*e_axis).  Only the
    neighbour on that side holds the perfect shift, so exactly the matching (axis, sign) pass
    improves p to D = 0."""
    lv = _copy_world(orc)
    nt = len(lv.targets)
    f = orc.NNF.empty(nt)
    bad = (1, 1, 0)  # a poor but valid shift for everyone
    f.dx[:] = bad[0]
    f.dy[:] = bad[1]
    f.dt[:] = bad[2]
    orc.evaluate(lv, f, 50)
    H, W = lv.H, lv.W
    p = (4 * H + 6) * W + 6  # centre target
    off = [0, 0, 0]
    off[axis] = sign * 2
    r = ((4 + off[2]) * H + 6 + off[1]) * W + 6 + off[0]
    sp, sr = lv.slot[p], lv.slot[r]
    assert sp >= 0 and sr >= 0
    f.dx[sr], f.dy[sr], f.dt[sr] = 20, 0, 0  # the perfect shift, on one side only
    orc.evaluate(lv, f, 50)
    assert f.D[sp] > 0
    for ax2 in range(3):
        for sg2 in (1, -1):
            g = f.copy()
            orc.propagate(lv, f, g, 50, 2, sg2)
            got = g.D[sp] == 0 and (g.dx[sp], g.dy[sp], g.dt[sp]) == (20, 0, 0)
            assert got == (sg2 == sign), (ax2, sg2)
    g = f.copy()
    orc.propagate(lv, f, g, 50, 2, 0)  # both directions always see it
    assert g.D[sp] == 0


def test_upsample_spec_example(orc):
    """coarse shift (2, -1, 3) at (x, y, t) -> fine (4, -2, 3) at (2x, 2y, t); a zero
    map stays zero where valid; invalid results are re-drawn inside D~ (R21)."""
    T, H, W = 12, 24, 40
    rgb = _vol(T, H, W, seed=2)
    occ = np.zeros((T, H, W), np.uint8)
    occ[5:7, 10:14, 16:20] = 1
    fine = _level(orc, rgb, occ)
    rc, oc = orc.pyramid_down(rgb, occ)
    coarse = _level(orc, rc, oc)
    cn = orc.NNF.empty(len(coarse.targets))
    cn.dx[:] = 2
    cn.dy[:] = -1
    cn.dt[:] = 3
    fn = orc.NNF.empty(len(fine.targets))
    orc.upsample(coarse, cn, fine, fn, 7, 1)
    Wc = coarse.W
    n_ok = 0
    for s, p in enumerate(fine.targets):
        t, y, x = p // (H * W), (p // W) % H, p % W
        q = (t + fn.dt[s], y + fn.dy[s], x + fn.dx[s])
        assert fine.src[q] == 1  # always valid after repair
        cs = coarse.slot[(t * coarse.H + y // 2) * Wc + x // 2]
        want_ok = cs >= 0 and 0 <= t + 3 < T and 0 <= y - 2 < H and 0 <= x + 4 < W and \
            fine.src[t + 3, y - 2, x + 4] == 1
        if want_ok:
            assert (fn.dx[s], fn.dy[s], fn.dt[s]) == (4, -2, 3)
            n_ok += 1
    assert n_ok > 100
    cn.dx[:] = 0
    cn.dy[:] = 0
    cn.dt[:] = 0  # zero map: invalid everywhere (targets are not sources), so all re-drawn
    orc.upsample(coarse, cn, fine, fn, 7, 1)
    assert all(fine.src[(p // (H * W) + fn.dt[s], (p // W) % H + fn.dy[s], p % W + fn.dx[s])]
               for s, p in enumerate(fine.targets))


# ----------------------------------------------------------------------------- App. B (NEXT #3)
def test_ambiguity_exact_closed_forms(orc):
    """N = 1: P(Y^2 < 2XY) for independent standard normals = atan(2)/pi (planar angle); N = 2:
    (1 - 1/sqrt 5)/2 (Rayleigh, by parts); N >= 9 vs scipy's quadrature of E[Q(sqrt(chi2_N)/2)]."""
    import math
    from scipy import integrate, stats
    assert orc.ambiguity_exact(1) == pytest.approx(math.atan(2) / math.pi, rel=1e-9)
    assert orc.ambiguity_exact(2) == pytest.approx((1 - 1 / math.sqrt(5)) / 2, rel=1e-9)  # by parts
    for N in (9, 25, 27, 125):
        f = lambda r: stats.norm.sf(np.sqrt(r) / 2) * stats.chi2.pdf(r, N)
        ref, _ = integrate.quad(f, 0, np.inf, limit=500, epsabs=0, epsrel=1e-12)
        assert orc.ambiguity_exact(N) == pytest.approx(ref, rel=1e-7)


def test_ambiguity_paper_table2(orc):
    """Table 2: 3x3 -> 8e-2, 5x5 -> 1e-2 (the paper's simulation; our exact values agree
    within 5%).  The rarer entries are reported, not pinned."""
    assert orc.ambiguity_exact(9) == pytest.approx(8e-2, rel=0.06)
    assert orc.ambiguity_exact(25) == pytest.approx(1e-2, rel=0.05)
    vals = [orc.ambiguity_exact(N) for N in (9, 25, 27, 49, 81, 121, 125)]
    assert all(a > b for a, b in zip(vals, vals[1:]))  # strictly decreasing (SPEC acceptance 1)


def test_ambiguity_simulation_matches_exact(orc):
    for N in (9, 25):
        n = 1_000_000
        p = orc.ambiguity_exact(N)
        h = orc.ambiguity_mc(N, n, sigma=5.0, seed=3)
        assert abs(h / n - p) < 5 * (p * (1 - p) / n) ** 0.5


# ----------------------------------------------------------------------------- NEXT #2 sequential scan
def test_sequential_scan_invariants_and_reuse(orc):
    lv = _c1_level(orc)
    a = orc.NNF.empty(len(lv.targets))
    orc.init_random(lv, a, 5, 1, 0)
    b = a.copy()
    orc.evaluate(lv, b, 50)
    d0 = b.D.copy()
    cnt = orc.ann_search_sequential(lv, b, 50, 5, 1, 0, 4)
    assert cnt > 0 and (b.D <= d0).all()
    _check_nnf(orc, lv, b, 50)
    bf = orc.NNF.empty(len(lv.targets))
    orc.brute_force(lv, bf, 50)
    assert (b.D >= bf.D).all()
    assert (b.D / (4.0 * b.n)).mean() <= 1.5 * (bf.D / (4.0 * bf.n)).mean()


def test_sequential_scan_propagates_along_a_row_in_one_pass(orc):
    """in-place scans reuse entries already updated, so one forward scan carries a good
    shift along a whole row of targets; a single Jacobi pass moves it by one step only."""
    lv = _copy_world(orc)
    nt = len(lv.targets)
    f = orc.NNF.empty(nt)
    f.dx[:], f.dy[:], f.dt[:] = 1, 1, 0
    H, W = lv.H, lv.W
    row = [s for s, p in enumerate(lv.targets) if p // (H * W) == 4 and (p // W) % H == 6]
    xs = [lv.targets[s] % W for s in row]
    first = row[int(np.argmin(xs))]
    f.dx[first], f.dy[first], f.dt[first] = 20, 0, 0  # perfect shift at the row's left end
    g = f.copy()
    # K = 0 evaluates only; K = 2 runs one reverse (+1) and one forward (-1) scan before RS
    orc.ann_search_sequential(lv, g, 0, 3, 1, 0, 2, rmax=1)
    assert all(g.D[s] == 0 for s in row)
    j = f.copy()
    orc.evaluate(lv, j, 0)
    k2 = j.copy()
    orc.propagate(lv, j, k2, 0, 1, -1)
    assert sum(k2.D[s] == 0 for s in row) == 2  # the first target and its right neighbour only
