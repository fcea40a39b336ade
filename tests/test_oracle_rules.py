"""Pins of the oracle's selection, onion and stopping rules (CPU only, `-m "not gpu"`).

Each case is constructed so that its expected value is fixed by the rule itself, not by the
oracle's arithmetic, and so that the plausible one-character mistake in the rule changes the
answer.  `tools/mutation_check.py` re-applies those mistakes to a copy of oracle.c and checks
that these pins turn red (mutation table).

* Eq. 13: the contributors of an onion-layer-j voxel are N'_p = {q : layer(q) < j};
  Alg. 3 writes each hole voxel exactly once, at its own layer.
* R25 ("smaller", "<"): a candidate replaces the incumbent only if its distance is
  strictly smaller; among equal new candidates the lowest rank wins.
* R19 / P:930-939: stop after outer iteration k iff e <= 0.1 or k = 20.
* R20: right after upsampling (n = 0, no distances yet) the reconstruction is the
  unweighted mean over all contributors.
"""
import numpy as np
import pytest

from gen.synth import generate


def _level(orc, rgb, occ, tex=None, layers=False):
    if tex is None:
        tex = np.zeros(rgb.shape[:3] + (2,), np.uint8)
    return orc.Level(rgb, tex, occ, with_layers=layers)


def _xyz(lv, p):
    p = int(p)
    return p % lv.W, (p // lv.W) % lv.H, p // (lv.W * lv.H)


def _lin(lv, x, y, t):
    return (t * lv.H + y) * lv.W + x


# ------------------------------------------------------------------------- Eq. 13 / Alg. 3
def _onion_world(orc):
    """W=40, H=T=15; hole = 7x7x7 box x in [16,23), y,t in [4,11) -> layers 1..4.  Known colour
    200 for x < 8 and 100 for x >= 32.  Contributors with layer < j get shift +16 (p + phi lands
    in the 100 region), all others shift -15 (lands in the 200 region)."""
    T, H, W = 15, 15, 40
    rgb = np.full((T, H, W, 3), 150, np.uint8)
    rgb[:, :, :8] = 200
    rgb[:, :, 32:] = 100
    occ = np.zeros((T, H, W), np.uint8)
    occ[4:11, 4:11, 16:23] = 1
    lv = _level(orc, rgb, occ, layers=True)
    assert lv.n_layers == 4
    return lv


def _onion_nnf(orc, lv, j):
    nt = len(lv.targets)
    nnf = orc.NNF.empty(nt)
    lay = lv.layer.ravel()[lv.targets]
    nnf.dx[:nt] = np.where(lay < j, 16, -15)
    nnf.D[:nt] = np.arange(nt) % 997 + 1
    nnf.n[:nt] = 125
    return nnf


@pytest.mark.parametrize("mode", ["weighted", "unweighted"])
def test_eq13_layer_contributors_exclude_own_layer(orc, mode):
    """Every contributor with layer(q) < j proposes 100, every other one 200: Eq. 13's N'_p gives
    exactly 100 at every layer-j voxel; counting layer-j contributors (<= j) would pull it up."""
    lv = _onion_world(orc)
    m = orc.WEIGHTED if mode == "weighted" else orc.UNWEIGHTED
    for j in range(1, lv.n_layers + 1):
        nnf = _onion_nnf(orc, lv, j)
        out, tex = orc.reconstruct(lv, nnf, m, layer_j=j)
        lay = lv.layer.ravel()[lv.holes]
        assert (lay == j).any()
        assert np.array_equal(out[lay == j], np.full(((lay == j).sum(), 3), 100, np.float32)), j


def test_onion_layer_reconstruction_writes_only_its_layer(orc):
    """reconstructing layer j touches exactly the layer-j hole rows; over all layers
    every hole voxel is written exactly once."""
    lv = _onion_world(orc)
    nh = len(lv.holes)
    writes = np.zeros(nh, np.int32)
    for j in range(1, lv.n_layers + 1):
        nnf = _onion_nnf(orc, lv, j)
        out = np.full((nh, 3), -1.0, np.float32)
        tex = np.full((nh, 2), -1.0, np.float32)
        orc.reconstruct(lv, nnf, orc.WEIGHTED, layer_j=j, out_rgb=out, out_tex=tex)
        written = (out != -1.0).all(1)
        untouched = (out == -1.0).all(1)
        assert (written | untouched).all()
        assert np.array_equal(written, lv.layer.ravel()[lv.holes] == j), j
        writes += written
    assert (writes == 1).all()


def test_onion_peel_commits_each_hole_voxel_once(orc):
    """Alg. 3 inside or_inpaint: the number of hole-voxel commits during the peel equals |H| at
    the coarsest level, for a 1-level and a 2-level run."""
    v, m, _ = generate("c1")
    for L in (1, 2):
        _, st = orc.inpaint(v.numpy(), m.numpy(), L, pm_iters=2, fixed_outer=1)
        assert st["onion_commits"] == st["n_holes"][L - 1]


# ------------------------------------------------------------------------- R25 ties
def _tie_world(orc, constant=False, seed=7):
    T, H, W = 16, 18, 32
    rng = np.random.default_rng(seed)
    rgb = (np.full((T, H, W, 3), 9, np.uint8) if constant
           else rng.integers(0, 256, (T, H, W, 3), dtype=np.uint8))
    occ = np.zeros((T, H, W), np.uint8)
    occ[5:7, 6:8, 12:15] = 1
    return _level(orc, rgb, occ)


def _valid_shift(lv, p, v):
    x, y, t = _xyz(lv, p)
    qx, qy, qt = x + v[0], y + v[1], t + v[2]
    if not (0 <= qx < lv.W and 0 <= qy < lv.H and 0 <= qt < lv.T):
        return False
    return lv.src.ravel()[_lin(lv, qx, qy, qt)] == 1


def _pick_target(lv, step, sign):
    """A hole voxel (hence a target) whose sign*step neighbours along x, y, t are targets."""
    for p in lv.holes:
        s = int(lv.slot[p])
        x, y, t = _xyz(lv, p)
        nb = [(x + sign * step, y, t), (x, y + sign * step, t), (x, y, t + sign * step)]
        if all(0 <= a < lv.W and 0 <= b < lv.H and 0 <= c < lv.T for a, b, c in nb):
            sl = [lv.slot[_lin(lv, *n)] for n in nb]
            if min(sl) >= 0:
                return s, int(p), sl
    raise AssertionError("no interior target")


def _set(nnf, s, v, D=None, n=125):
    nnf.dx[s], nnf.dy[s], nnf.dt[s] = v
    if D is not None:
        nnf.D[s] = D
    nnf.n[s] = n


def _shift(nnf, s):
    return (int(nnf.dx[s]), int(nnf.dy[s]), int(nnf.dt[s]))


def test_propagation_equal_distance_keeps_incumbent(orc):
    """P:379 'smaller': a neighbour's shift whose distance equals the incumbent's does not replace
    it; one unit more on the incumbent and it does."""
    lv = _tie_world(orc)
    lam = 50
    s, p, (sx, sy, st_) = _pick_target(lv, 1, 1)
    v0, v1 = (-9, 0, 0), (10, 0, 0)
    assert _valid_shift(lv, p, v0) and _valid_shift(lv, p, v1)
    x, y, t = _xyz(lv, p)
    D1, _ = orc.patch_ssd(lv, p, _lin(lv, x + v1[0], y, t), lam)
    D0, _ = orc.patch_ssd(lv, p, _lin(lv, x + v0[0], y, t), lam)
    assert D0 != D1
    nt = len(lv.targets)
    for incumbent_D, expect in ((D1, v0), (D1 + 1, v1)):
        a = orc.NNF.empty(nt)
        a.dx[:nt], a.n[:nt], a.D[:nt] = v0[0], 125, 0
        _set(a, s, v0, incumbent_D)   # stored distance (stale on purpose: only the rule matters)
        _set(a, sx, v1, 0)            # rank 1: the x neighbour proposes v1
        _set(a, sy, v0, 0)            # y and t neighbours propose the incumbent (duplicates)
        _set(a, st_, v0, 0)
        b = a.copy()
        orc.propagate(lv, a, b, lam, 1, 1)
        assert _shift(b, s) == expect
        assert b.D[s] == min(incumbent_D, D1)


@pytest.mark.parametrize("sign", [1, -1, 0])
def test_propagation_equal_new_candidates_lowest_rank_wins(orc, sign):
    """Constant video: every candidate has D = 0 < the incumbent's 1, so the lowest-rank candidate
    (x before y before t; sign 0: the -step neighbours first) must win."""
    lv = _tie_world(orc, constant=True)
    step = 2
    nt = len(lv.targets)
    s, p, sl = _pick_target(lv, step, sign if sign else -1)
    vs = [(-9, 0, 0), (10, 0, 0), (0, 6, 0), (0, 0, 5)]
    assert all(_valid_shift(lv, p, v) for v in vs)
    a = orc.NNF.empty(nt)
    a.dx[:nt], a.n[:nt] = -9, 125
    _set(a, s, vs[0], 1)
    for k, r in enumerate(sl):
        _set(a, r, vs[k + 1], 0)
    if sign == 0:  # the +step neighbours are ranks 4-6 and propose yet other shifts
        x, y, t = _xyz(lv, p)
        for k, n in enumerate([(x + step, y, t), (x, y + step, t), (x, y, t + step)]):
            r = lv.slot[_lin(lv, *n)]
            if r >= 0:
                _set(a, r, ((-8, 0, 0), (-7, 0, 0), (11, 0, 0))[k], 0)
    b = a.copy()
    orc.propagate(lv, a, b, 50, step, sign)
    assert _shift(b, s) == vs[1] and b.D[s] == 0


def test_random_search_equal_distance_keeps_incumbent(orc):
    """P:438 '<': constant video with every stored D = 0 -> no candidate may replace anything,
    although candidates are evaluated."""
    lv = _tie_world(orc, constant=True)
    nt = len(lv.targets)
    a = orc.NNF.empty(nt)
    orc.init_random(lv, a, 3, 1, 0)
    orc.evaluate(lv, a, 50)
    assert (a.D[:nt] == 0).all()
    b = a.copy()
    cnt = orc.random_search(lv, a, b, 50, 3, 0.5, lv.rmax, 1, 0, 1)
    assert cnt > nt
    for f in ("dx", "dy", "dt", "D"):
        assert np.array_equal(getattr(a, f)[:nt], getattr(b, f)[:nt]), f


def test_random_search_equal_new_candidates_first_wins(orc):
    """Constant video, stored D = 1: every valid candidate has D = 0; the first valid one (rank
    i = 1 when valid) must win.  Candidate 1 is derived here from Philox (pinned against cuRAND)
    and Eq. 3: R_1 = rmax rho, offset = floor(R_1 (U - 2^31) 2^-31)."""
    lv = _tie_world(orc, constant=True)
    nt = len(lv.targets)
    seed, level, outer, k, rho = 11, 1, 3, 2, 0.5
    a = orc.NNF.empty(nt)
    orc.init_random(lv, a, seed, level, 0)
    orc.evaluate(lv, a, 50)
    a.D[:nt] = 1
    b = a.copy()
    orc.random_search(lv, a, b, 50, seed, rho, lv.rmax, level, outer, k)
    R1 = lv.rmax * rho
    checked = 0
    for s, p in enumerate(lv.targets):
        u = orc.philox([int(p), k, (level << 24) | (2 << 16) | 1, outer], seed)
        off = [int(np.floor(R1 * ((float(u[c]) - 2.0 ** 31) / 2.0 ** 31))) for c in range(3)]
        v = (int(a.dx[s]) + off[0], int(a.dy[s]) + off[1], int(a.dt[s]) + off[2])
        if v != _shift(a, s) and _valid_shift(lv, p, v):
            assert _shift(b, s) == v and b.D[s] == 0
            checked += 1
    assert checked >= 10


# ------------------------------------------------------------------------- R19 stopping rule
def test_stop_rule_constructed(orc):
    """e = e_fixed / 2^20 / (3|H|): stop iff e <= 0.1, or k = 20."""
    nh = 10  # 0.1 * 3|H| * 2^20 = 3 * 2^20
    edge = 3 * 2 ** 20
    assert orc.stop(edge, nh, 1)
    assert not orc.stop(edge + 1, nh, 1)
    assert not orc.stop(10 * edge, nh, 19)
    assert orc.stop(10 * edge, nh, 20)
    assert orc.stop(0, nh, 1)
    # e = 0.5 and e = 1.0 continue (a threshold of 1.0 would stop here)
    assert not orc.stop(5 * edge, nh, 1) and not orc.stop(10 * edge, nh, 1)
    # literal P:988 form: sqrt(e2 / 2^20) / (3|H|) <= 0.1  <=>  e2 <= 0.09 |H|^2 2^20
    e2 = 9 * nh * nh * 2 ** 20 // 100
    assert orc.stop(e2, nh, 1, stop_rule=1) and not orc.stop(e2 + 1, nh, 1, stop_rule=1)


def test_change_l2_constructed(orc):
    a = np.array([1.0, 2.5, 100.0, 0.25], np.float32)
    b = np.array([0.5, 3.0, 100.0, 1.0], np.float32)
    assert orc.change_l2(a, b) == int((0.25 + 0.25 + 0 + 0.5625) * 2 ** 20)


@pytest.mark.parametrize("levels", [1, 2])
def test_stop_rule_in_pipeline(orc, levels):
    """or_inpaint's outer-iteration counts obey the rule on the recorded change statistics: every
    level continues while e > 0.1 and stops at the first e <= 0.1 (or at max_outer).  The c1 runs
    pass through 0.1 < e <= 1 before stopping, so a wrong threshold changes k."""
    v, m, _ = generate("c1")
    _, st = orc.inpaint(v.numpy(), m.numpy(), levels, pm_iters=4)
    saw_mid = False
    for l in range(levels):
        k, nh, es = st["outer_iters"][l], st["n_holes"][l], st["change_fixed"][l]
        e = [x / 2 ** 20 / (3 * nh) for x in es]
        assert len(e) == k
        assert all(x > 0.1 for x in e[:-1]) and (e[-1] <= 0.1 or k == 20), (l, e)
        saw_mid |= any(0.1 < x <= 1.0 for x in e)
    assert saw_mid
    # the iteration cap decides when it is reached first
    _, st2 = orc.inpaint(v.numpy(), m.numpy(), levels, pm_iters=4, max_outer=2)
    assert st2["outer_iters"] == [2] * levels


# ------------------------------------------------------------------------- R20
def test_unweighted_after_upsampling_uses_all_contributors(orc):
    """Right after upsampling no distances exist (n = 0 everywhere): Eq. 4 with s = 1 still
    averages every contributor; WEIGHTED has no defined distances and writes nothing."""
    T, H, W = 11, 11, 30
    rgb = np.full((T, H, W, 3), 150, np.uint8)
    rgb[:, :, 22:] = 100
    rgb[:, :, :4] = 220
    occ = np.zeros((T, H, W), np.uint8)
    occ[5, 5, 12] = 1
    lv = _level(orc, rgb, occ)
    nt = len(lv.targets)
    nnf = orc.NNF.empty(nt)
    nnf.dx[:nt] = np.where(np.arange(nt) % 3 == 0, -10, 12)  # -> x = 2 (220) or x = 24 (100)
    nnf.n[:nt] = 0
    out, _ = orc.reconstruct(lv, nnf, orc.UNWEIGHTED)
    k220 = int((np.arange(nt) % 3 == 0).sum())
    assert nt == 125
    assert out[0] == pytest.approx([(k220 * 220 + (nt - k220) * 100) / nt] * 3, abs=1e-4)
    sent = np.full((1, 3), -1.0, np.float32)
    orc.reconstruct(lv, nnf, orc.WEIGHTED, out_rgb=sent, out_tex=np.full((1, 2), -1.0, np.float32))
    assert (sent == -1.0).all()


def test_upsample_then_unweighted_matches_brute_mean(orc):
    """The same on a real level transition: a coarse NNF upsampled, n = 0, then the
    unweighted mean of u(p + phi(q)) over N_p (direct double loop)."""
    v, m, _ = generate("c1")
    rgb, occ = v.numpy(), m.numpy()
    rc, oc = orc.pyramid_down(rgb, occ)
    coarse = _level(orc, rc, oc)
    fine = _level(orc, rgb, occ)
    cn = orc.NNF.empty(len(coarse.targets))
    orc.init_random(coarse, cn, 4, 2, 0)
    fn = orc.NNF.empty(len(fine.targets))
    orc.upsample(coarse, cn, fine, fn, 4, 1)
    assert (fn.n[:len(fine.targets)] == 0).all()
    out, _ = orc.reconstruct(fine, fn, orc.UNWEIGHTED)
    rng = np.random.default_rng(0)
    for h in rng.choice(len(fine.holes), 40, replace=False):
        x, y, t = _xyz(fine, fine.holes[h])
        vals = []
        for dt in range(-2, 3):
            for dy in range(-2, 3):
                for dx in range(-2, 3):
                    qx, qy, qt = x + dx, y + dy, t + dt
                    if 0 <= qx < fine.W and 0 <= qy < fine.H and 0 <= qt < fine.T:
                        s = fine.slot[_lin(fine, qx, qy, qt)]
                        vals.append(fine.rgb[t + fn.dt[s], y + fn.dy[s], x + fn.dx[s]].astype(np.float64))
        assert np.allclose(out[h], np.mean(vals, 0), atol=1e-4)


# ------------------------------------------------------------------------- R33 counts
def test_random_search_counts_distinct_valid_candidates(orc):
    """R33/R34: a random-search candidate equal to the incumbent or to an earlier valid candidate
    is neither evaluated nor counted.  rmax = 4, rho = 1/2: radii R_1 = 2, R_2 = 1, so offsets lie
    in [-2, 1] and [-1, 0] and repeats are frequent; the count is derived here from Philox (pinned
    against cuRAND) and Eq. 3."""
    lv = _tie_world(orc)
    nt = len(lv.targets)
    seed, level, outer, k = 5, 1, 0, 1
    a = orc.NNF.empty(nt)
    orc.init_random(lv, a, seed, level, 0)
    orc.evaluate(lv, a, 50)
    b = a.copy()
    cnt = orc.random_search(lv, a, b, 50, seed, 0.5, 4, level, outer, k)
    ref = dups = 0
    for s, p in enumerate(lv.targets):
        seen = {_shift(a, s)}
        for i, R in ((1, 2.0), (2, 1.0)):
            u = orc.philox([int(p), k, (level << 24) | (2 << 16) | i, outer], seed)
            off = [int(np.floor(R * ((float(u[c]) - 2.0 ** 31) / 2.0 ** 31))) for c in range(3)]
            v = (int(a.dx[s]) + off[0], int(a.dy[s]) + off[1], int(a.dt[s]) + off[2])
            if not _valid_shift(lv, p, v):
                continue
            if v in seen:
                dups += 1
                continue
            seen.add(v)
            ref += 1
    assert dups > 10
    assert cnt == ref


def test_driver_stop_decision_equals_oracle(orc):
    """The driver's host-side loop exit (driver.stop_now, python integers) takes the oracle's
    decision (or_stop, __int128) on random and boundary statistics, for both norms."""
    from paper_1503_05528_b200.driver import stop_now
    import random
    rng = random.Random(1)
    for _ in range(3000):
        nh = rng.randint(1, 20_000_000)
        rule = rng.randint(0, 1)
        edge = 3 * nh * 2 ** 20 // 10 if rule == 0 else 9 * nh * nh * 2 ** 20 // 100
        e = max(0, edge + rng.randint(-3, 3)) if rng.random() < 0.5 else rng.randint(0, 4 * edge + 2)
        e = min(e, 2 ** 63 - 1)  # the statistic is an int64 on both sides
        k = rng.randint(1, 21)
        assert stop_now(e, nh, k, 20, rule) == orc.stop(e, nh, k, 20, rule), (e, nh, k, rule)


# ------------------------------------------------------------------------- R41 stale candidates
def _candidates(lv, f, s, step, sign):
    """The propagation candidates of target slot s that are evaluated (Alg. 1 P:418-434 with R2,
    R6): neighbour r = p + sg*step*e_axis in H~, shift v = phi(r) valid at p, v different from the
    incumbent and every earlier candidate.  Returns [(rank, neighbour slot, v)]."""
    p = int(lv.targets[s])
    x, y, t = _xyz(lv, p)
    seen = [_shift(f, s)]
    out = []
    order = [(sign, a) for a in range(3)] if sign else [(-1, a) for a in range(3)] + [(1, a) for a in range(3)]
    for rank, (sg, ax) in enumerate(order, start=1):
        r = [x, y, t]
        r[ax] += sg * step
        if not (0 <= r[0] < lv.W and 0 <= r[1] < lv.H and 0 <= r[2] < lv.T):
            continue
        rs = int(lv.slot[_lin(lv, *r)])
        if rs < 0:
            continue
        v = _shift(f, rs)
        if not _valid_shift(lv, p, v) or v in seen:
            continue
        seen.append(v)
        out.append((rank, rs, v))
    return out


@pytest.mark.parametrize("sign_policy", [0, 1])
def test_stale_candidates_brute_force(orc, sign_policy):
    """R41 by brute force on a tiny level: a candidate whose neighbour holds the same shift as at
    the previous pass with the same (step, sign) of the search is (i) counted exactly as the
    oracle's stale count and (ii) never strictly better than the target's incumbent, which is
    why the GPU may skip it without changing the NNF (strict improvement, R25)."""
    from gen.synth import random_volume
    v, m, _ = random_volume(22, 18, 9, seed=3, hole_frac=0.08)
    rgb, occ = v.numpy(), m.numpy()
    lv = _level(orc, rgb, occ, tex=orc.texture(rgb, occ, 1))
    lam = 50
    nt = len(lv.targets)
    f = orc.NNF.empty(nt)
    orc.init_random(lv, f, 1, 1, 0)
    orc.evaluate(lv, f, lam)
    snaps = {}
    n_stale_total = 0
    for k in range(1, 7):
        sign = 0 if sign_policy else (1 if k % 2 else -1)
        for step in (4, 2, 1):
            prev = snaps.get((step, sign))
            want = 0
            for s in range(nt):
                for rank, rs, cand in _candidates(lv, f, s, step, sign):
                    if prev is not None and _shift(prev, rs) == cand:
                        want += 1
                        x, y, t = _xyz(lv, lv.targets[s])
                        q = _lin(lv, x + cand[0], y + cand[1], t + cand[2])
                        D, _ = orc.patch_ssd(lv, int(lv.targets[s]), q, lam)
                        assert D >= int(f.D[s]), (k, step, s, rank)
            g = f.copy()
            st = np.zeros(1, np.int64)
            orc.propagate(lv, f, g, lam, step, sign, prev=prev, stale=st)
            assert int(st[0]) == want, (k, step)
            n_stale_total += want
            snaps[(step, sign)] = f
            f = g
        g = f.copy()
        orc.random_search(lv, f, g, lam, 1, 0.5, lv.rmax, 1, 0, k)
        f = g
    assert n_stale_total > 0
