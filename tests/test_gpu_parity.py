"""GPU (libvinp, sm_100a) vs CPU oracle parity, stage by stage, through the C ABI.

Integer work (pyramid, features, sets, SSDs, NNFs, counts) must be bit-exact; reconstructed
pixel values within 1e-3 (north_star).  Stage-wise: the oracle is fed the GPU's state at each
stage boundary (SURVEY §7 "Hard parts"), then the end-to-end c1 pipeline is compared as a whole.
"""
import numpy as np
import pytest
import torch

from gen.synth import generate, random_volume
import _bridge as B

pytestmark = pytest.mark.gpu

CASES = {
    "c1": dict(src=("c1",), levels=1),
    "c2": dict(src=("c2",), levels=2),
    "odd": dict(src=("rand", 45, 37, 11, 7), levels=3),
}


def _input(case):
    s = CASES[case]["src"]
    if s[0] == "rand":
        v, m, _ = random_volume(s[1], s[2], s[3], seed=s[4], hole_frac=0.06)
    else:
        v, m, _ = generate(s[0])
    return v, m


@pytest.fixture(scope="module")
def V():
    from paper_1503_05528_b200 import vinp
    return vinp


_cache = {}


def _setup(case, lam=50):
    key = (case, lam)
    if key in _cache:
        return _cache[key]
    from paper_1503_05528_b200 import Config, Inpainter
    v, m = _input(case)
    T, H, W, _ = v.shape
    cfg = Config(levels=CASES[case]["levels"], lam=lam)
    ip = Inpainter(W, H, T, cfg, "cuda")
    ip.load(v.cuda(), m.cuda())
    torch.cuda.synchronize()
    _cache[key] = (ip, v.numpy(), m.numpy())
    return _cache[key]


# ----------------------------------------------------------------------------- Philox
def test_philox_gpu_vs_oracle(V, orc):
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2 ** 32, (4096, 4), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0
    ctr[1] = 0xFFFFFFFF
    for seed in (0, 5, 0xFFFFFFFFFFFFFFFF, 0x243F6A8885A308D3):
        g = V.philox(torch.from_numpy(ctr.view(np.int32)).cuda(), seed).cpu().numpy().view(np.uint32)
        for i in range(0, 4096, 97):
            assert list(g[i]) == list(orc.philox(ctr[i], seed))


# ----------------------------------------------------------------------------- setup stages
@pytest.mark.parametrize("case", list(CASES))
def test_pyramid_texture_sets_bit_exact(orc, case):
    ip, rgb, occ = _setup(case)
    L = ip.cfg.levels
    o_rgb, o_occ = [rgb], [occ]
    for l in range(1, L):
        r, o = orc.pyramid_down(o_rgb[-1], o_occ[-1])
        o_rgb.append(r)
        o_occ.append(o)
    h = max(1, 2 ** (L - 2)) if L >= 2 else 1
    tex1 = orc.texture(rgb, occ, h)
    for l, lv in enumerate(ip.levels):
        g_rgb, g_tex, g_flags = B.level_to_host(lv)
        assert np.array_equal(g_flags & 1, o_occ[l]), f"occlusion level {l + 1}"
        assert np.array_equal(g_rgb[~o_occ[l].astype(bool)], o_rgb[l][~o_occ[l].astype(bool)]), \
            f"colour level {l + 1}"
        # hole colour at coarse levels is 0 in both (masked filter of occluded coarse voxels)
        assert np.array_equal(g_rgb, o_rgb[l]) or l == 0
        o_tex = tex1 if l == 0 else orc.texture_decimate(tex1, l + 1, lv.W, lv.H)
        assert np.array_equal(g_tex, o_tex), f"texture level {l + 1}"
        src, tgt = orc.sets(o_occ[l])
        assert np.array_equal((g_flags >> 1) & 1, src) and np.array_equal((g_flags >> 2) & 1, tgt)
        assert lv.n_targets == int(tgt.sum()) and lv.n_holes == int(o_occ[l].sum())
        assert lv.n_sources == int(src.sum())
        assert np.array_equal(lv.targets[:lv.n_targets].cpu().numpy(), np.flatnonzero(tgt.ravel()))
        assert np.array_equal(lv.holes[:lv.n_holes].cpu().numpy(), np.flatnonzero(o_occ[l].ravel()))
        assert np.array_equal(lv.sources[:lv.n_sources].cpu().numpy(), np.flatnonzero(src.ravel()))
        slot = np.full(lv.N, -1, np.int64)
        slot[np.flatnonzero(tgt.ravel())] = np.arange(int(tgt.sum()))
        assert np.array_equal(lv.slot.cpu().numpy(), slot)
    top = ip.levels[-1]
    lay, n = orc.layers(o_occ[-1])
    assert ip.n_layers == n
    assert np.array_equal(top.layer.view(top.T, top.H, top.W).cpu().numpy(), lay)


def test_c2_set_sizes_match_survey_appendix():
    ip, _, _ = _setup("c2")
    lv1, lv2 = ip.levels
    assert (lv1.n_holes, lv1.n_targets, lv1.n_sources) == (180540, 212700, 3977736)
    assert (lv2.n_holes, lv2.n_targets, lv2.n_sources) == (47100, 63900, 953736)
    assert ip.n_layers == 11


# ----------------------------------------------------------------------------- SSD
@pytest.mark.parametrize("case", ["c1", "odd"])
@pytest.mark.parametrize("lam", [0, 50, 126])
def test_patch_ssd_bit_exact(V, orc, case, lam):
    ip, _, _ = _setup(case)
    lv = ip.levels[-1]
    ol = B.oracle_level(orc, lv, layers=True)
    rng = np.random.default_rng(lam)
    n = 3000
    p = rng.choice(lv.N, n).astype(np.int32)
    p[:50] = np.arange(50)  # volume corner: clipped patches (R23)
    q = lv.sources[:lv.n_sources].cpu().numpy()[rng.integers(0, lv.n_sources, n)]
    prm = V.Params(lam=lam)
    for kb in (-1, 1, 2):
        D, c = V.patch_ssd(lv, torch.from_numpy(p).cuda(), torch.from_numpy(q).cuda(), prm, kb)
        D, c = D.cpu().numpy().view(np.uint32), c.cpu().numpy()
        for i in range(0, n, 7):
            assert (int(D[i]), int(c[i])) == orc.patch_ssd(ol, p[i], q[i], lam, kb), (i, kb)


# ----------------------------------------------------------------------------- NNF passes
def _fresh_nnf(V, ip, lv, seed_outer=0):
    st = ip.states[lv.level - 1]
    a = V.NNF.alloc(lv.n_targets, "cuda")
    b = V.NNF.alloc(lv.n_targets, "cuda", n=a.n)
    V.nnf_init_random(lv, a, ip.prm, seed_outer)
    return a, b


@pytest.mark.parametrize("case", ["c1", "c2", "odd"])
def test_init_evaluate_propagate_random_search_bit_exact(V, orc, case):
    ip, _, _ = _setup(case)
    for lv in ip.levels:
        ol = B.oracle_level(orc, lv)
        lam, seed = ip.prm.lam, ip.prm.seed
        a, b = _fresh_nnf(V, ip, lv, 7)
        f = orc.NNF.empty(lv.n_targets)
        orc.init_random(ol, f, seed, lv.level, 7)
        assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0, "init"
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        V.nnf_evaluate(lv, a, ip.prm, counter=cnt)
        c_o = orc.evaluate(ol, f, lam)
        assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0, "evaluate"
        assert int(cnt.item()) == c_o
        g = f.copy()
        for k, (step, sign) in enumerate([(8, 1), (4, 1), (2, 1), (1, 1), (1, -1), (4, -1), (2, 0), (1, 0)]):
            cnt.zero_()
            V.propagate(lv, a, b, ip.prm, step, sign, counter=cnt)
            c_o = orc.propagate(ol, f, g, lam, step, sign)
            assert len(B.nnf_equal(orc, lv, b.e, b.n, g)) == 0, f"propagate {step},{sign}"
            assert int(cnt.item()) == c_o
            a, b = b, a
            f, g = g, f
            cnt.zero_()
            V.random_search(lv, a, b, ip.prm, 3, k + 1, counter=cnt)
            c_o = orc.random_search(ol, f, g, lam, seed, 0.5, lv.rmax, lv.level, 3, k + 1)
            assert len(B.nnf_equal(orc, lv, b.e, b.n, g)) == 0, f"random search {k + 1}"
            assert int(cnt.item()) == c_o
            a, b = b, a
            f, g = g, f


def test_onion_restricted_passes_bit_exact(V, orc):
    ip, _, _ = _setup("c2")
    lv = ip.levels[-1]
    ol = B.oracle_level(orc, lv, layers=True)
    lam, seed = ip.prm.lam, ip.prm.seed
    a, b = _fresh_nnf(V, ip, lv, 0)
    f = orc.NNF.empty(lv.n_targets)
    orc.init_random(ol, f, seed, lv.level, 0)
    for j in (0, 1, 3):
        kb = max(j, 1)
        oc = V.ONION | j
        V.nnf_evaluate(lv, a, ip.prm, kb, j)
        orc.evaluate(ol, f, lam, kb, j)
        assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0
        # the warp-per-target onion kernels: both sign policies (3 and 6 candidates per target)
        for step, sign in ((2, -1), (1, 0), (4, 1)):
            g = f.copy()
            V.propagate(lv, a, b, ip.prm, step, sign, kb, j)
            orc.propagate(ol, f, g, lam, step, sign, kb, j)
            assert len(B.nnf_equal(orc, lv, b.e, b.n, g)) == 0
            a, b = b, a
            f = g
        a, b = b, a  # b: the last propagation result
        g, f = f, f.copy()
        V.random_search(lv, b, a, ip.prm, oc, 1, kb, j)
        orc.random_search(ol, g, f, lam, seed, 0.5, lv.rmax, lv.level, oc, 1, kb, j)
        assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0


@pytest.mark.parametrize("case", ["c1", "odd"])
def test_ann_search_schedule_bit_exact(V, orc, case):
    ip, _, _ = _setup(case)
    lv = ip.levels[0]
    ol = B.oracle_level(orc, lv)
    a, b = _fresh_nnf(V, ip, lv, 11)
    f = orc.NNF.empty(lv.n_targets)
    orc.init_random(ol, f, ip.prm.seed, lv.level, 11)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    V.ann_search(lv, a, b, ip.prm, 11, 10, counter=cnt)
    f, c_o = orc.ann_search(ol, f, ip.prm.lam, ip.prm.seed, lv.level, 11, 10)
    assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0
    assert int(cnt.item()) == c_o


def test_upsample_bit_exact(V, orc):
    ip, _, _ = _setup("odd")
    for l in range(len(ip.levels) - 1, 0, -1):
        c, fl = ip.levels[l], ip.levels[l - 1]
        oc, of = B.oracle_level(orc, c), B.oracle_level(orc, fl)
        a, _ = _fresh_nnf(V, ip, c, 2)
        fa = V.NNF.alloc(fl.n_targets, "cuda")
        V.nnf_upsample(c, a, fl, fa, ip.prm)
        fc = B.nnf_to_oracle(orc, c, a.e, a.n)
        ff = orc.NNF.empty(fl.n_targets)
        orc.upsample(oc, fc, of, ff, ip.prm.seed, fl.level)
        assert len(B.nnf_equal(orc, fl, fa.e, fa.n, ff)) == 0


# ----------------------------------------------------------------------------- reconstruction
@pytest.mark.parametrize("case", ["c1", "odd"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_reconstruct_matches_oracle(V, orc, case, mode):
    ip, _, _ = _setup(case)
    lv = ip.levels[0]
    a, b = _fresh_nnf(V, ip, lv, 5)
    V.ann_search(lv, a, b, ip.prm, 5, 2)
    ol = B.oracle_level(orc, lv)
    f = B.nnf_to_oracle(orc, lv, a.e, a.n)
    vox0 = lv.vox.clone()
    nh = lv.n_holes
    g_rgb = torch.zeros((nh, 3), dtype=torch.float32, device="cuda")
    g_tex = torch.zeros((nh, 2), dtype=torch.float32, device="cuda")
    V.reconstruct(lv, a, mode, g_rgb, g_tex, commit=True)
    o_rgb, o_tex = orc.reconstruct(ol, f, mode)
    d = max(np.abs(g_rgb.cpu().numpy() - o_rgb[:nh]).max(), np.abs(g_tex.cpu().numpy() - o_tex[:nh]).max())
    assert d <= 1e-3, d
    exact = np.mean(g_rgb.cpu().numpy() == o_rgb[:nh])
    assert exact > 0.999
    orc.commit(ol, o_rgb, o_tex)
    g_rgb8, g_tex8, _ = B.level_to_host(lv)
    assert np.array_equal(g_rgb8, ol.rgb) and np.array_equal(g_tex8, ol.tex)
    lv.vox.copy_(vox0)


def test_onion_layer_reconstruct_matches_oracle(V, orc):
    ip, _, _ = _setup("c2")
    lv = ip.levels[-1]
    a, b = _fresh_nnf(V, ip, lv, 0)
    vox0 = lv.vox.clone()
    nh = lv.n_holes
    g_rgb = torch.zeros((nh, 3), dtype=torch.float32, device="cuda")
    g_tex = torch.zeros((nh, 2), dtype=torch.float32, device="cuda")
    o_rgb = np.zeros((nh, 3), np.float32)
    o_tex = np.zeros((nh, 2), np.float32)
    for j in range(0, 4):
        V.ann_search(lv, a, b, ip.prm, V.ONION | j, 2, kb=max(j, 1), only_layer=j)
        if j == 0:
            continue
        ol = B.oracle_level(orc, lv, layers=True)
        f = B.nnf_to_oracle(orc, lv, a.e, a.n)
        V.reconstruct(lv, a, 0, g_rgb, g_tex, layer_j=j, commit=True)
        orc.reconstruct(ol, f, 0, layer_j=j, out_rgb=o_rgb, out_tex=o_tex)
        sel = ol.layer.ravel()[ol.holes] == j
        assert sel.any()
        assert np.abs(g_rgb.cpu().numpy()[sel] - o_rgb[sel]).max() <= 1e-3
        assert np.abs(g_tex.cpu().numpy()[sel] - o_tex[sel]).max() <= 1e-3
    lv.vox.copy_(vox0)


def test_change_l1_and_energy(V, orc):
    rng = np.random.default_rng(1)
    a = (rng.random(100003) * 255).astype(np.float32)
    b = (rng.random(100003) * 255).astype(np.float32)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    V.change_l1(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), out)
    assert int(out.item()) == orc.change_l1(a, b)
    ip, _, _ = _setup("c1")
    lv = ip.levels[0]
    x, y = _fresh_nnf(V, ip, lv, 1)
    V.nnf_evaluate(lv, x, ip.prm)
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    V.energy(lv, x, E)
    ol = B.oracle_level(orc, lv)
    assert float(E.item()) == pytest.approx(orc.energy(ol, B.nnf_to_oracle(orc, lv, x.e, x.n)), rel=1e-12)


def test_brute_force_bit_exact(V, orc):
    ip, _, _ = _setup("c1")
    lv = ip.levels[0]
    out = V.NNF.alloc(lv.n_targets, "cuda")
    V.brute_force(lv, out, ip.prm, 0, 600)
    ol = B.oracle_level(orc, lv)
    f = orc.NNF.empty(lv.n_targets)
    orc.brute_force(ol, f, ip.prm.lam, 0, 600)
    g = B.nnf_to_oracle(orc, lv, out.e, out.n)
    for arr in ("dx", "dy", "dt", "D", "n"):
        assert np.array_equal(getattr(g, arr)[:600], getattr(f, arr)[:600]), arr


# ----------------------------------------------------------------------------- end to end
def test_pipeline_c1_end_to_end(orc):
    from paper_1503_05528_b200 import Config, inpaint
    v, m, _ = generate("c1")
    cfg = Config(levels=1, pm_iters=4, fixed_outer=3)
    out, stats, ip = inpaint(v, m, cfg)
    ref, st = orc.inpaint(v.numpy(), m.numpy(), 1, pm_iters=4, fixed_outer=3)
    g = out.cpu().numpy()
    assert np.array_equal(g, ref)
    # R41: the GPU skips the stale candidates the oracle evaluates (and counts them apart)
    assert stats.total_patch_updates == sum(st["patch_updates"]) - sum(st["stale"])
    assert stats.total_stale_skipped == sum(st["stale"]) > 0
    assert stats.onion_layers == st["onion_layers"]


def test_pipeline_two_levels_end_to_end(orc):
    from paper_1503_05528_b200 import Config, inpaint
    v, m, _ = random_volume(64, 48, 12, seed=9, hole_frac=0.05)
    cfg = Config(levels=2, pm_iters=3, max_outer=4)
    out, stats, ip = inpaint(v, m, cfg)
    ref, st = orc.inpaint(v.numpy(), m.numpy(), 2, pm_iters=3, max_outer=4)
    assert [l["outer"] for l in stats.levels] == st["outer_iters"]
    assert np.array_equal(out.cpu().numpy(), ref)


def test_native_onion_peel_equals_stepwise(V):
    """vinp_onion_peel (per-layer lists, one call) == the per-pass only_layer path, bit for bit."""
    from paper_1503_05528_b200 import Config, Inpainter
    v, m, _ = generate("c2")
    T, H, W, _ = v.shape
    res = []
    for native in (True, False):
        ip = Inpainter(W, H, T, Config(levels=2, pm_iters=3), "cuda")
        ip.load(v.cuda(), m.cuda())
        ip.counter.zero_()
        (ip.onion_peel if native else ip.onion_peel_stepwise)()
        st = ip.states[-1]
        torch.cuda.synchronize()
        res.append((st.a.e.clone(), st.a.n.clone(), st.cur_rgb.clone(), st.cur_tex.clone(),
                    st.lv.vox.clone(), tuple(ip.counter.tolist())))
    for x, y in zip(res[0][:5], res[1][:5]):
        assert torch.equal(x, y)
    assert res[0][5] == res[1][5]


def test_pipeline_c2_full_config_end_to_end(orc):
    """BASELINE c2 as configured (2 levels, K = 10, stopping rule, max 20): the whole Alg. 4 on the
    GPU equals the oracle's whole pipeline, including every level's outer-iteration count."""
    from paper_1503_05528_b200 import Config, inpaint
    from gen.synth import CONFIGS
    c = CONFIGS["c2"]
    v, m, _ = generate("c2")
    cfg = Config(levels=c.levels, pm_iters=c.pm_iters, max_outer=c.max_outer, lam=c.lam, seed=c.seed)
    out, stats, _ = inpaint(v, m, cfg)
    ref, st = orc.inpaint(v.numpy(), m.numpy(), c.levels, pm_iters=c.pm_iters, max_outer=c.max_outer,
                          lam=c.lam, seed=c.seed)
    assert [l["outer"] for l in stats.levels] == st["outer_iters"]
    # per level (onion in L); R41: evaluated = the oracle's count minus the stale candidates skipped
    assert [l["stale_skipped"] for l in stats.levels] == st["stale"]
    assert [l["patch_updates"] for l in stats.levels] == [a - b for a, b in zip(st["patch_updates"], st["stale"])]
    assert np.array_equal(out.cpu().numpy(), ref)


def test_cuda_graph_replay_equals_eager(orc):
    """Config.graphs: the first run captures each (level, outer iteration) body, the second run
    replays the graphs; both equal the eager driver (video, counts, stopping statistics)."""
    from paper_1503_05528_b200 import Config, Inpainter
    from gen.synth import CONFIGS
    c = CONFIGS["c2"]
    v, m, _ = generate("c2")
    T, H, W, _ = v.shape
    res = []
    for graphs in (False, True):
        ip = Inpainter(W, H, T, Config(levels=c.levels, pm_iters=c.pm_iters, max_outer=c.max_outer, lam=c.lam,
                                       seed=c.seed, graphs=graphs), "cuda")
        for _ in range(2 if graphs else 1):
            ip.load(v.cuda(), m.cuda())
            st = ip.run(timing=False)
            res.append((ip.output(v.cuda()).cpu(), [dict(d) for d in st.levels], st.total_patch_updates,
                        st.total_stale_skipped))
        if graphs:
            assert len(ip._graphs) == sum(d["outer"] for d in st.levels)
            assert ip.graph_launches > 0
    ref = res[0]
    for r in res[1:]:
        assert torch.equal(r[0], ref[0])
        assert [d["outer"] for d in r[1]] == [d["outer"] for d in ref[1]]
        assert [d["change_fixed"] for d in r[1]] == [d["change_fixed"] for d in ref[1]]
        assert r[2:] == ref[2:]
