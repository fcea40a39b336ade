"""The product default of the R41-active propagation passes (`vinp_level.active`, Config.count_stale
= False): targets that read no changed entry generate no candidates.  Must give the same NNF,
stamps and patch-update counts as the exhaustive passes, and whole inpaintings equal to the oracle's.
"""
import numpy as np
import pytest
import torch

from gen.synth import generate, random_volume

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    from paper_1503_05528_b200 import vinp
    return vinp


def _loaded(case, **kw):
    from paper_1503_05528_b200 import Config, Inpainter
    if case == "c2":
        v, m, _ = generate("c2")
    else:
        v, m, _ = random_volume(45, 37, 11, seed=7, hole_frac=0.06)
    T, H, W, _ = v.shape
    ip = Inpainter(W, H, T, Config(levels=2, **kw), "cuda")
    ip.load(v.cuda(), m.cuda())
    return ip


@pytest.mark.parametrize("case,sign_policy,slabs", [("c2", 0, 1), ("c2", 1, 1), ("odd", 0, 1), ("odd", 1, 1),
                                                    ("c2", 0, 3), ("odd", 1, 2)])
def test_flagged_passes_equal_exhaustive_passes(V, case, sign_policy, slabs):
    """One ANN search pass by pass on two copies of the state, with and without `active`; with
    slabs > 1 the flagged pass runs slab by slab (the multi-GPU call pattern: stamps of the whole
    level current, entries copied and targets listed per slab)."""
    ip = _loaded(case, count_stale=False)
    for st in ip.states:
        lv = st.lv
        assert lv.active is not None and int(lv.active.abs().sum()) == 0
        n = lv.n_targets
        V.nnf_init_random(lv, st.a, ip.prm, 4)
        V.nnf_evaluate(lv, st.a, ip.prm)
        bufs = {}
        for mode in ("flag", "all"):
            a = V.NNF.alloc(n, "cuda", stamp=True)
            b = V.NNF.alloc(n, "cuda", n=a.n, stamp=True)
            a.e.copy_(st.a.e[:max(n, 1)])
            a.n.copy_(st.a.n[:max(n, 1)])
            bufs[mode] = [a, b, torch.zeros(2, dtype=torch.int64, device="cuda"), V.PassClock()]
        act = lv.active
        flagged_passes = 0
        for k in range(1, 7):
            signs = (0,) if sign_policy else ((1,) if k % 2 else (-1,))
            for s in (8, 4, 2, 1):
                for sign in signs:
                    for mode in ("flag", "all"):
                        a, b, cnt, clk = bufs[mode]
                        lv.active = act if mode == "flag" else None
                        nsl = slabs if mode == "flag" else 1
                        for i in range(nsl):
                            V.propagate(lv, a, b, ip.prm, s, sign, counter=cnt, pass_id=clk.pass_id,
                                        since=clk.since(s, sign), b=i * n // nsl, e=(i + 1) * n // nsl)
                        flagged_passes += mode == "flag" and clk.since(s, sign) > 0
                        clk.tick(s, sign)
                        bufs[mode][0], bufs[mode][1] = b, a
                    lv.active = act
                    assert torch.equal(bufs["flag"][0].e[:n], bufs["all"][0].e[:n]), (k, s, sign)
                    assert torch.equal(bufs["flag"][0].stamp[:n], bufs["all"][0].stamp[:n]), (k, s, sign)
                    assert int(bufs["flag"][2][0]) == int(bufs["all"][2][0]), (k, s, sign)
                    assert int(act[8:8 + (n + 31) // 32].abs().sum()) == 0  # bitmap cleared by the pass that used it
            for mode in ("flag", "all"):
                a, b, cnt, clk = bufs[mode]
                V.random_search(lv, a, b, ip.prm, 4, k, counter=cnt, pass_id=clk.pass_id)
                clk.tick()
                bufs[mode][0], bufs[mode][1] = b, a
        assert flagged_passes > 0
        assert int(bufs["flag"][2][1]) < int(bufs["all"][2][1])  # the flagged passes do not count stale ones


@pytest.mark.parametrize("case", ["c1", "c2", "rand"])
def test_default_mode_inpainting_equals_oracle(orc, case):
    from paper_1503_05528_b200 import Config, inpaint
    if case == "c1":
        (v, m, _), kw, okw, L = generate("c1"), dict(pm_iters=4, fixed_outer=3), dict(pm_iters=4, fixed_outer=3), 1
    elif case == "c2":
        (v, m, _), kw, okw, L = generate("c2"), {}, {}, 2
    else:
        (v, m, _), kw, okw, L = random_volume(61, 45, 12, seed=33, hole_frac=0.07), {}, {}, 3
    out, stats, _ = inpaint(v, m, Config(levels=L, count_stale=False, **kw), device="cuda")
    ref, st = orc.inpaint(v.numpy(), m.numpy(), L, **okw)
    assert np.array_equal(out.cpu().numpy(), ref)
    assert [l["patch_updates"] for l in stats.levels] == [a - b for a, b in zip(st["patch_updates"], st["stale"])]
    assert [l["outer"] for l in stats.levels] == st["outer_iters"]
    assert stats.total_stale_skipped < sum(st["stale"])


def test_default_mode_equals_counting_mode_on_c3():
    """A larger run (c3, 3 levels): output video and patch-update counts of the two modes."""
    from paper_1503_05528_b200 import Config, inpaint
    v, m, _ = generate("c3", frames=40)
    res = []
    for cs in (False, True):
        out, stats, _ = inpaint(v, m, Config(levels=3, count_stale=cs, max_outer=3), device="cuda")
        res.append((out.cpu(), [l["patch_updates"] for l in stats.levels], [l["outer"] for l in stats.levels]))
    assert torch.equal(res[0][0], res[1][0])
    assert res[0][1:] == res[1][1:]


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_full_size_modes_agree(name):
    """BASELINE's full-size configs, whole Alg. 4: the product default (listed targets, R42 lower
    bound) against the exhaustive counting mode without the lower bound — the mode the full-size
    oracle parity test (tests/test_gpu_fullsize_e2e.py) runs c4 in.  Output video, outer iterations
    and patch-update counts per level must be equal."""
    from gen.synth import CONFIGS
    from paper_1503_05528_b200 import Config, Inpainter
    c = CONFIGS[name]
    v, m, _ = generate(name, device="cuda")
    res = []
    for fast in (True, False):
        cfg = Config(levels=c.levels, pm_iters=c.pm_iters, fixed_outer=c.fixed_outer, max_outer=c.max_outer,
                     lam=c.lam, seed=c.seed, count_stale=not fast, lower_bound=fast)
        ip = Inpainter(c.W, c.H, c.T, cfg, "cuda")
        ip.load(v, m)
        st = ip.run()
        res.append((ip.output(v).clone(), [l["patch_updates"] for l in st.levels], [l["outer"] for l in st.levels]))
        del ip
        torch.cuda.empty_cache()
    assert torch.equal(res[0][0], res[1][0])
    assert res[0][1:] == res[1][1:]
