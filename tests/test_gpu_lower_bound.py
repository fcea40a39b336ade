"""R42: the patch-sum lower bound of random search (include/vinp.h `vinp_patch_sums`).

The sums are checked against box sums computed with torch; the bound against the distances of
`vinp_patch_ssd`; and every result with the bound (NNF, patch-update counts, whole inpaintings) must
equal the result without it, which the other parity tests compare with the oracle.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from gen.synth import generate, random_volume

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    from paper_1503_05528_b200 import vinp
    return vinp


def _loaded(case, lower_bound=True):
    from paper_1503_05528_b200 import Config, Inpainter
    if case == "c2":
        v, m, _ = generate("c2")
        levels = 2
    else:
        v, m, _ = random_volume(45, 37, 11, seed=7, hole_frac=0.06)
        levels = 2
    T, H, W, _ = v.shape
    ip = Inpainter(W, H, T, Config(levels=levels, lower_bound=lower_bound), "cuda")
    ip.load(v.cuda(), m.cuda())
    return ip


def _box_sums(lv):
    """int64 [N, 5]: sums of R, G, B, Tx, Ty over the 5x5x5 patch (zero padding), by torch."""
    vox = lv.vox.view(1, 1, lv.T, lv.H, lv.W)
    out = []
    for sh in (0, 8, 16, 32, 40):
        ch = ((vox >> sh) & 255).double()
        out.append((F.avg_pool3d(ch, 5, stride=1, padding=2, count_include_pad=True) * 125.0).round().long().view(-1))
    return torch.stack(out, 1)


def _interior(lv):
    t, y, x = torch.meshgrid(torch.arange(lv.T), torch.arange(lv.H), torch.arange(lv.W), indexing="ij")
    ok = (x >= 2) & (x < lv.W - 2) & (y >= 2) & (y < lv.H - 2) & (t >= 2) & (t < lv.T - 2)
    return ok.reshape(-1).cuda()


@pytest.mark.parametrize("case", ["c2", "odd"])
def test_patch_sums_equal_box_sums(V, case):
    ip = _loaded(case)
    for lv in ip.levels:
        ref = _box_sums(lv)
        ins = _interior(lv)
        got = lv.psum.view(-1, 8).long() & 0xFFFF
        assert torch.equal(got[ins][:, :5], ref[ins])
        assert int(got[:, 5:].abs().sum()) == 0
        assert int(got[~ins].abs().sum()) == 0
    # after u changes in the hole, evaluate refreshes the targets' sums
    st = ip.states[0]
    lv = st.lv
    holes = lv.holes[:lv.n_holes].long()
    g = torch.Generator(device="cuda").manual_seed(3)
    lv.vox[holes] = torch.randint(0, 256, (holes.numel(),), device="cuda", generator=g) * 0x010101 + \
        (torch.randint(0, 256, (holes.numel(),), device="cuda", generator=g) << 32)
    V.nnf_init_random(lv, st.a, ip.prm, 5)
    V.nnf_evaluate(lv, st.a, ip.prm)
    ref = _box_sums(lv)
    tg = lv.targets[:lv.n_targets].long()
    tg = tg[_interior(lv)[tg]]
    got = lv.psum.view(-1, 8).long() & 0xFFFF
    assert torch.equal(got[tg][:, :5], ref[tg])


@pytest.mark.parametrize("case", ["c2", "odd"])
def test_bound_never_exceeds_distance(V, case):
    ip = _loaded(case)
    lv = ip.states[0].lv
    V.nnf_init_random(lv, ip.states[0].a, ip.prm, 5)
    V.nnf_evaluate(lv, ip.states[0].a, ip.prm)
    g = torch.Generator(device="cuda").manual_seed(11)
    tg = lv.targets[:lv.n_targets].long()
    tg = tg[_interior(lv)[tg]]
    src = lv.sources[:lv.n_sources].long()
    n = 200000
    p = tg[torch.randint(0, tg.numel(), (n,), device="cuda", generator=g)]
    q = src[torch.randint(0, src.numel(), (n,), device="cuda", generator=g)]
    # half of the pairs close to each other (small distances, where a wrong bound would show)
    near = p[: n // 2] + torch.randint(-3, 4, (n // 2,), device="cuda", generator=g)
    flags = lv.flags
    near = torch.where((near >= 0) & (near < lv.N) & ((flags[near.clamp(0, lv.N - 1)] & 2) != 0), near, q[: n // 2])
    q = torch.cat([near, q[n // 2:]])
    D, cnt = V.patch_ssd(lv, p.int(), q.int(), ip.prm)
    assert int(cnt.min()) == 125
    s = lv.psum.view(-1, 8).long() & 0xFFFF
    d = s[p] - s[q]
    lam = ip.prm.lam
    lhs = 4 * (d[:, :3] ** 2).sum(1) + lam * (d[:, 3:5] ** 2).sum(1)
    assert bool((lhs <= 125 * D.long()).all())
    assert int((lhs > 0).sum()) > n // 2  # the bound is not vacuous


@pytest.mark.parametrize("case", ["c2", "odd"])
def test_random_search_with_bound_equals_without(V, case):
    ip = _loaded(case)
    rejected_any = False
    for st in ip.states:
        lv = st.lv
        V.nnf_init_random(lv, st.a, ip.prm, 9)
        V.ann_search(lv, st.a, st.b, ip.prm, 9, 2)  # a partly converged NNF
        res = []
        for use in (True, False):
            ps = lv.psum
            if not use:
                lv.psum = None
            out = V.NNF.alloc(lv.n_targets, "cuda", stamp=st.a.stamp is not None)
            cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
            V.random_search(lv, st.a, out, ip.prm, 9, 3, counter=cnt)
            torch.cuda.synchronize()
            res.append((out.e[:lv.n_targets].clone(), int(cnt[0])))
            lv.psum = ps
        assert torch.equal(res[0][0], res[1][0])
        assert res[0][1] == res[1][1] > 0
        rejected_any = True
    assert rejected_any


def test_inpaint_with_bound_equals_without():
    from paper_1503_05528_b200 import Config, inpaint
    v, m, _ = random_volume(61, 45, 12, seed=21, hole_frac=0.07)
    outs = []
    for lb in (True, False):
        out, stats, _ = inpaint(v, m, Config(levels=2, lower_bound=lb), device="cuda")
        outs.append((out.cpu(), stats.total_patch_updates, stats.total_stale_skipped))
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][1:] == outs[1][1:]


def test_patch_sums_argument_errors(V):
    ip = _loaded("odd", lower_bound=False)
    lv = ip.levels[0]
    assert lv.psum is None
    with pytest.raises(V.VinpError):
        V.patch_sums(lv, 0)
    lv.psum = torch.empty((lv.N, 8), dtype=torch.int16, device="cuda")
    with pytest.raises(V.VinpError):
        V.patch_sums(lv, 2)
    with pytest.raises(V.VinpError):
        V.patch_sums(lv, 1, 0, lv.n_targets + 1)
    V.patch_sums(lv, 0)
    V.patch_sums(lv, 1)
    lv.psum = None
