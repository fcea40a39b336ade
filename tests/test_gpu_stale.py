"""R41 stale-candidate skip: GPU passes with change stamps vs the CPU oracle, which
evaluates every candidate and counts separately those whose neighbour proposes the same shift as
in the previous pass with the same (step, sign).  The NNF must be bit-identical to the unskipped
oracle pass, counter[0] + counter[1] the oracle's count, and counter[1] its stale count.
"""
import numpy as np
import pytest
import torch

import _bridge as B
from gen.synth import generate, random_volume

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    from paper_1503_05528_b200 import vinp
    return vinp


def _ip(case, levels):
    from paper_1503_05528_b200 import Config, Inpainter
    if case == "odd":
        v, m, _ = random_volume(45, 37, 11, seed=7, hole_frac=0.06)
    else:
        v, m, _ = generate(case)
    T, H, W, _ = v.shape
    ip = Inpainter(W, H, T, Config(levels=levels), "cuda")
    ip.load(v.cuda(), m.cuda())
    torch.cuda.synchronize()
    return ip


def _pair(V, lv):
    a = V.NNF.alloc(lv.n_targets, "cuda", stamp=True)
    b = V.NNF.alloc(lv.n_targets, "cuda", n=a.n, stamp=True)
    return a, b


def _search_both(V, orc, ip, lv, ol, a, b, f, K, sign_policy, kb=-1, j=-1, oc=3, b0=0, e0=None):
    """K PatchMatch iterations, pass by pass, GPU (stamps) vs oracle (prev snapshots)."""
    lam, seed = ip.prm.lam, ip.prm.seed
    e0 = lv.n_targets if e0 is None else e0
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    V.nnf_evaluate(lv, a, ip.prm, kb, j, counter=cnt)
    orc.evaluate(ol, f, lam, kb, j)
    assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0
    assert int(a.stamp[:lv.n_targets].max()) == 0
    clk = V.PassClock()
    snaps = {}
    tot_stale = 0
    for k in range(1, K + 1):
        sign = 0 if sign_policy else (1 if k % 2 else -1)
        for s in (8, 4, 2, 1):
            cnt.zero_()
            V.propagate(lv, a, b, ip.prm, s, sign, kb, j, counter=cnt, pass_id=clk.pass_id,
                        since=clk.since(s, sign))
            g = f.copy()
            stale = np.zeros(1, np.int64)
            c_o = orc.propagate(ol, f, g, lam, s, sign, kb, j, prev=snaps.get((s, sign)), stale=stale)
            assert len(B.nnf_equal(orc, lv, b.e, b.n, g)) == 0, (k, s, sign)
            assert int(cnt[1]) == int(stale[0]), (k, s, sign)
            assert int(cnt[0]) + int(cnt[1]) == c_o, (k, s, sign)
            # stamps: this pass's index exactly where the entry changed
            ch = (b.e[:lv.n_targets] != a.e[:lv.n_targets])
            assert torch.equal(b.stamp[:lv.n_targets] == clk.pass_id, ch)
            snaps[(s, sign)] = f
            clk.tick(s, sign)
            a, b, f = b, a, g
            tot_stale += int(stale[0])
        cnt.zero_()
        V.random_search(lv, a, b, ip.prm, oc, k, kb, j, counter=cnt, pass_id=clk.pass_id)
        g = f.copy()
        c_o = orc.random_search(ol, f, g, lam, seed, 0.5, lv.rmax, lv.level, oc, k, kb, j)
        assert len(B.nnf_equal(orc, lv, b.e, b.n, g)) == 0, (k, "rs")
        assert int(cnt[0]) == c_o and int(cnt[1]) == 0
        clk.tick()
        a, b, f = b, a, g
    return a, b, f, tot_stale


@pytest.mark.parametrize("case,sign_policy", [("c2", 0), ("c2", 1), ("odd", 0)])
def test_stale_skip_passes_bit_exact(V, orc, case, sign_policy):
    ip = _ip(case, 2 if case == "c2" else 3)
    lv = ip.levels[0]
    ol = B.oracle_level(orc, lv)
    a, b = _pair(V, lv)
    V.nnf_init_random(lv, a, ip.prm, 7)
    f = orc.NNF.empty(lv.n_targets)
    orc.init_random(ol, f, ip.prm.seed, lv.level, 7)
    _, _, _, st = _search_both(V, orc, ip, lv, ol, a, b, f, 6, sign_policy)
    assert st > 0  # the skip is exercised


def test_stale_skip_onion_restricted(V, orc):
    """The warp-per-target K-restricted kernels (onion layers) with stamps."""
    ip = _ip("c2", 2)
    lv = ip.levels[-1]
    ol = B.oracle_level(orc, lv, layers=True)
    a, b = _pair(V, lv)
    V.nnf_init_random(lv, a, ip.prm, 0)
    f = orc.NNF.empty(lv.n_targets)
    orc.init_random(ol, f, ip.prm.seed, lv.level, 0)
    tot = 0
    for j in (0, 1, 4):
        a, b, f, st = _search_both(V, orc, ip, lv, ol, a, b, f, 4, 0, kb=max(j, 1), j=j,
                                   oc=V.ONION | j)
        tot += st
    assert tot > 0


@pytest.mark.parametrize("case,sign_policy", [("c1", 0), ("c2", 1)])
def test_native_ann_search_with_stamps(V, orc, case, sign_policy):
    ip = _ip(case, 1 if case == "c1" else 2)
    lv = ip.levels[0]
    ol = B.oracle_level(orc, lv)
    a, b = _pair(V, lv)
    V.nnf_init_random(lv, a, ip.prm, 11)
    f = orc.NNF.empty(lv.n_targets)
    orc.init_random(ol, f, ip.prm.seed, lv.level, 11)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")
    V.ann_search(lv, a, b, ip.prm, 11, 10, counter=cnt, sign_policy=sign_policy)
    f, c_o, st_o = orc.ann_search(ol, f, ip.prm.lam, ip.prm.seed, lv.level, 11, 10,
                                  sign_policy=sign_policy, with_stale=True)
    assert len(B.nnf_equal(orc, lv, a.e, a.n, f)) == 0
    assert int(cnt[1]) == st_o > 0
    assert int(cnt[0]) + int(cnt[1]) == c_o


def test_stale_skip_on_slabs(V):
    """A stamped pass split into slabs [b, e) equals the full-range pass (entries, stamps, counts)."""
    ip = _ip("c2", 2)
    lv = ip.levels[0]
    n = lv.n_targets
    a, b = _pair(V, lv)
    V.nnf_init_random(lv, a, ip.prm, 5)
    V.ann_search(lv, a, b, ip.prm, 5, 2)  # a converged-ish NNF, stamps from its last pass
    V.nnf_evaluate(lv, a, ip.prm)
    clk = V.PassClock()
    for s in (8, 4, 2, 1):  # pass 1..4 with sign +1, then the same with sign -1 and +1 again
        V.propagate(lv, a, b, ip.prm, s, 1, pass_id=clk.pass_id, since=clk.since(s, 1))
        clk.tick(s, 1)
        a, b = b, a
    V.random_search(lv, a, b, ip.prm, 5, 1, pass_id=clk.pass_id)
    clk.tick()
    a, b = b, a
    ref = V.NNF(b.e.clone(), a.n, b.stamp.clone())
    c_full = torch.zeros(2, dtype=torch.int64, device="cuda")
    V.propagate(lv, a, ref, ip.prm, 4, 1, counter=c_full, pass_id=clk.pass_id, since=clk.since(4, 1))
    for parts in (2, 3, 8):
        out = V.NNF(b.e.clone(), a.n, b.stamp.clone())
        c = torch.zeros(2, dtype=torch.int64, device="cuda")
        cuts = [n * i // parts for i in range(parts + 1)]
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            V.propagate(lv, a, out, ip.prm, 4, 1, b=lo, e=hi, counter=c, pass_id=clk.pass_id,
                        since=clk.since(4, 1))
        assert torch.equal(out.e[:n], ref.e[:n]) and torch.equal(out.stamp[:n], ref.stamp[:n])
        assert torch.equal(c, c_full)
    assert int(c_full[1]) > 0


def test_stamp_argument_errors(V):
    ip = _ip("c1", 1)
    lv = ip.levels[0]
    a, b = _pair(V, lv)
    plain = V.NNF.alloc(lv.n_targets, "cuda", n=a.n)
    with pytest.raises(V.VinpError):
        V.propagate(lv, a, plain, ip.prm, 1, 1)  # stamps on one buffer only
    with pytest.raises(V.VinpError):
        V.propagate(lv, a, b, ip.prm, 1, 1, pass_id=0)
    with pytest.raises(V.VinpError):
        V.propagate(lv, a, b, ip.prm, 1, 1, pass_id=256)
    with pytest.raises(V.VinpError):
        V.propagate(lv, a, b, ip.prm, 1, 1, pass_id=3, since=3)
    with pytest.raises(V.VinpError):
        V.random_search(lv, a, V.NNF(b.e, b.n, a.stamp), ip.prm, 0, 1, pass_id=2)  # shared array
