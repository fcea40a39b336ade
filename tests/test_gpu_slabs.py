"""The §8(e) slab path on the GPU (VERDICT r01 "Next round" 3).

1. Every pass of the hot path called on target (hole) slabs [b, e) -- 2, 3 and 8 slabs, in an
   arbitrary order -- writes exactly what the full-range call writes (NNF words, n, counts, fp32
   hole values), so a rank's slab call is the full call restricted to its slab.
2. W ranks emulated on one GPU: W Inpainters on cuda:0, one Python thread each, joined by an
   in-process exchange with the driver's collective semantics (all-gather of equal-count slabs,
   halo point-to-point ranges, int64 all-reduce) implemented by host barriers and device copies.
   No kernel waits on another rank's kernel; every exchange is a host-synchronised copy, so this is
   a correctness emulation, not a timing.  The result must be bit-identical to world size 1 for
   both exchange modes (and with coarse levels replicated).
"""
import threading

import numpy as np
import pytest
import torch

from gen.synth import CONFIGS, generate, random_volume

pytestmark = pytest.mark.gpu


def _split(n, k, seed=0):
    """k slabs covering [0, n), uneven, returned in a shuffled order."""
    if n == 0:
        return []
    rng = np.random.default_rng(seed + k)
    cuts = sorted(set([0, n] + list(rng.integers(1, max(2, n), k - 1))))
    sl = [(int(a), int(b)) for a, b in zip(cuts[:-1], cuts[1:])]
    rng.shuffle(sl)
    return sl


@pytest.fixture(scope="module")
def state():
    """c2 at the first outer iteration of level 1 (onion peel, one outer iteration at level 2,
    upsample + unweighted reconstruction), as Alg. 4 gets there."""
    from paper_1503_05528_b200 import Config, Inpainter, vinp as V
    c = CONFIGS["c2"]
    v, m, _ = generate("c2", device="cuda")
    ip = Inpainter(c.W, c.H, c.T, Config(levels=2, lam=c.lam, seed=c.seed), "cuda")
    ip.load(v, m)
    ip.onion_peel()
    s2, s1 = ip.states[1], ip.states[0]
    ip.ann_search(s2, 0)
    ip.reconstruct(s2, V.WEIGHTED)
    torch.cuda.synchronize()
    return ip


def _nnf_clone(V, x):
    return V.NNF(x.e.clone(), x.n.clone())


@pytest.mark.parametrize("k", [2, 3, 8])
def test_passes_on_slabs_equal_full_range(state, k):
    from paper_1503_05528_b200 import vinp as V
    ip = state
    prm = ip.prm
    s2, s1 = ip.states[1], ip.states[0]
    lv = s1.lv
    n = lv.n_targets
    slabs = _split(n, k)
    cnt_f = torch.zeros(1, dtype=torch.int64, device="cuda")
    cnt_s = torch.zeros(1, dtype=torch.int64, device="cuda")

    def same(x, y, what):
        assert torch.equal(x.e[:n], y.e[:n]), what
        assert torch.equal(x.n[:n], y.n[:n]), what

    # upsample (level 2 -> 1) on fine-target slabs
    full = V.NNF.alloc(s1.a.e.numel(), "cuda")
    part = V.NNF.alloc(s1.a.e.numel(), "cuda")
    V.nnf_upsample(s2.lv, s2.a, lv, full, prm)
    for b, e in slabs:
        V.nnf_upsample(s2.lv, s2.a, lv, part, prm, b, e)
    same(full, part, "upsample")
    # evaluate
    V.nnf_evaluate(lv, full, prm, counter=cnt_f)
    for b, e in slabs:
        V.nnf_evaluate(lv, part, prm, b=b, e=e, counter=cnt_s)
    same(full, part, "evaluate")
    # propagation (both alternating signs and the 'both' policy) and random search
    cur = full
    for step, sign in ((8, 1), (2, -1), (1, 0), (4, 1)):
        out_f = V.NNF.alloc(cur.e.numel(), "cuda", n=cur.n)
        out_s = V.NNF.alloc(cur.e.numel(), "cuda", n=cur.n)
        V.propagate(lv, cur, out_f, prm, step, sign, counter=cnt_f)
        for b, e in slabs:
            V.propagate(lv, cur, out_s, prm, step, sign, b=b, e=e, counter=cnt_s)
        same(out_f, out_s, f"propagate s={step} sign={sign}")
        cur = out_f
    for it in (1, 2):
        out_f = V.NNF.alloc(cur.e.numel(), "cuda", n=cur.n)
        out_s = V.NNF.alloc(cur.e.numel(), "cuda", n=cur.n)
        V.random_search(lv, cur, out_f, prm, 0, it, counter=cnt_f)
        for b, e in slabs:
            V.random_search(lv, cur, out_s, prm, 0, it, b=b, e=e, counter=cnt_s)
        same(out_f, out_s, f"random search k={it}")
        cur = out_f
    assert int(cnt_f) == int(cnt_s) > 0
    # reconstruction in all three modes on hole slabs (no commit: the working copy stays as is)
    nh = lv.n_holes
    hs = _split(nh, k, seed=5)
    for mode in (V.WEIGHTED, V.UNWEIGHTED, V.BEST_PATCH):
        rf = torch.full((nh, 3), -1.0, device="cuda")
        tf = torch.full((nh, 2), -1.0, device="cuda")
        rs, ts = rf.clone(), tf.clone()
        V.reconstruct(lv, cur, mode, rf, tf, commit=False)
        for hb, he in hs:
            V.reconstruct(lv, cur, mode, rs, ts, hb=hb, he=he, commit=False)
        assert torch.equal(rf, rs) and torch.equal(tf, ts), mode
        assert (rf >= 0).all()
    # random init on slabs
    V.nnf_init_random(lv, full, prm, 7)
    for b, e in slabs:
        V.nnf_init_random(lv, part, prm, 7, b, e)
    assert torch.equal(full.e[:n], part.e[:n])


# ----------------------------------------------------------------------------- W-rank emulation
class _Hub:
    """Shared state of the emulated process group."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world, timeout=600)
        self.box = [None] * world
        self.nnf = [dict() for _ in range(world)]  # fused exchange: each rank's NNF buffers by key
        self.error = None

    def sync(self):
        torch.cuda.synchronize()
        self.bar.wait()


def _emulated_exchange(hub, rank):
    from paper_1503_05528_b200.driver import Exchange

    class EmuExchange(Exchange):
        def __init__(self):
            self.dist = None
            self.group = None
            self.world = hub.world
            self.rank = rank
            self.gathers = 0
            self.halos = 0
            self.barriers = 0

        # NEXT #4 second stage: the "symmetric" buffers are plain device tensors of the emulated
        # ranks (one GPU), the peers' copies are their tensors, the barrier is a host barrier
        def alloc_nnf(self, key, npad, device, n=None, stamp=True):
            from paper_1503_05528_b200 import vinp as V
            f = V.NNF.alloc(npad, device, n=n, zero=False, stamp=stamp)
            f.key = key
            hub.nnf[rank][key] = f
            return f

        def mirror(self, key):
            from paper_1503_05528_b200 import vinp as V
            peers = [hub.nnf[r][key] for r in range(hub.world) if r != rank]
            return V.Mirror(e=[f.e for f in peers], n=[f.n for f in peers],
                            stamp=[f.stamp for f in peers if f.stamp is not None])

        def pass_barrier(self):
            hub.sync()
            self.barriers += 1

        def gather(self, t, n):
            c = self.padded(n) // self.world
            hub.box[rank] = t
            hub.sync()
            for r in range(self.world):
                if r != rank:
                    t[r * c:(r + 1) * c].copy_(hub.box[r][r * c:(r + 1) * c])
            hub.sync()
            self.gathers += 1

        def allreduce_sum(self, t):
            hub.box[rank] = t.clone()
            hub.sync()
            tot = sum(b.to(torch.int64) for b in hub.box).to(t.dtype)
            hub.sync()
            t.copy_(tot)

        def halo(self, t, n, need):
            sl = self.slabs(n)
            hub.box[rank] = t
            hub.sync()
            lo, hi = need[rank]
            for r in range(self.world):
                if r == rank:
                    continue
                rb, re_ = sl[r]
                r0, r1 = max(rb, lo), min(re_, hi)
                if r1 > r0:
                    t[r0:r1].copy_(hub.box[r][r0:r1])
            hub.sync()
            self.halos += 1

    return EmuExchange()


def _run_world(v, m, cfg, world):
    from paper_1503_05528_b200 import Inpainter
    T, H, W, _ = v.shape
    hub = _Hub(world)
    res = [None] * world

    def body(rank):
        try:
            ex = _emulated_exchange(hub, rank) if world > 1 else None
            ip = Inpainter(W, H, T, cfg, "cuda", exchange=ex)
            ip.load(v, m)
            st = ip.run()
            out = ip.output(v).clone()
            torch.cuda.synchronize()
            res[rank] = (out, [dict(d) for d in st.levels], st.total_patch_updates,
                         getattr(ex, "gathers", 0), getattr(ex, "halos", 0), getattr(ex, "barriers", 0))
        except BaseException as exc:  # surface the first failure, release the others
            hub.error = hub.error or exc
            hub.bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if hub.error is not None:
        raise hub.error
    return res


CASES = {
    "c2": lambda: generate("c2", device="cuda")[:2],
    "odd": lambda: tuple(x.cuda() for x in random_volume(47, 33, 26, seed=9, hole_frac=0.06)[:2]),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("exchange", ["allgather", "halo"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_bit_identical_to_one(case, exchange, world):
    from paper_1503_05528_b200 import Config
    v, m = CASES[case]()
    L = 2 if case == "c2" else 3
    cfg1 = Config(levels=L, exchange=exchange, replicate_below=0)  # every level in slabs
    ref = _run_world(v, m, cfg1, 1)[0]
    got = _run_world(v, m, cfg1, world)
    for rank, (out, lev, pu, ng, nh, nb) in enumerate(got):
        assert torch.equal(out, ref[0]), (rank, "output video")
        assert [d["outer"] for d in lev] == [d["outer"] for d in ref[1]], rank
        assert [d["patch_updates"] for d in lev] == [d["patch_updates"] for d in ref[1]], rank
        assert pu == ref[2]
        assert (nh > 0) if exchange == "halo" else (ng > 0)


@pytest.mark.parametrize("world", [2, 4])
def test_emulated_ranks_replicated_coarse_level(world):
    """c2 with the coarse level (63,900 targets) replicated and level 1 (212,700) in slabs"""
    from paper_1503_05528_b200 import Config
    v, m = CASES["c2"]()
    cfg = Config(levels=2, exchange="halo", replicate_below=100_000)
    ref = _run_world(v, m, Config(levels=2), 1)[0]
    for rank, (out, lev, pu, ng, nh, nb) in enumerate(_run_world(v, m, cfg, world)):
        assert torch.equal(out, ref[0]), (rank, "output video")
        assert [d["outer"] for d in lev] == [d["outer"] for d in ref[1]], rank
        assert [d["patch_updates"] for d in lev] == [d["patch_updates"] for d in ref[1]], rank
        assert pu == ref[2] and nh > 0


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_fused_exchange(case, world):
    """NEXT #4 second stage: every pass kernel stores its slab into all emulated ranks' NNF copies
    (vinp_mirror peer pointers), a barrier per pass, no NNF collective: bit-identical to one rank"""
    from paper_1503_05528_b200 import Config
    v, m = CASES[case]()
    L = 2 if case == "c2" else 3
    ref = _run_world(v, m, Config(levels=L), 1)[0]
    got = _run_world(v, m, Config(levels=L, exchange="fused", replicate_below=0), world)
    for rank, (out, lev, pu, ng, nh, nb) in enumerate(got):
        assert torch.equal(out, ref[0]), (rank, "output video")
        assert [d["outer"] for d in lev] == [d["outer"] for d in ref[1]], rank
        assert [d["patch_updates"] for d in lev] == [d["patch_updates"] for d in ref[1]], rank
        assert [d["stale_skipped"] for d in lev] == [d["stale_skipped"] for d in ref[1]], rank
        assert pu == ref[2] and nb > 0


@pytest.mark.parametrize("exchange,world", [("halo", 2), ("halo", 4), ("allgather", 3)])
def test_emulated_ranks_listed_target_passes(exchange, world):
    """The product default (Config.count_stale = False: R41-active passes over the listed targets
    only, per slab) under emulated ranks, against one rank in the counting mode: same output video,
    outer iterations and patch-update counts (the stale count is not reported in this mode)."""
    from paper_1503_05528_b200 import Config
    v, m = CASES["c2"]()
    ref = _run_world(v, m, Config(levels=2, count_stale=True), 1)[0]
    got = _run_world(v, m, Config(levels=2, exchange=exchange, replicate_below=0, count_stale=False), world)
    for rank, (out, lev, pu, ng, nh, nb) in enumerate(got):
        assert torch.equal(out, ref[0]), (rank, "output video")
        assert [d["outer"] for d in lev] == [d["outer"] for d in ref[1]], rank
        assert [d["patch_updates"] for d in lev] == [d["patch_updates"] for d in ref[1]], rank
        assert pu == ref[2]
