"""World-size-2 run of the multi-GPU driver logic on CPU (gloo): target/hole slabs, NNF and hole
all-gathers after every pass, exact int64 all-reduce of the stopping-rule change.  The compute is
the CPU oracle behind the libvinp signatures (tests/oracle_ops.py).  The result must be
bit-identical to a single-rank run and to the oracle's own whole-pipeline or_inpaint (SURVEY §8(e):
the schedule is partition-independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen.synth import random_volume

# replicate_below=0: every level split into slabs (these volumes are far below the default
# threshold, which would run them replicated)
CFG = dict(levels=2, pm_iters=2, max_outer=3, replicate_below=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _vol(T):
    return random_volume(40, 32, T, seed=4, hole_frac=0.06)


def _run(rank, world, port, out_path, T=10, exchange="allgather"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_ops
        from paper_1503_05528_b200 import Config, Exchange, inpaint
        v, m, _ = _vol(T)
        out, stats, ip = inpaint(v, m, Config(exchange=exchange, **CFG), device="cpu", exchange=Exchange(),
                                 ops=oracle_ops)
        if rank == 0:
            np.save(out_path, out.numpy())
            np.save(out_path + ".stats.npy", np.array([l["outer"] for l in stats.levels] +
                                                      [stats.total_patch_updates]))
    finally:
        dist.destroy_process_group()


def _spawn(world, tmp_path, T=10, exchange="allgather"):
    out = str(tmp_path / f"out_w{world}_{T}_{exchange}.npy")
    mp.spawn(_run, args=(world, _free_port(), out, T, exchange), nprocs=world, join=True)
    return np.load(out), np.load(out + ".stats.npy")


def test_two_ranks_bit_identical_to_one_and_to_oracle(tmp_path, orc):
    import oracle_ops  # noqa: F401  (importable from tests/)
    o1, s1 = _spawn(1, tmp_path)
    o2, s2 = _spawn(2, tmp_path)
    assert np.array_equal(o1, o2)
    assert np.array_equal(s1, s2)
    v, m, _ = random_volume(40, 32, 10, seed=4, hole_frac=0.06)
    ref, st = orc.inpaint(v.numpy(), m.numpy(), CFG["levels"], pm_iters=CFG["pm_iters"],
                          max_outer=CFG["max_outer"])
    assert np.array_equal(o1, ref)
    assert list(s1[:-1]) == st["outer_iters"] and int(s1[-1]) == sum(st["patch_updates"])


def test_exchange_slabs_cover_and_pad():
    from paper_1503_05528_b200.driver import Exchange
    ex = Exchange()
    ex.world = 3
    spans = []
    for r in range(3):
        ex.rank = r
        spans.append(ex.slab(10))
    assert ex.padded(10) == 12 and spans == [(0, 4), (4, 8), (8, 10)]
    ex.rank = 2
    assert ex.slab(0) == (0, 0)


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_bit_identical(tmp_path, orc, world):
    """NEXT #4 halo exchange: with 36 frames the slabs are ~12-18 frames, so every rank receives
    only part of the other slabs (+-8 frames of NNF, +-2 frames of hole values); the result must
    still equal the single-rank run and the oracle bit for bit."""
    T = 36
    o1, s1 = _spawn(1, tmp_path, T)
    oh, sh = _spawn(world, tmp_path, T, "halo")
    assert np.array_equal(o1, oh) and np.array_equal(s1, sh)
    v, m, _ = _vol(T)
    ref, st = orc.inpaint(v.numpy(), m.numpy(), CFG["levels"], pm_iters=CFG["pm_iters"],
                          max_outer=CFG["max_outer"])
    assert np.array_equal(o1, ref)


def test_halo_ranges_are_partial():
    """the halo really is partial for the test geometry (the exchange is exercised)"""
    import torch
    from paper_1503_05528_b200 import Config
    from paper_1503_05528_b200.driver import Exchange, Inpainter
    import oracle_ops
    v, m, _ = _vol(36)
    ex = Exchange()
    ex.world, ex.rank = 3, 0
    ip = Inpainter(40, 32, 36, Config(exchange="halo", **CFG), "cpu", ex, oracle_ops)
    ip.load(v, m)
    st = ip.states[0]
    n = st.lv.n_targets
    spans = [hi - lo for lo, hi in st.halo_nnf]
    assert all(sp > 0 for sp in spans) and sum(sp < n for sp in spans) >= 2, (spans, n)


def _run_aligned(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_ops
        from paper_1503_05528_b200 import Config, Exchange, inpaint
        v, m = _aligned_video()
        out, stats, ip = inpaint(v, m, Config(align=True, **CFG), device="cpu", exchange=Exchange(), ops=oracle_ops)
        if rank == 0:
            np.save(out_path, out.numpy())
            np.save(out_path + ".theta.npy", ip.align_info["theta"].numpy())
    finally:
        dist.destroy_process_group()


def _aligned_video():
    from gen.synth import camera_video
    T = 9
    cams = [np.array([1.5 * t, 1, 0, -0.5 * t, 0, 1]) for t in range(T)]
    v = camera_video(48, 40, T, 6, cams, noise=1.0)
    m = torch.zeros((T, 40, 48), dtype=torch.uint8)
    m[:, 15:23, 20:28] = 1
    v[m.bool()] = 0
    return v, m


def test_aligned_two_ranks_split_pairs(tmp_path, orc):
    """realignment under torch.distributed: each rank estimates its slab of the frame pairs and the
    estimates are all-gathered; the result equals the oracle's align -> inpaint -> unwarp"""
    out = str(tmp_path / "aligned_w2.npy")
    mp.spawn(_run_aligned, args=(2, _free_port(), out), nprocs=2, join=True)
    v, m = _aligned_video()
    ar, am, fwd, inv, pairs, st = orc.align_pipeline(v.numpy(), m.numpy())
    assert np.array_equal(np.load(out + ".theta.npy"), pairs)
    o, _ = orc.inpaint(ar, am, CFG["levels"], pm_iters=CFG["pm_iters"], max_outer=CFG["max_outer"])
    assert np.array_equal(np.load(out), orc.unwarp(o, v.numpy(), m.numpy(), fwd))


def _run_cfg(rank, world, port, out_path, spec):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_ops
        from gen.synth import random_holes
        from paper_1503_05528_b200 import Config, Exchange, inpaint
        W, H, T, seed, levels, steps, exchange = spec[:7]
        rb = spec[7] if len(spec) > 7 else 0
        v, _, _ = random_volume(W, H, T, seed=seed)
        m = random_holes(W, H, T, seed, 2)
        v[m.bool()] = 0
        cfg = Config(levels=levels, pm_iters=2, max_outer=2, steps=steps, exchange=exchange, replicate_below=rb)
        out, stats, _ = inpaint(v, m, cfg, device="cpu", exchange=Exchange(), ops=oracle_ops)
        if rank == 0:
            np.save(out_path, out.numpy())
            np.save(out_path + ".stats.npy", np.array([l["outer"] for l in stats.levels] +
                                                      [l["patch_updates"] for l in stats.levels]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,T,seed,levels,steps", [
    (2, 36, 28, 30, 11, 2, (8, 4, 2, 1)),
    (3, 30, 24, 41, 12, 1, (16, 8, 4, 2, 1)),
    (4, 28, 24, 44, 13, 2, (4, 2, 1)),
])
def test_halo_fuzz_equals_single_rank(tmp_path, world, W, H, T, seed, levels, steps):
    """random hole shapes, frame counts, level counts and step schedules (max step 16 widens the
    halo): the halo exchange at world sizes 2-4 equals the single-rank run, per-level counts too"""
    outs = []
    for wsz, ex in ((1, "allgather"), (world, "halo")):
        out = str(tmp_path / f"fz_{wsz}_{ex}.npy")
        mp.spawn(_run_cfg, args=(wsz, _free_port(), out, (W, H, T, seed, levels, steps, ex)), nprocs=wsz,
                 join=True)
        outs.append((np.load(out), np.load(out + ".stats.npy")))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("exchange", ["halo", "allgather"])
def test_replicated_coarse_levels_equal_single_rank(tmp_path, exchange):
    """levels below the target-count threshold run replicated (no exchange, counted once), the
    finer ones in slabs: world 3 equals world 1 (video, outer counts, per-level patch-updates)"""
    W, H, T, seed, levels, steps = 44, 36, 30, 21, 3, (8, 4, 2, 1)
    from gen.synth import random_holes
    from oracle.oracle import sets
    m = random_holes(W, H, T, seed, 2)
    # threshold = the level-1 target count: level 1 is not below it (slabs), levels 2-3 are (replicated)
    rb = int(sets(np.ascontiguousarray(m.numpy()))[1].sum())
    outs = []
    for wsz in (1, 3):
        out = str(tmp_path / f"rp_{wsz}_{exchange}.npy")
        mp.spawn(_run_cfg, args=(wsz, _free_port(), out, (W, H, T, seed, levels, steps, exchange, rb)),
                 nprocs=wsz, join=True)
        outs.append((np.load(out), np.load(out + ".stats.npy")))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def test_stage_dumps(tmp_path):
    """Config.dump_dir writes the per-level stage arrays; the last one is the final level-1 state"""
    import oracle_ops
    from paper_1503_05528_b200 import Config, Inpainter
    v, m, _ = _vol(8)
    T, H, W, _ = v.shape
    d = str(tmp_path / "dump")
    ip = Inpainter(W, H, T, Config(levels=2, pm_iters=2, max_outer=2, dump_dir=d), "cpu", ops=oracle_ops)
    ip.load(v, m)
    ip.run(timing=False)
    names = sorted(os.listdir(d))
    for tag in ("onion", "level2", "level1"):
        for k in ("nnf_e", "nnf_n", "targets", "holes", "hole_rgb", "hole_tex", "vox"):
            assert f"{tag}_{k}.npy" in names
    st = ip.states[0]
    nt = st.lv.n_targets
    e = np.load(os.path.join(d, "level1_nnf_e.npy"))
    assert np.array_equal(e, st.a.e[:nt].numpy())  # level 1 dumped before best-patch, after its loop
    assert np.load(os.path.join(d, "level1_hole_rgb.npy")).shape == (st.lv.n_holes, 3)


def _cpu_emulated_world(v, m, cfg, world):
    """W ranks as threads in one process (CPU, oracle ops): the exchanges through shared tensors and
    a host barrier, the fused exchange's peer copies are the other ranks' tensors."""
    import threading
    import oracle_ops
    from paper_1503_05528_b200 import Exchange, Inpainter, vinp as V

    bar = threading.Barrier(world, timeout=600)
    box = [None] * world
    nnf = [dict() for _ in range(world)]
    res = [None] * world
    err = []

    class Emu(Exchange):
        def __init__(self, rank):
            self.dist, self.group, self.world, self.rank = None, None, world, rank
            self.barriers = 0

        def gather(self, t, n):
            c = self.padded(n) // self.world
            box[self.rank] = t
            bar.wait()
            for r in range(self.world):
                if r != self.rank:
                    t[r * c:(r + 1) * c].copy_(box[r][r * c:(r + 1) * c])
            bar.wait()

        def allreduce_sum(self, t):
            box[self.rank] = t.clone()
            bar.wait()
            tot = sum(b.to(torch.int64) for b in box).to(t.dtype)
            bar.wait()
            t.copy_(tot)

        def halo(self, t, n, need):
            sl = self.slabs(n)
            box[self.rank] = t
            bar.wait()
            lo, hi = need[self.rank]
            for r in range(self.world):
                if r != self.rank:
                    r0, r1 = max(sl[r][0], lo), min(sl[r][1], hi)
                    if r1 > r0:
                        t[r0:r1].copy_(box[r][r0:r1])
            bar.wait()

        def alloc_nnf(self, key, npad, device, n=None, stamp=True):
            f = V.NNF.alloc(npad, device, n=n, stamp=stamp)
            nnf[self.rank][key] = f
            return f

        def mirror(self, key):
            peers = [nnf[r][key] for r in range(self.world) if r != self.rank]
            return V.Mirror(e=[f.e for f in peers], n=[f.n for f in peers],
                            stamp=[f.stamp for f in peers if f.stamp is not None])

        def pass_barrier(self):
            bar.wait()
            self.barriers += 1

    def body(rank):
        try:
            ex = Emu(rank)
            T, H, W, _ = v.shape
            ip = Inpainter(W, H, T, cfg, "cpu", exchange=ex, ops=oracle_ops)
            ip.load(v, m)
            st = ip.run(timing=False)
            res[rank] = (ip.output(v).clone(), [d["outer"] for d in st.levels], st.total_patch_updates, ex.barriers)
        except BaseException as exc:  # release the others
            err.append(exc)
            bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_host_logic(world, orc):
    """NEXT #4 second stage, host logic on CPU: passes store their slab into every rank's copy
    (oracle ops honour vinp_mirror), one barrier before each evaluate and after each pass, no NNF
    collective: every rank's video equals the oracle's whole pipeline"""
    from paper_1503_05528_b200 import Config
    v, m, _ = _vol(10)
    cfg = Config(exchange="fused", **CFG)
    res = _cpu_emulated_world(v, m, cfg, world)
    ref, st = orc.inpaint(v.numpy(), m.numpy(), CFG["levels"], pm_iters=CFG["pm_iters"],
                          max_outer=CFG["max_outer"])
    for out, outer, pu, nb in res:
        assert np.array_equal(out.numpy(), ref)
        assert outer == st["outer_iters"] and pu == sum(st["patch_updates"]) and nb > 0
