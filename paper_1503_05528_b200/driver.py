"""Alg. 4 driver over the libvinp C ABI, with the optional Alg. 2 realignment and the
final unwarp (NEXT #1, `Config(align=True)`).

Host logic only: which kernel runs on which level, the onion-peel loop (Alg. 3), the stopping
rule (R19) and, under torch.distributed, the target-slab partition and the exchanges between
passes.  Every arithmetic step runs in libvinp's kernels.

Multi-GPU: every rank holds the full pyramid; the sorted target list (and hole list) of a level is
cut into W contiguous equal-count slabs.  After every pass that a later pass reads, each rank
receives the NNF rows (entries and R41 stamps) its next pass reads: by default only those rows,
point to point (`exchange="halo"`, NEXT #4 first stage), or every slab (`exchange="allgather"`).
After reconstruction the fp32 hole values are exchanged the same way and committed; the change e
is an exact int64 all-reduce.  Levels with fewer than `replicate_below` targets (the coarse ones)
and the onion peel run replicated on every rank, with no exchange, and are counted once.  Because
every pass is a Jacobi pass whose candidates are drawn from counter-based Philox streams keyed on
the voxel, the result is bit-identical for any number of ranks.
"""
from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import vinp as V


@dataclass
class Config:
    levels: int = 4
    pm_iters: int = 10          # PatchMatch iterations per ANN search
    fixed_outer: int = 0        # >0: exactly this many outer iterations per level (c1)
    max_outer: int = 20
    lam: int = 50
    seed: int = 1
    steps: Sequence[int] = (8, 4, 2, 1)  # jump-flood steps per PM iteration (R6)
    sign_policy: int = 0        # 0: Alg. 1 alternation (R5); 1: both directions every pass (R6)
    rho: float = 0.5
    tex_half: int = -1          # R15
    onion: bool = True          # Alg. 3 initialisation at the coarsest level
    align: bool = False         # NEXT #1: Alg. 2 realignment before, unwarp after
    align_levels: int = 3       # R36: estimation pyramid levels
    align_iters: int = 20       # R38: IRLS iterations per level
    align_tol: float = 1e-4     # R38: update-norm stop
    # multi-GPU: "halo" (NEXT #4: the rows a rank reads, P2P), "allgather", or "fused" (NEXT #4
    # second stage: the pass kernels store their slab into every rank's NNF copy themselves, through
    # peer pointers / an NVLS multicast address of symmetric-memory buffers; one barrier per pass)
    exchange: str = "halo"
    # multi-GPU: a level with fewer targets than this runs replicated on every rank (no exchange;
    # its work counted once): a coarse level split W ways is launch- and exchange-bound
    replicate_below: int = 1 << 21
    # per-level stage dumps (.npy, rank 0): after the onion peel and after each level's outer loop,
    # the NNF (entries, n), the hole values (fp32) and the level's u8 voxel words; None = off
    dump_dir: Optional[str] = None
    # single GPU: each outer iteration's fixed launch sequence (copy of the hole values, the ANN
    # search, the weighted reconstruction, the change) is captured once per (level, iteration) as a
    # CUDA graph and replayed on later runs over same-sized buffers
    graphs: bool = True
    stop_rule: int = 0          # 0: R19 e = ||u_H - v_H||_1 / (3|H|); 1: literal P:988 ||.||_2 / (3|H|)
    skip_stale: bool = True     # R41: exact skip of stale propagation candidates (NNF unchanged)
    lower_bound: bool = True    # R42: exact patch-sum lower-bound rejection in random search (NNF unchanged)
    # R41 diagnostics: count the stale candidates skipped (Stats.total_stale_skipped; equal to the
    # oracle's stale count).  False (not with the fused exchange): the R41-active passes first flag the targets that
    # read a changed entry and only those generate candidates (vinp_level.active): same NNF and
    # patch-update counts, faster, but the skipped candidates are never enumerated (count reported 0).
    # Default from VINP_COUNT_STALE (the test suite sets it to 1).
    count_stale: bool = field(default_factory=lambda: os.environ.get("VINP_COUNT_STALE", "0") == "1")

    def params(self) -> V.Params:
        return V.Params(lam=self.lam, tex_half=self.tex_half, seed=self.seed, rho=self.rho)


def stop_now(e_fixed: int, n_holes: int, k: int, max_outer: int, stop_rule: int = 0) -> bool:
    """Alg. 4 P:979-988 loop exit after outer iteration k (e <= 0.1, at most 20
    iterations).  e_fixed = the change statistic x 2^20 (exact integer, python ints: no overflow).
    stop_rule 0 (R19): e = e_fixed / 2^20 / (3|H|); 1 (literal P:988): e = sqrt(e_fixed / 2^20) / (3|H|)."""
    if k >= max_outer:
        return True
    if stop_rule == 0:
        return 10 * e_fixed <= 3 * n_holes * (1 << 20)
    return 100 * e_fixed <= 9 * n_holes * n_holes * (1 << 20)


class Exchange:
    """Slab partition + collectives.  World size 1: identity."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist if (dist.is_available() and dist.is_initialized()) else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0

    def padded(self, n: int) -> int:
        return -(-max(n, 1) // self.world) * self.world

    def slab(self, n: int):
        c = self.padded(n) // self.world
        return min(n, self.rank * c), min(n, (self.rank + 1) * c)

    def gather(self, t: torch.Tensor, n: int):
        """All-gather the rank slabs of the first padded(n) rows of t, in place."""
        if self.world == 1:
            return
        c = self.padded(n) // self.world
        mine = t[self.rank * c:(self.rank + 1) * c].clone()
        self.dist.all_gather_into_tensor(t[:self.world * c], mine, group=self.group)

    def allreduce_sum(self, t: torch.Tensor):
        if self.world > 1:
            self.dist.all_reduce(t, group=self.group)

    # ---- NEXT #4 second stage ("fused"): symmetric-memory NNF buffers written by every rank's kernels
    def alloc_nnf(self, key, npad: int, device, n=None, stamp=True):
        """An NNF buffer whose e (and n, stamp) live in symmetric memory, peer-mapped on every rank."""
        import torch.distributed._symmetric_memory as sm
        gname = (self.group or self.dist.group.WORLD).group_name
        self._sym = getattr(self, "_sym", {})

        def sym(dtype):
            t = sm.empty(npad, dtype=dtype, device=device)
            return t, sm.rendezvous(t, gname)

        e, he = sym(torch.int64)
        nn, hn = (n, self._sym.get(("n", key[0]))) if n is not None else sym(torch.uint8)
        st, hs = sym(torch.uint8) if stamp else (None, None)
        self._sym[key] = (he, hn, hs)
        self._sym[("n", key[0])] = hn
        self._barrier_handle = he
        return V.NNF(e, nn, st, key=key)

    def mirror(self, key):
        """The peer copies of buffer `key` for the pass kernels' epilogues."""
        he, hn, hs = self._sym[key]
        peers = [r for r in range(self.world) if r != self.rank]
        mc = int(he.multicast_ptr) if getattr(he, "has_multicast_support", lambda: False)() else 0
        return V.Mirror(e=[] if mc else [int(he.buffer_ptrs[r]) for r in peers],
                        n=[int(hn.buffer_ptrs[r]) for r in peers] if hn is not None else [],
                        stamp=[int(hs.buffer_ptrs[r]) for r in peers] if hs is not None else [],
                        mc_e=mc)

    def pass_barrier(self):
        """After a fused pass: every rank's stores are visible before any rank reads (device-side
        barrier on the current stream)."""
        self._barrier_handle.barrier(channel=0)

    def slabs(self, n: int):
        c = self.padded(n) // self.world
        return [(min(n, r * c), min(n, (r + 1) * c)) for r in range(self.world)]

    def halo(self, t: torch.Tensor, n: int, need):
        """Point-to-point halo exchange (NEXT #4): need[r] = (lo, hi), the rows rank r reads.  Every
        rank sends the part of its slab that each other rank needs and receives the parts of the
        other slabs it needs; all ranks derive the same ranges, so sends and receives pair up."""
        if self.world == 1:
            return
        sl = self.slabs(n)
        me = self.rank
        b, e = sl[me]
        ops = []
        for r in range(self.world):
            if r == me:
                continue
            lo, hi = need[r]
            s0, s1 = max(b, lo), min(e, hi)
            if s1 > s0:
                ops.append(self.dist.P2POp(self.dist.isend, t[s0:s1], r, self.group))
            rb, re_ = sl[r]
            lo2, hi2 = need[me]
            r0, r1 = max(rb, lo2), min(re_, hi2)
            if r1 > r0:
                ops.append(self.dist.P2POp(self.dist.irecv, t[r0:r1], r, self.group))
        if ops:
            for q in self.dist.batch_isend_irecv(ops):
                q.wait()


@dataclass
class LevelState:
    lv: V.Level
    a: V.NNF
    b: V.NNF
    cur_rgb: torch.Tensor
    cur_tex: torch.Tensor
    prev_rgb: torch.Tensor
    prev_tex: torch.Tensor
    outer: int = 0
    ms: float = 0.0
    patch_updates: int = 0


@dataclass
class Stats:
    levels: List[dict] = field(default_factory=list)
    onion_layers: int = 0
    setup_ms: float = 0.0
    total_ms: float = 0.0
    onion_ms: float = 0.0

    total_patch_updates: int = 0   # evaluated candidates (patch-updates)
    total_stale_skipped: int = 0   # R41 stale propagation candidates skipped (not patch-updates)

    @property
    def patch_updates(self):
        return self.total_patch_updates


class Inpainter:
    """Holds the pyramid of one video in HBM and runs Alg. 4 on it."""

    def __init__(self, W: int, H: int, T: int, cfg: Config, device="cuda", exchange: Exchange = None,
                 ops=None):
        """ops: the kernel module (default: the libvinp binding).  Tests substitute an oracle-backed
        module with the same call signatures to exercise the multi-rank logic on CPU (gloo)."""
        self.V = ops or V
        self.W, self.H, self.T, self.cfg = W, H, T, cfg
        self.device = torch.device(device)
        self.ex = exchange or Exchange()
        self.prm = cfg.params()
        self.levels: List[V.Level] = []
        for l, (w, h, _) in enumerate(V.level_dims(W, H, T, cfg.levels), start=1):
            self.levels.append(V.Level.alloc(w, h, T, l, self.device))
            if cfg.lower_bound and self.device.type == "cuda":  # 16 B per voxel (R42)
                self.levels[-1].psum = torch.empty((w * h * T, 8), dtype=torch.int16, device=self.device)
        n1 = W * H * T
        self.ws = torch.empty(max(self.V.texture_ws_bytes(self.levels[0]), self.V.sets_ws_bytes(self.levels[0])) + 256,
                              dtype=torch.uint8, device=self.device)
        # [0] patch-updates (evaluated candidates), [1] stale candidates skipped (R41)
        self.counter = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.change = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.states: List[LevelState] = []
        self.stats = Stats()
        self.n_layers = 0
        self.native = True  # False: every pass through its own C-ABI call (per-launch timing)
        self.native_onion = False  # True: Alg. 3 through vinp_onion_peel even when native is False
        self._graphs = {}  # (level, outer iteration) -> (torch.cuda.CUDAGraph, libvinp kernels in it)
        self.graph_launches = 0

    # ------------------------------------------------------------------ setup (a1-a3)
    def load(self, rgb: torch.Tensor, mask: torch.Tensor):
        """rgb u8 [T,H,W,3], mask u8 [T,H,W] (0 known, 2 invalid X after realignment, other
        nonzero = occluded), on this device."""
        assert rgb.shape == (self.T, self.H, self.W, 3) and mask.shape == (self.T, self.H, self.W)
        rgb = rgb.contiguous()
        mask = mask.contiguous()
        self.V.build_pyramid(rgb, mask, self.levels)
        self.V.texture_features(self.prm, self.levels, self.ws)
        for lv in self.levels:
            if lv.psum is not None:
                self.V.patch_sums(lv, 0)  # every voxel once (D~ never changes); targets: at each evaluate
        counts = self.V.build_sets(self.levels, self.ws)
        for lv in self.levels:
            if lv.n_sources == 0:
                raise V.VinpError(f"D~ is empty at level {lv.level} (S:237)")
            lv.alloc_lists()
            if (not self.cfg.count_stale and self.cfg.skip_stale and self.device.type == "cuda"
                    and (self.ex.world == 1 or self.cfg.exchange != "fused")):
                nw = self.V.active_ws_bytes(lv) // 4
                if lv.active is None or lv.active.numel() != nw:
                    lv.active = torch.empty(nw, dtype=torch.int32, device=self.device)
                lv.active.zero_()
            else:
                lv.active = None
        self.V.build_lists(self.levels, self.ws)
        old = {id(st.lv): st for st in self.states}
        self.states = []
        reused = 0
        for lv in self.levels:
            # >= 1 row so that an empty H (nothing to inpaint) still passes valid device pointers
            npad = max(self.ex.padded(lv.n_targets), 1)
            hpad = max(self.ex.padded(lv.n_holes), 1)
            st = old.get(id(lv))
            if st is not None and st.a.e.numel() == npad and st.cur_rgb.shape[0] == hpad:
                self.states.append(st)  # same sizes: reuse the buffers (repeated calls)
                reused += 1
                continue
            # every NNF entry / hole value is written (init, upsample, evaluate, reconstruct)
            # before it is read, so no zero fill is needed
            li = lv.level - 1
            if self.cfg.exchange == "fused" and self.ex.world > 1:
                a = self.ex.alloc_nnf((li, 0), npad, self.device, stamp=self.cfg.skip_stale)
                b = self.ex.alloc_nnf((li, 1), npad, self.device, n=a.n, stamp=self.cfg.skip_stale)
            else:
                a = V.NNF.alloc(npad, self.device, zero=False, stamp=self.cfg.skip_stale)
                b = V.NNF.alloc(npad, self.device, n=a.n, zero=False, stamp=self.cfg.skip_stale)
            a.key, b.key = (li, 0), (li, 1)
            z = lambda k: torch.empty((hpad, k), dtype=torch.float32, device=self.device)
            self.states.append(LevelState(lv, a, b, z(3), z(2), z(3), z(2)))
        if reused != len(self.levels):
            self._graphs = {}  # captured graphs hold the old buffers' addresses
        self.fused = self.cfg.exchange == "fused" and self.ex.world > 1
        self.halo = self.cfg.exchange in ("halo", "fused") and self.ex.world > 1
        if self.halo:
            self._halo_ranges()
        top = self.levels[-1]
        if top.layer is None:
            top.layer = torch.empty(top.N, dtype=torch.uint8, device=self.device)
        self.n_layers = self.V.layers(top, self.ws)
        self.stats.onion_layers = self.n_layers
        return counts

    def _halo_ranges(self):
        """Per level and rank: the NNF rows (targets within max(step) frames of the rank's target slab,
        or within 2 frames of its hole slab) and the hole rows (within 2 frames of its target slab)
        the rank reads.  Targets and holes are sorted t-major, so each is one contiguous range."""
        smax = max(max(self.cfg.steps), 2)
        for st in self.states:
            lv = st.lv
            hw = lv.W * lv.H
            tf = (lv.targets[:lv.n_targets].cpu().to(torch.int64) // hw)
            hf = (lv.holes[:lv.n_holes].cpu().to(torch.int64) // hw)

            def rng(frames, f0, f1):
                lo = int(torch.searchsorted(frames, torch.tensor(f0), right=False))
                hi = int(torch.searchsorted(frames, torch.tensor(f1), right=True))
                return lo, hi

            nnf, hole = [], []
            for (b, e), (hb, he) in zip(self.ex.slabs(lv.n_targets), self.ex.slabs(lv.n_holes)):
                lo, hi = (0, 0)
                hlo, hhi = (0, 0)
                if e > b:
                    f0, f1 = int(tf[b]), int(tf[e - 1])
                    lo, hi = rng(tf, f0 - smax, f1 + smax)
                    hlo, hhi = rng(hf, f0 - 2, f1 + 2)
                if he > hb:
                    g0, g1 = int(hf[hb]), int(hf[he - 1])
                    l2, h2 = rng(tf, g0 - 2, g1 + 2)
                    lo, hi = (l2, h2) if hi <= lo else (min(lo, l2), max(hi, h2))
                nnf.append((lo, hi))
                hole.append((hlo, hhi))
            st.halo_nnf, st.halo_hole = nnf, hole

    # ------------------------------------------------------------------ ANN search (a5-a8)
    def ann_search(self, st: LevelState, outer_code: int, kb=-1, only_layer=-1, replicated=False):
        lv, prm, cfg = st.lv, self.prm, self.cfg
        n = lv.n_targets
        if self.native and (replicated or self.ex.world == 1):  # Alg. 1 in one native call
            self.V.ann_search(lv, st.a, st.b, prm, outer_code, cfg.pm_iters, tuple(cfg.steps), kb, only_layer,
                              self.counter, sign_policy=cfg.sign_policy)
            return
        b, e = self.ex.slab(n)
        if replicated:
            gather1 = lambda t: None  # noqa: E731
        elif self.halo:
            gather1 = lambda t: self.ex.halo(t, n, st.halo_nnf)  # noqa: E731
        else:
            gather1 = lambda t: self.ex.gather(t, n)  # noqa: E731

        def gather(f):  # an NNF buffer: entries, and the R41 stamps the next pass reads
            gather1(f.e)
            if f.stamp is not None:
                gather1(f.stamp)

        use = st.a.stamp is not None and cfg.pm_iters * (len(cfg.steps) + 1) <= 255
        a_nnf, b_nnf = (st.a, st.b) if use else (V.NNF(st.a.e, st.a.n, key=st.a.key),
                                                 V.NNF(st.b.e, st.b.n, key=st.b.key))
        fused = self.fused and not replicated

        def out(f):  # the buffer a pass writes: with the fused exchange, also every peer's copy
            f.mirror = self.ex.mirror(f.key) if fused else None
            if fused and f.stamp is None:
                f.mirror.stamp = []
            return f

        def published(f):  # make the pass's output readable by the next pass on every rank
            if fused:
                self.ex.pass_barrier()
            else:
                gather(f)

        if fused:  # evaluate rewrites every rank's copy of `a`: no rank may still be reading it
            self.ex.pass_barrier()
        self.V.nnf_evaluate(lv, out(a_nnf), prm, kb, only_layer, b, e, self.counter)
        published(a_nnf)
        if not fused:
            gather1(a_nnf.n)
        clk = V.PassClock()
        for k in range(1, cfg.pm_iters + 1):
            sign = 0 if cfg.sign_policy else (1 if k % 2 == 1 else -1)
            for s in cfg.steps:
                self.V.propagate(lv, a_nnf, out(b_nnf), prm, s, sign, kb, only_layer, b, e, self.counter,
                                 pass_id=clk.pass_id, since=clk.since(s, sign))
                clk.tick(s, sign)
                a_nnf, b_nnf = b_nnf, a_nnf
                st.a, st.b = st.b, st.a
                published(a_nnf)
            self.V.random_search(lv, a_nnf, out(b_nnf), prm, outer_code, k, kb, only_layer, b, e, self.counter,
                                 pass_id=clk.pass_id)
            clk.tick()
            a_nnf, b_nnf = b_nnf, a_nnf
            st.a, st.b = st.b, st.a
            published(a_nnf)
        a_nnf.mirror = b_nnf.mirror = None

    def reconstruct(self, st: LevelState, mode: int, layer_j=-1, replicated=False, full=False):
        lv = st.lv
        n = lv.n_holes
        hb, he = (0, n) if replicated else self.ex.slab(n)
        self.V.reconstruct(lv, st.a, mode, st.cur_rgb, st.cur_tex, layer_j, hb, he, commit=True)
        if not replicated and self.ex.world > 1:
            if self.halo and not full:
                # only the hole values this rank's target patches read (holes outside that range
                # are never read here: sources lie in D~, which excludes H)
                self.ex.halo(st.cur_rgb, n, st.halo_hole)
                self.ex.halo(st.cur_tex, n, st.halo_hole)
                lo, hi = st.halo_hole[self.ex.rank]
                self.V.commit(lv, st.cur_rgb, st.cur_tex, layer_j, lo, hi)
            else:
                self.ex.gather(st.cur_rgb, n)
                self.ex.gather(st.cur_tex, n)
                self.V.commit(lv, st.cur_rgb, st.cur_tex, layer_j, 0, n)

    def _outer_body(self, st: LevelState, k: int, rp: bool):
        """One outer iteration of Alg. 4 up to the change e: v <- u_H, ANN search,
        weighted reconstruction, e (device scalar self.change)."""
        lv, cfg = st.lv, self.cfg
        st.prev_rgb.copy_(st.cur_rgb)
        st.prev_tex.copy_(st.cur_tex)
        self.ann_search(st, k, replicated=rp)
        self.reconstruct(st, V.WEIGHTED, replicated=rp)
        self.change.zero_()
        hb, he = (0, lv.n_holes) if rp else self.ex.slab(lv.n_holes)
        chg = self.V.change_l2 if cfg.stop_rule == 1 else self.V.change_l1
        chg(st.cur_rgb[hb:he], st.prev_rgb[hb:he], self.change)
        if not rp:
            self.ex.allreduce_sum(self.change)

    def _outer_iteration(self, l: int, st: LevelState, k: int, rp: bool):
        """The outer-iteration body, eagerly or as a CUDA graph (single GPU, native passes): the
        first run of each (level, k) captures it, later runs over the same buffers replay it."""
        use = (self.cfg.graphs and self.native and self.ex.world == 1 and self.device.type == "cuda"
               and self.V is V)
        if not use:
            return self._outer_body(st, k, rp)
        g = self._graphs.get((l, k))
        if g is None:
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            n0 = V.launch_count()
            with torch.cuda.graph(g):
                self._outer_body(st, k, rp)
            self._graphs[(l, k)] = (g, V.launch_count() - n0)
            g = self._graphs[(l, k)]
        g[0].replay()
        self.graph_launches += g[1]  # libvinp kernels this replay ran (the library counts launches, not replays)

    def _dump(self, tag: str, st: LevelState):
        """Stage dump (Config.dump_dir): `<tag>_{nnf_e,nnf_n,holes,hole_rgb,hole_tex,vox}.npy`."""
        import os
        import numpy as np
        if self.ex.rank != 0:
            return
        lv = st.lv
        nt, nh = lv.n_targets, lv.n_holes
        os.makedirs(self.cfg.dump_dir, exist_ok=True)
        arrs = dict(nnf_e=st.a.e[:nt], nnf_n=st.a.n[:nt], targets=lv.targets[:nt], holes=lv.holes[:nh],
                    hole_rgb=st.cur_rgb[:nh], hole_tex=st.cur_tex[:nh], vox=lv.vox)
        for k, t in arrs.items():
            np.save(os.path.join(self.cfg.dump_dir, f"{tag}_{k}.npy"), t.cpu().numpy())

    def replicated(self, l: int) -> bool:
        """Level l runs replicated on every rank (multi-GPU only): fewer than replicate_below targets."""
        return self.ex.world > 1 and self.states[l - 1].lv.n_targets < self.cfg.replicate_below

    # ------------------------------------------------------------------ Alg. 3 onion peel
    def onion_peel(self):
        """Alg. 3, replicated on every rank: one native call (per-layer index lists, all passes)."""
        st = self.states[-1]
        self.V.nnf_init_random(st.lv, st.a, self.prm, 0)  # phi^L <- Random
        self.V.onion_peel(st.lv, st.a, st.b, self.prm, self.cfg.pm_iters, self.n_layers, st.cur_rgb,
                          st.cur_tex, tuple(self.cfg.steps), self.counter, sign_policy=self.cfg.sign_policy)

    def onion_peel_stepwise(self):
        """The same Alg. 3 through the per-pass C-ABI calls (only_layer filter); reference path."""
        st = self.states[-1]
        self.V.nnf_init_random(st.lv, st.a, self.prm, 0)
        for j in range(0, self.n_layers + 1):
            kb = max(j, 1)
            self.ann_search(st, V.ONION | j, kb=kb, only_layer=j, replicated=True)
            if j >= 1:
                self.reconstruct(st, V.WEIGHTED, layer_j=j, replicated=True)

    # ------------------------------------------------------------------ Alg. 4
    def run(self, timing=True) -> Stats:
        cfg = self.cfg
        L = cfg.levels
        cuda = self.device.type == "cuda"
        timing = timing and cuda

        class _NoEv:
            def record(self):
                pass

        ev = (lambda: torch.cuda.Event(enable_timing=True)) if cuda else (lambda: _NoEv())
        self.stats.levels = [dict(level=l, outer=0, patch_updates=0, ms=0.0) for l in range(1, L + 1)]
        t_all0 = ev(); t_all0.record()
        marks = {}
        self.counter.zero_()
        e0 = ev(); e0.record()
        if cfg.onion:
            self.onion_peel() if (self.native or self.native_onion) else self.onion_peel_stepwise()
        else:
            st = self.states[-1]
            self.V.nnf_init_random(st.lv, st.a, self.prm, 0)
        e_on = ev(); e_on.record()
        if cfg.dump_dir:
            self._dump("onion", self.states[-1])
        onion_pu = self.counter.clone()  # replicated work: counted once (rank 0) in the job total
        snaps = {}  # counter after each level (device tensors: no extra host syncs)
        repl = {l: self.replicated(l) for l in range(1, L + 1)}
        for l in range(L, 0, -1):
            st = self.states[l - 1]
            lv = st.lv
            rp = repl[l]
            k = 0
            changes = []
            while True:
                self._outer_iteration(l, st, k, rp)
                k += 1
                if cfg.fixed_outer > 0:
                    changes.append(self.change.clone())  # read once at the end (no sync here)
                    if k >= cfg.fixed_outer:
                        break
                else:
                    e_fixed = int(self.change.item())  # the one host sync per outer iteration
                    changes.append(e_fixed)
                    if stop_now(e_fixed, lv.n_holes, k, cfg.max_outer, cfg.stop_rule):
                        break
            self.stats.levels[l - 1]["change_fixed"] = changes
            if cfg.dump_dir:
                self._dump(f"level{l}", st)
            if l == 1:
                self.reconstruct(st, V.BEST_PATCH, full=True, replicated=rp)  # Eq. 6; every rank gets u
            else:
                if self.halo and not rp:  # upsampling reads the coarse NNF of any frame of the fine slab
                    self.ex.gather(st.a.e, lv.n_targets)
                    self.ex.gather(st.a.n, lv.n_targets)
                f = self.states[l - 2]
                frp = repl[l - 1]
                fb, fe = (0, f.lv.n_targets) if frp else self.ex.slab(f.lv.n_targets)
                self.V.nnf_upsample(lv, st.a, f.lv, f.a, self.prm, fb, fe)
                if not frp:
                    self.ex.gather(f.a.e, f.lv.n_targets)
                    self.ex.gather(f.a.n, f.lv.n_targets)
                self.reconstruct(f, V.UNWEIGHTED, replicated=frp)  # R20
            e1 = ev(); e1.record()
            marks[l] = (e0, e1)
            snaps[l] = self.counter.clone()
            self.stats.levels[l - 1]["outer"] = k
            e0 = e1
        t_all1 = ev(); t_all1.record()
        if timing:
            torch.cuda.synchronize()
            for l, (a, b) in marks.items():  # noqa: B007
                self.stats.levels[l - 1]["ms"] = a.elapsed_time(b)
            self.stats.total_ms = t_all0.elapsed_time(t_all1)
            self.stats.onion_ms = t_all0.elapsed_time(e_on)
        # per-level patch-update counts (the coarsest level includes the onion peel, counted once
        # in the job total: the replicated onion work is subtracted on ranks other than 0)
        prev = torch.zeros_like(self.counter)
        per = []
        for l in range(L, 0, -1):
            per.append(snaps[l] - prev)
            prev = snaps[l]
        per = torch.stack(per)  # [level (coarsest first), (evaluated, stale)]
        if self.ex.rank != 0:  # replicated work (onion peel, replicated levels) counted by rank 0 only
            per[0] -= onion_pu
            for i, l in enumerate(range(L, 0, -1)):
                if repl[l]:
                    per[i] = 0
        self.ex.allreduce_sum(per)
        per = per.tolist()
        for d in self.stats.levels:  # the stopping statistic of every outer iteration (x 2^20)
            d["change_fixed"] = [int(c) for c in d.get("change_fixed", [])]
        for i, l in enumerate(range(L, 0, -1)):
            self.stats.levels[l - 1]["patch_updates"] = int(per[i][0])
            self.stats.levels[l - 1]["stale_skipped"] = int(per[i][1])
        self.stats.total_patch_updates = int(sum(x[0] for x in per))
        self.stats.total_stale_skipped = int(sum(x[1] for x in per))
        return self.stats

    def output(self, rgb_in: torch.Tensor) -> torch.Tensor:
        """Final video: input outside H, the best-patch u8 values inside H (device tensor)."""
        lv = self.levels[0]
        if hasattr(self.V, "output_rgb"):  # the colour bytes of vox are exactly that video
            return self.V.output_rgb(lv)
        vb = lv.vox.view(torch.uint8).view(self.T, self.H, self.W, 8)[..., :3]
        m = (lv.flags.view(self.T, self.H, self.W) & 1).bool()
        return torch.where(m[..., None], vb, rgb_in)

    # ------------------------------------------------------------------ NEXT #1 (Alg. 2)
    def align(self, rgb: torch.Tensor, mask: torch.Tensor):
        """Alg. 2: theta_{n,n+1} by robust IRLS, the chain to the middle frame, bilinear warp of
        the video and its occlusion (mask codes 0 / 1 / 2 = invalid, R40).  Device tensors."""
        c = self.cfg
        npairs = self.T - 1
        if getattr(self, "_align_ws", None) is None:
            self._align_ws = torch.empty(max(self.V.affine_ws_bytes(self.W, self.H, self.T, c.align_levels), 1),
                                         dtype=torch.uint8, device=self.device)
            self._align_out = (torch.empty_like(rgb), torch.empty_like(mask))
            k = self.ex.padded(max(npairs, 1))
            self._align_est = (torch.empty((k, 6), dtype=torch.float64, device=self.device),
                               torch.zeros(k, dtype=torch.int32, device=self.device),
                               torch.zeros(k, dtype=torch.int32, device=self.device))
        # the frame pairs are independent: each rank estimates its slab, then an all-gather
        pairs = self.ex.slab(npairs) if npairs > 0 else (0, 0)
        self.V.affine_estimate(rgb, mask, c.align_levels, c.align_iters, c.align_tol, ws=self._align_ws,
                               out=self._align_est, pairs=pairs)
        if npairs > 0:
            for t in self._align_est:
                self.ex.gather(t, npairs)
        theta, status, iters = (t[:npairs] for t in self._align_est)
        fwd, inv, err = self.V.affine_chain(theta, self.T)
        self.align_info = dict(theta=theta, status=status, iters=iters, fwd=fwd, inv=inv, err=err)
        return self.V.align_warp(rgb, mask, inv, out=self._align_out)

    def unwarp(self, aligned_out: torch.Tensor, rgb: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
        """Inverse warp of the inpainted aligned video, pasted into the original occlusion (R40)."""
        return self.V.unwarp(aligned_out, rgb, mask, self.align_info["fwd"])


_PLANS = {}


def inpaint(rgb: torch.Tensor, mask: torch.Tensor, cfg: Config, device="cuda", exchange=None, ops=None):
    """Convenience: whole Alg. 4 on one video.  rgb/mask may live on the host (copied in; pinned
    host memory makes the copy asynchronous).  The device buffers of an Inpainter are cached per
    (shape, config, device, exchange), so repeated calls on same-shaped videos allocate nothing."""
    T, H, W, _ = rgb.shape
    key = (W, H, T, repr(cfg), str(torch.device(device)), id(exchange), id(ops))
    ip = _PLANS.get(key)
    if ip is None:
        ip = _PLANS[key] = Inpainter(W, H, T, cfg, device, exchange, ops)
    if rgb.dtype != torch.uint8 or tuple(rgb.shape[3:]) != (3,) or tuple(mask.shape) != (T, H, W):
        raise ValueError("inpaint: rgb must be u8 [T, H, W, 3] and mask [T, H, W]")
    rgb_d = rgb.to(device, non_blocking=True).contiguous()
    mask_d = mask.to(device, dtype=torch.uint8, non_blocking=True).contiguous()
    if cfg.align:
        a_rgb, a_mask = ip.align(rgb_d, mask_d)
        ip.load(a_rgb, a_mask)
        stats = ip.run()
        return ip.unwarp(ip.output(a_rgb), rgb_d, mask_d), stats, ip
    ip.load(rgb_d, mask_d)
    stats = ip.run()
    return ip.output(rgb_d), stats, ip
