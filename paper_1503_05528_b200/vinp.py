"""Thin ctypes binding of libvinp.so (include/vinp.h).  Argument marshalling only: every step of
the inpainting path runs in the library's sm_100a kernels.  Device memory is owned by torch
tensors; calls are enqueued on torch's current CUDA stream.

There is no fallback: if libvinp.so is missing or fails to load, import raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VINP_LIB_PATH") or os.path.join(HERE, "libvinp.so")  # override: A/B dev builds

WEIGHTED, UNWEIGHTED, BEST_PATCH = 0, 1, 2
ONION = 0x80000000  # outer_code marker for onion layer j: ONION | j


class VinpError(RuntimeError):
    pass


class _Level(C.Structure):
    _fields_ = [("W", C.c_int32), ("H", C.c_int32), ("T", C.c_int32), ("level", C.c_int32),
                ("vox", C.c_void_p), ("flags", C.c_void_p), ("layer", C.c_void_p),
                ("slot", C.c_void_p),
                ("targets", C.c_void_p), ("n_targets", C.c_int32),
                ("holes", C.c_void_p), ("n_holes", C.c_int32),
                ("sources", C.c_void_p), ("n_sources", C.c_int32),
                ("psum", C.c_void_p), ("active", C.c_void_p)]


MAX_PEERS = 7


class _Mirror(C.Structure):
    _fields_ = [("n_peers", C.c_int32), ("e", C.c_void_p * MAX_PEERS), ("n", C.c_void_p * MAX_PEERS),
                ("stamp", C.c_void_p * MAX_PEERS), ("mc_e", C.c_void_p)]


class _NNF(C.Structure):
    _fields_ = [("e", C.c_void_p), ("n", C.c_void_p), ("stamp", C.c_void_p), ("mirror", C.POINTER(_Mirror))]


class _Params(C.Structure):
    _fields_ = [("lambda_", C.c_int32), ("tex_half", C.c_int32), ("seed", C.c_uint64),
                ("rho", C.c_double), ("rmax", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise VinpError(f"{LIB_PATH} is missing: run `python -m paper_1503_05528_b200.build` "
                        "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, I, I32, I64, U32, U64 = C.c_void_p, C.c_int, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
    sigs = {
        "vinp_last_error": (C.c_char_p, []),
        "vinp_version": (I, []),
        "vinp_launch_count": (U64, []),
        "vinp_build_pyramid": (I, [P, P, P, I, P]),
        "vinp_texture_ws_bytes": (C.c_size_t, [P]),
        "vinp_texture_features": (I, [P, P, I, P, C.c_size_t, P]),
        "vinp_sets_ws_bytes": (C.c_size_t, [P]),
        "vinp_build_sets": (I, [P, I, P, P, C.c_size_t, P]),
        "vinp_build_lists": (I, [P, I, P, C.c_size_t, P]),
        "vinp_layers": (I, [P, P, P, P]),
        "vinp_nnf_init_random": (I, [P, P, P, U32, I32, I32, P]),
        "vinp_nnf_upsample": (I, [P, P, P, P, P, I32, I32, P]),
        "vinp_nnf_evaluate": (I, [P, P, P, I, I, I32, I32, P, P]),
        "vinp_propagate": (I, [P, P, P, P, I, I, I, I, I32, I32, I, I, P, P]),
        "vinp_random_search": (I, [P, P, P, P, U32, I, I, I, I32, I32, I, P, P]),
        "vinp_ann_search": (I, [P, P, P, P, U32, I, P, I, I, I, I, P, P]),
        "vinp_onion_ws_bytes": (C.c_size_t, [P]),
        "vinp_onion_peel": (I, [P, P, P, P, I, P, I, I, I, P, P, P, P, C.c_size_t, P]),
        "vinp_reconstruct": (I, [P, P, I, I, I32, I32, P, P, I, P]),
        "vinp_commit": (I, [P, P, P, I, I32, I32, P]),
        "vinp_change_l1": (I, [P, P, I64, P, P]),
        "vinp_change_l2": (I, [P, P, I64, P, P]),
        "vinp_energy": (I, [P, P, P, P]),
        "vinp_brute_force_ws_bytes": (C.c_size_t, [P]),
        "vinp_brute_force": (I, [P, P, P, I32, I32, P, C.c_size_t, P]),
        "vinp_brute_force_list": (I, [P, P, P, P, I32, P]),
        "vinp_brute_force_tc_ws_bytes": (C.c_size_t, [P, I32, I32]),
        "vinp_brute_force_tc": (I, [P, P, P, I32, I32, P, C.c_size_t, P]),
        "vinp_patch_ssd": (I, [P, P, P, I64, P, I, P, P, P]),
        "vinp_patch_sums": (I, [P, I, I32, I32, P]),
        "vinp_active_ws_bytes": (C.c_size_t, [P]),
        "vinp_philox": (I, [P, I64, U64, P, P]),
        "vinp_tc_gemm_u8": (I, [P, P, I, P, P]),
        "vinp_patch_ambiguity": (I, [I, C.c_double, U64, U64, U64, P, P]),
        "vinp_affine_ws_bytes": (C.c_size_t, [I, I, I, I]),
        "vinp_affine_estimate": (I, [P, P, I, I, I, I, I, C.c_double, I32, I32, P, P, P, P, C.c_size_t, P]),
        "vinp_affine_chain": (I, [P, I, P, P, P, P]),
        "vinp_align_warp": (I, [P, P, I, I, I, P, P, P, P]),
        "vinp_unwarp": (I, [P, P, P, I, I, I, P, P, P]),
        "vinp_output_rgb": (I, [P, P, P]),
        "vinp_level_dims": (I, [I, I, I, I, P]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()
EXPORTED = [
    "vinp_last_error", "vinp_version", "vinp_launch_count", "vinp_build_pyramid",
    "vinp_texture_ws_bytes", "vinp_texture_features", "vinp_sets_ws_bytes", "vinp_build_sets",
    "vinp_build_lists", "vinp_layers", "vinp_nnf_init_random", "vinp_nnf_upsample",
    "vinp_nnf_evaluate", "vinp_propagate", "vinp_random_search", "vinp_ann_search",
    "vinp_onion_ws_bytes", "vinp_onion_peel",
    "vinp_reconstruct", "vinp_commit", "vinp_change_l1", "vinp_change_l2", "vinp_energy",
    "vinp_brute_force_ws_bytes", "vinp_brute_force", "vinp_patch_ssd", "vinp_philox",
    "vinp_tc_gemm_u8", "vinp_patch_ambiguity", "vinp_brute_force_list", "vinp_brute_force_tc_ws_bytes", "vinp_brute_force_tc",
    "vinp_affine_ws_bytes", "vinp_affine_estimate", "vinp_affine_chain", "vinp_align_warp", "vinp_unwarp",
    "vinp_output_rgb", "vinp_level_dims", "vinp_patch_sums", "vinp_active_ws_bytes"]


def _check(rc: int, what: str):
    if rc != 0:
        msg = _lib.vinp_last_error()
        raise VinpError(f"{what} failed ({rc}): {msg.decode() if msg else ''}")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def launch_count() -> int:
    return int(_lib.vinp_launch_count())


@dataclass
class Params:
    lam: int = 50
    tex_half: int = -1
    seed: int = 1
    rho: float = 0.5
    rmax: int = -1

    def struct(self):
        return _Params(self.lam, self.tex_half, self.seed, self.rho, self.rmax)


@dataclass
class Level:
    """One pyramid level in HBM (layout: include/vinp.h)."""
    W: int
    H: int
    T: int
    level: int
    device: torch.device
    vox: torch.Tensor = None
    flags: torch.Tensor = None
    layer: Optional[torch.Tensor] = None
    slot: Optional[torch.Tensor] = None
    targets: Optional[torch.Tensor] = None
    holes: Optional[torch.Tensor] = None
    sources: Optional[torch.Tensor] = None
    psum: Optional[torch.Tensor] = None  # patch sums (R42), int16 [N, 8], or None = no lower bound
    active: Optional[torch.Tensor] = None  # zeroed workspace of active_ws_bytes(lv) (see vinp_propagate), or None
    n_targets: int = 0
    n_holes: int = 0
    n_sources: int = 0
    _s: object = field(default=None, repr=False)

    @classmethod
    def alloc(cls, W, H, T, level, device):
        lv = cls(W, H, T, level, torch.device(device))
        N = W * H * T
        # every element is written by vinp_build_pyramid / vinp_texture_features before any read
        lv.vox = torch.empty(N, dtype=torch.int64, device=device)
        lv.flags = torch.empty(N, dtype=torch.uint8, device=device)
        return lv

    @property
    def N(self):
        return self.W * self.H * self.T

    @property
    def rmax(self):
        return max(self.W, self.H, self.T)

    def struct(self):
        s = _Level(self.W, self.H, self.T, self.level, _ptr(self.vox), _ptr(self.flags),
                   _ptr(self.layer), _ptr(self.slot), _ptr(self.targets), self.n_targets,
                   _ptr(self.holes), self.n_holes, _ptr(self.sources), self.n_sources, _ptr(self.psum),
                   _ptr(self.active))
        self._s = s
        return C.byref(s)

    def alloc_lists(self):
        """(Re)allocate the list buffers only when a size changes (repeated calls reuse them)."""
        d = self.device

        def fit(t, n):
            return t if (t is not None and t.numel() == max(n, 1)) else torch.empty(max(n, 1), dtype=torch.int32, device=d)
        self.targets = fit(self.targets, self.n_targets)
        self.holes = fit(self.holes, self.n_holes)
        self.sources = fit(self.sources, self.n_sources)
        self.slot = fit(self.slot, self.N)


@dataclass
class Mirror:
    """Peer copies of an NNF buffer (NEXT #4 second stage): the kernels that write the buffer also
    store every entry into these (P2P), or e through an NVLS multicast address."""
    e: list = field(default_factory=list)       # peer e tensors / device pointers (ints)
    n: list = field(default_factory=list)       # peer n (or None)
    stamp: list = field(default_factory=list)   # peer stamps (or None)
    mc_e: int = 0                               # multicast address of e, 0 = none

    def struct(self):
        m = _Mirror()
        m.n_peers = len(self.e)
        if m.n_peers > MAX_PEERS:
            raise VinpError(f"at most {MAX_PEERS} peers")
        for i in range(m.n_peers):
            m.e[i] = _addr(self.e[i])
            m.n[i] = _addr(self.n[i]) if i < len(self.n) else None
            m.stamp[i] = _addr(self.stamp[i]) if i < len(self.stamp) else None
        m.mc_e = self.mc_e or None
        return m


def _addr(x):
    if x is None:
        return None
    return x if isinstance(x, int) else x.data_ptr()


@dataclass
class NNF:
    e: torch.Tensor
    n: torch.Tensor
    stamp: Optional[torch.Tensor] = None  # R41 change stamps (one per ping-pong buffer) or None
    mirror: Optional[Mirror] = None       # NEXT #4 stage 2: peer copies written by the same kernels
    key: object = None                    # (level index, ping-pong index): names the peer copies
    _s: object = field(default=None, repr=False)

    @classmethod
    def alloc(cls, n_slots, device, n=None, zero=True, stamp=False):
        mk = torch.zeros if zero else torch.empty
        e = mk(max(n_slots, 1), dtype=torch.int64, device=device)
        if n is None:
            n = mk(max(n_slots, 1), dtype=torch.uint8, device=device)
        st = torch.zeros(max(n_slots, 1), dtype=torch.uint8, device=device) if stamp else None
        return cls(e, n, st)

    def struct(self):
        self._m = self.mirror.struct() if self.mirror is not None else None
        self._s = _NNF(_ptr(self.e), _ptr(self.n), _ptr(self.stamp),
                       C.pointer(self._m) if self._m is not None else None)
        return C.byref(self._s)


def _levels_array(levels):
    arr = (_Level * len(levels))()
    for i, lv in enumerate(levels):
        lv.struct()
        arr[i] = lv._s
    return arr


def _sync_back(levels, arr):
    for i, lv in enumerate(levels):
        lv.n_targets, lv.n_holes, lv.n_sources = arr[i].n_targets, arr[i].n_holes, arr[i].n_sources


# ----------------------------------------------------------------------------- calls
def build_pyramid(rgb: torch.Tensor, mask: torch.Tensor, levels):
    arr = _levels_array(levels)
    _check(_lib.vinp_build_pyramid(_ptr(rgb), _ptr(mask), arr, len(levels), _stream()),
           "vinp_build_pyramid")


def texture_features(prm: Params, levels, ws: torch.Tensor):
    arr = _levels_array(levels)
    _check(_lib.vinp_texture_features(C.byref(prm.struct()), arr, len(levels), _ptr(ws),
                                      ws.numel() * ws.element_size(), _stream()),
           "vinp_texture_features")


def texture_ws_bytes(lv1: Level) -> int:
    return int(_lib.vinp_texture_ws_bytes(lv1.struct()))


def sets_ws_bytes(lv1: Level) -> int:
    return int(_lib.vinp_sets_ws_bytes(lv1.struct()))


def build_sets(levels, ws: torch.Tensor):
    arr = _levels_array(levels)
    counts = (C.c_int32 * (3 * len(levels)))()
    _check(_lib.vinp_build_sets(arr, len(levels), counts, _ptr(ws), ws.numel(), _stream()),
           "vinp_build_sets")
    _sync_back(levels, arr)
    return [tuple(counts[3 * i:3 * i + 3]) for i in range(len(levels))]


def build_lists(levels, ws: torch.Tensor):
    arr = _levels_array(levels)
    _check(_lib.vinp_build_lists(arr, len(levels), _ptr(ws), ws.numel(), _stream()),
           "vinp_build_lists")


def layers(lv: Level, ws: torch.Tensor) -> int:
    n = C.c_int32(0)
    _check(_lib.vinp_layers(lv.struct(), C.byref(n), _ptr(ws), _stream()), "vinp_layers")
    return n.value


def nnf_init_random(lv, nnf, prm, outer_code, b=0, e=None):
    e = lv.n_targets if e is None else e
    _check(_lib.vinp_nnf_init_random(lv.struct(), nnf.struct(), C.byref(prm.struct()), outer_code,
                                     b, e, _stream()), "vinp_nnf_init_random")


def nnf_upsample(coarse, cn, fine, fn, prm, b=0, e=None):
    e = fine.n_targets if e is None else e
    _check(_lib.vinp_nnf_upsample(coarse.struct(), cn.struct(), fine.struct(), fn.struct(),
                                  C.byref(prm.struct()), b, e, _stream()), "vinp_nnf_upsample")


def nnf_evaluate(lv, nnf, prm, kb=-1, only_layer=-1, b=0, e=None, counter=None):
    e = lv.n_targets if e is None else e
    _check(_lib.vinp_nnf_evaluate(lv.struct(), nnf.struct(), C.byref(prm.struct()), kb, only_layer,
                                  b, e, _ptr(counter), _stream()), "vinp_nnf_evaluate")


def active_ws_bytes(lv) -> int:
    return int(_lib.vinp_active_ws_bytes(lv.struct()))


def patch_sums(lv, which=0, b=0, e=None):
    """R42: which = 0 fills lv.psum for every voxel, 1 refreshes the targets of slots [b, e)."""
    e = lv.n_targets if e is None else e
    _check(_lib.vinp_patch_sums(lv.struct(), which, b, e, _stream()), "vinp_patch_sums")


class PassClock:
    """Pass numbering of one ANN search for the R41 stale skip (host logic, as csrc/common.cuh):
    evaluate = pass 0, then 1, 2, ... in schedule order; since(step, sign) = the index of the last
    earlier propagation pass with that (step, sign) in the search, 0 if none."""

    def __init__(self):
        self.pass_id = 1
        self.last = {}

    def since(self, step, sign):
        return self.last.get((step, sign), 0)

    def tick(self, step=None, sign=None):  # step None: a random-search pass
        if step is not None:
            self.last[(step, sign)] = self.pass_id
        self.pass_id += 1


def _counter2(counter, nnf):
    """With R41 stamps the library adds skipped stale candidates to counter[1]."""
    if counter is not None and nnf.stamp is not None and counter.numel() < 2:
        raise VinpError("stamped NNF buffers need a 2-element counter (evaluated, stale)")


def propagate(lv, nin, nout, prm, step, sign, kb=-1, only_layer=-1, b=0, e=None, counter=None,
              pass_id=1, since=0):
    """pass_id / since: the R41 pass numbering (used only when both buffers carry stamps; counter
    must then hold 2 int64: [0] evaluated, [1] skipped stale candidates)."""
    _counter2(counter, nin)
    e = lv.n_targets if e is None else e
    _check(_lib.vinp_propagate(lv.struct(), nin.struct(), nout.struct(), C.byref(prm.struct()), step,
                               sign, kb, only_layer, b, e, pass_id, since, _ptr(counter), _stream()),
           "vinp_propagate")


def random_search(lv, nin, nout, prm, outer_code, pm_iter, kb=-1, only_layer=-1, b=0, e=None,
                  counter=None, pass_id=1):
    e = lv.n_targets if e is None else e
    _check(_lib.vinp_random_search(lv.struct(), nin.struct(), nout.struct(), C.byref(prm.struct()),
                                   outer_code, pm_iter, kb, only_layer, b, e, pass_id, _ptr(counter),
                                   _stream()), "vinp_random_search")


def ann_search(lv, a, b, prm, outer_code, K, steps=(8, 4, 2, 1), kb=-1, only_layer=-1, counter=None,
               sign_policy=0):
    _counter2(counter, a)
    st = (C.c_int32 * len(steps))(*steps)
    _check(_lib.vinp_ann_search(lv.struct(), a.struct(), b.struct(), C.byref(prm.struct()), outer_code,
                                K, st, len(steps), sign_policy, kb, only_layer, _ptr(counter), _stream()),
           "vinp_ann_search")


def onion_peel(lv, a, b, prm, K, n_layers, out_rgb, out_tex, steps=(8, 4, 2, 1), counter=None, ws=None,
               sign_policy=0):
    nbytes = int(_lib.vinp_onion_ws_bytes(lv.struct()))
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=lv.device)
    _counter2(counter, a)
    st = (C.c_int32 * len(steps))(*steps)
    _check(_lib.vinp_onion_peel(lv.struct(), a.struct(), b.struct(), C.byref(prm.struct()), K, st,
                                len(steps), sign_policy, n_layers, _ptr(out_rgb), _ptr(out_tex), _ptr(counter),
                                _ptr(ws), ws.numel(), _stream()), "vinp_onion_peel")


def reconstruct(lv, nnf, mode, out_rgb, out_tex, layer_j=-1, hb=0, he=None, commit=True):
    he = lv.n_holes if he is None else he
    _check(_lib.vinp_reconstruct(lv.struct(), nnf.struct(), mode, layer_j, hb, he, _ptr(out_rgb),
                                 _ptr(out_tex), int(commit), _stream()), "vinp_reconstruct")


def commit(lv, out_rgb, out_tex, layer_j=-1, hb=0, he=None):
    he = lv.n_holes if he is None else he
    _check(_lib.vinp_commit(lv.struct(), _ptr(out_rgb), _ptr(out_tex), layer_j, hb, he, _stream()),
           "vinp_commit")


def change_l1(a, b, out):
    _check(_lib.vinp_change_l1(_ptr(a), _ptr(b), a.numel(), _ptr(out), _stream()), "vinp_change_l1")


def change_l2(a, b, out):
    _check(_lib.vinp_change_l2(_ptr(a), _ptr(b), a.numel(), _ptr(out), _stream()), "vinp_change_l2")


def energy(lv, nnf, out):
    _check(_lib.vinp_energy(lv.struct(), nnf.struct(), _ptr(out), _stream()), "vinp_energy")


def brute_force(lv, nnf, prm, b=0, e=None, ws=None):
    e = lv.n_targets if e is None else e
    nbytes = int(_lib.vinp_brute_force_ws_bytes(lv.struct()))
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=lv.device)
    _check(_lib.vinp_brute_force(lv.struct(), nnf.struct(), C.byref(prm.struct()), b, e, _ptr(ws),
                                 ws.numel(), _stream()), "vinp_brute_force")


def brute_force_tc(lv, nnf, prm, b=0, e=None, ws=None):
    """Exact NN on the tensor cores (tcgen05 kind::i8); border targets on CUDA cores."""
    e = lv.n_targets if e is None else e
    nbytes = int(_lib.vinp_brute_force_tc_ws_bytes(lv.struct(), b, e))
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=lv.device)
    _check(_lib.vinp_brute_force_tc(lv.struct(), nnf.struct(), C.byref(prm.struct()), b, e, _ptr(ws),
                                    ws.numel(), _stream()), "vinp_brute_force_tc")


def brute_force_list(lv, nnf, prm, slots: torch.Tensor):
    _check(_lib.vinp_brute_force_list(lv.struct(), nnf.struct(), C.byref(prm.struct()), _ptr(slots),
                                      slots.numel(), _stream()), "vinp_brute_force_list")


def patch_ssd(lv, p, q, prm, kb=-1):
    n = p.numel()
    D = torch.empty(n, dtype=torch.int32, device=lv.device)
    cnt = torch.empty(n, dtype=torch.uint8, device=lv.device)
    _check(_lib.vinp_patch_ssd(lv.struct(), _ptr(p), _ptr(q), n, C.byref(prm.struct()), kb, _ptr(D),
                               _ptr(cnt), _stream()), "vinp_patch_ssd")
    return D, cnt


def philox(ctr: torch.Tensor, seed: int):
    out = torch.empty_like(ctr)
    _check(_lib.vinp_philox(_ptr(ctr), ctr.shape[0], seed, _ptr(out), _stream()), "vinp_philox")
    return out


def tc_gemm_u8(A: torch.Tensor, B: torch.Tensor):
    """C = A B^T on the tensor cores (tcgen05 kind::i8); A, B u8 [128, K]."""
    K = A.shape[1]
    C = torch.empty((128, 128), dtype=torch.int32, device=A.device)
    _check(_lib.vinp_tc_gemm_u8(_ptr(A), _ptr(B), K, _ptr(C), _stream()), "vinp_tc_gemm_u8")
    return C


def patch_ambiguity(N: int, n_trials: int, sigma=5.0, seed=1, trial0=0, hits=None):
    """App. B Monte-Carlo: returns the device int64 hit counter (accumulated)."""
    if hits is None:
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
    _check(_lib.vinp_patch_ambiguity(N, sigma, seed, trial0, n_trials, _ptr(hits), _stream()),
           "vinp_patch_ambiguity")
    return hits


# ---- NEXT #1: affine realignment (Alg. 2; R36-R40) -----------------------------------------------
def affine_ws_bytes(W: int, H: int, T: int, levels: int = 3) -> int:
    return int(_lib.vinp_affine_ws_bytes(W, H, T, levels))


def affine_estimate(rgb: torch.Tensor, mask: torch.Tensor, levels=3, max_iter=20, tol=1e-4, ws=None,
                    out=None, pairs=None):
    """theta_{n,n+1} for the consecutive frame pairs n in `pairs` = (b, e) (default: all): (theta
    f64 [T-1, 6], status i32 [T-1], iters i32 [T-1]), device tensors; rows outside the range are
    left as they were.  rgb u8 [T, H, W, 3], mask u8 [T, H, W] on the device."""
    T, H, W, _ = rgb.shape
    dev = rgb.device
    nb = affine_ws_bytes(W, H, T, levels)
    if ws is None or ws.numel() < nb:
        ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    npairs = max(T - 1, 1)
    if out is None:
        out = (torch.empty((npairs, 6), dtype=torch.float64, device=dev),
               torch.zeros(npairs, dtype=torch.int32, device=dev),
               torch.zeros(npairs, dtype=torch.int32, device=dev))
    theta, status, iters = out
    pb, pe = pairs if pairs is not None else (0, -1)
    _check(_lib.vinp_affine_estimate(_ptr(rgb), _ptr(mask), W, H, T, levels, max_iter, tol, pb, pe, _ptr(theta),
                                     _ptr(status), _ptr(iters), _ptr(ws), ws.numel(), _stream()),
           "vinp_affine_estimate")
    return theta[:T - 1], status[:T - 1], iters[:T - 1]


def affine_chain(pairs: torch.Tensor, T: int, out=None):
    """(fwd, inv) f64 [T, 6] on the device: theta_{n,N_m} and its inverse (R39)."""
    dev = pairs.device
    if out is None:
        out = (torch.empty((T, 6), dtype=torch.float64, device=dev),
               torch.empty((T, 6), dtype=torch.float64, device=dev),
               torch.zeros(1, dtype=torch.int32, device=dev))
    fwd, inv, err = out
    p = pairs.contiguous() if pairs.numel() else None
    _check(_lib.vinp_affine_chain(_ptr(p), T, _ptr(fwd), _ptr(inv), _ptr(err), _stream()), "vinp_affine_chain")
    return fwd, inv, err


def align_warp(rgb: torch.Tensor, mask: torch.Tensor, inv: torch.Tensor, out=None):
    T, H, W, _ = rgb.shape
    if out is None:
        out = (torch.empty_like(rgb), torch.empty_like(mask))
    ro, mo = out
    _check(_lib.vinp_align_warp(_ptr(rgb), _ptr(mask), W, H, T, _ptr(inv), _ptr(ro), _ptr(mo), _stream()),
           "vinp_align_warp")
    return ro, mo


def unwarp(rgb_aligned: torch.Tensor, rgb_orig: torch.Tensor, mask_orig: torch.Tensor, fwd: torch.Tensor,
           out=None):
    T, H, W, _ = rgb_orig.shape
    out = torch.empty_like(rgb_orig) if out is None else out
    _check(_lib.vinp_unwarp(_ptr(rgb_aligned), _ptr(rgb_orig), _ptr(mask_orig), W, H, T, _ptr(fwd), _ptr(out),
                            _stream()), "vinp_unwarp")
    return out


def output_rgb(lv1: Level, out: Optional[torch.Tensor] = None):
    if out is None:
        out = torch.empty((lv1.T, lv1.H, lv1.W, 3), dtype=torch.uint8, device=lv1.vox.device)
    _check(_lib.vinp_output_rgb(lv1.struct(), _ptr(out), _stream()), "vinp_output_rgb")
    return out


def level_dims(W: int, H: int, T: int, L: int):
    """[(W_l, H_l, T)] for l = 1..L (ceil halving of W, H; T unchanged)."""
    out = (C.c_int32 * (3 * L))()
    _check(_lib.vinp_level_dims(W, H, T, L, out), "vinp_level_dims")
    return [tuple(out[3 * l:3 * l + 3]) for l in range(L)]
