"""ctypes wrapper of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by paper_1503_05528_b200/.
The arithmetic lives in oracle.c (cited there, line by line, to PAPER.md); this module only
marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None
# tools/mutation_check.py: build a mutated copy of oracle.c (in a temp dir) instead of this one
_SRC_OVERRIDE = os.environ.get("VINP_ORACLE_SRC")
if _SRC_OVERRIDE:
    _LIB_PATH = os.path.join(os.path.dirname(_SRC_OVERRIDE), "liboracle_mut.so")


def build(force: bool = False) -> str:
    src = _SRC_OVERRIDE or os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = (f"gcc -O2 -std=c11 -ffp-contract=off -fopenmp -fPIC -shared -I {_HERE} -o {_LIB_PATH} "
               f"{src} -lm")
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
    return _LIB_PATH


class OrLevel(C.Structure):
    _fields_ = [("W", C.c_int), ("H", C.c_int), ("T", C.c_int),
                ("rgb", C.c_void_p), ("tex", C.c_void_p), ("occ", C.c_void_p),
                ("src", C.c_void_p), ("tgt", C.c_void_p), ("layer", C.c_void_p),
                ("slot", C.c_void_p),
                ("targets", C.c_void_p), ("n_targets", C.c_int32),
                ("holes", C.c_void_p), ("n_holes", C.c_int32),
                ("sources", C.c_void_p), ("n_sources", C.c_int32)]


class OrNNF(C.Structure):
    _fields_ = [("dx", C.c_void_p), ("dy", C.c_void_p), ("dt", C.c_void_p),
                ("D", C.c_void_p), ("n", C.c_void_p)]


class OrParams(C.Structure):
    _fields_ = [("levels", C.c_int), ("pm_iters", C.c_int), ("fixed_outer", C.c_int),
                ("max_outer", C.c_int), ("lambda_", C.c_int), ("tex_half", C.c_int),
                ("n_steps", C.c_int), ("sign_policy", C.c_int), ("steps", C.c_int * 8), ("seed", C.c_uint64),
                ("rho", C.c_double), ("stop_rule", C.c_int)]


class OrStats(C.Structure):
    _fields_ = [("outer_iters", C.c_int * 16), ("patch_updates", C.c_int64 * 16),
                ("onion_layers", C.c_int), ("change_fixed", (C.c_int64 * 32) * 16),
                ("n_holes", C.c_int64 * 16), ("onion_commits", C.c_int64), ("stale", C.c_int64 * 16)]


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB_PATH)
        P, I, I32, I64, U64, D = C.c_void_p, C.c_int, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "or_philox4x32_10": (None, [P, U64, P]),
            "or_pyramid_down": (None, [P, P, I, I, I, P, P]),
            "or_texture": (None, [P, P, I, I, I, I, P]),
            "or_texture_decimate": (None, [P, I, I, I, I, I, I, P]),
            "or_sets": (None, [P, I, I, I, P, P]),
            "or_layers": (I, [P, I, I, I, P]),
            "or_patch_ssd": (None, [P, I32, I32, I, I, P, P]),
            "or_nnf_init_random": (I64, [P, P, U64, I, C.c_uint32, I32, I32]),
            "or_nnf_upsample": (None, [P, P, P, P, U64, I, I32, I32]),
            "or_nnf_evaluate": (I64, [P, P, I, I, I, I32, I32]),
            "or_propagate": (I64, [P, P, P, I, I, I, I, I, I32, I32, P, P]),
            "or_random_search": (I64, [P, P, P, I, U64, D, I, I, C.c_uint32, I, I, I, I32, I32]),
            "or_reconstruct": (None, [P, P, I, I, I32, I32, P, P]),
            "or_commit": (None, [P, P, P, I32, I32]),
            "or_change_l1": (I64, [P, P, I64]),
            "or_change_l2": (I64, [P, P, I64]),
            "or_stop": (I, [I64, I64, I, I, I]),
            "or_energy": (D, [P, P]),
            "or_brute_force": (I64, [P, P, I, I32, I32]),
            "or_inpaint": (I, [P, P, I, I, I, P, P, P]),
            "or_ambiguity_exact": (D, [I]),
            "or_ann_search_sequential": (I64, [P, P, I, U64, D, I, I, C.c_uint32, I]),
            "or_ambiguity_mc": (I64, [I, D, U64, U64, U64]),
            "or_sets_x": (None, [P, P, I, I, I, P, P]),
            "or_mask_down": (None, [P, I, I, I, P]),
            "or_affine_compose": (None, [P, P, P]),
            "or_affine_invert": (I, [P, P]),
            "or_affine_estimate": (I, [P, P, P, P, I, I, I, I, D, P, P]),
            "or_affine_chain": (I, [P, I, P, P]),
            "or_align_warp": (None, [P, P, I, I, I, P, P, P]),
            "or_unwarp": (None, [P, P, P, I, I, I, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def philox(ctr, seed):
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), seed, _p(out))
    return out


def pyramid_down(rgb, occ):
    T, H, W, _ = rgb.shape
    Wc, Hc = (W + 1) // 2, (H + 1) // 2
    rc = np.zeros((T, Hc, Wc, 3), np.uint8)
    oc = np.zeros((T, Hc, Wc), np.uint8)
    rgb, occ = np.ascontiguousarray(rgb), np.ascontiguousarray(occ)  # keep alive across the call
    lib().or_pyramid_down(_p(rgb), _p(occ), W, H, T,
                          _p(rc), _p(oc))
    return rc, oc


def texture(rgb, occ, h):
    T, H, W, _ = rgb.shape
    tex = np.zeros((T, H, W, 2), np.uint8)
    rgb, occ = np.ascontiguousarray(rgb), np.ascontiguousarray(occ)
    lib().or_texture(_p(rgb), _p(occ), W, H, T, h,
                     _p(tex))
    return tex


def texture_decimate(tex1, level, Wl, Hl):
    T, H1, W1, _ = tex1.shape
    out = np.zeros((T, Hl, Wl, 2), np.uint8)
    tex1 = np.ascontiguousarray(tex1)
    lib().or_texture_decimate(_p(tex1), W1, H1, T, level, Wl, Hl, _p(out))
    return out


def sets(occ):
    T, H, W = occ.shape
    src = np.zeros_like(occ)
    tgt = np.zeros_like(occ)
    occ = np.ascontiguousarray(occ)
    lib().or_sets(_p(occ), W, H, T, _p(src), _p(tgt))
    return src, tgt


def layers(occ):
    T, H, W = occ.shape
    lay = np.zeros_like(occ)
    occ = np.ascontiguousarray(occ)
    n = lib().or_layers(_p(occ), W, H, T, _p(lay))
    return lay, n


class Level:
    """One pyramid level on host buffers (the oracle's own data model)."""

    def __init__(self, rgb, tex, occ, with_layers=False):
        self.rgb = np.ascontiguousarray(rgb, dtype=np.uint8)
        self.tex = np.ascontiguousarray(tex, dtype=np.uint8)
        self.occ = np.ascontiguousarray(occ, dtype=np.uint8)
        self.T, self.H, self.W = occ.shape
        self.src, self.tgt = sets(self.occ)
        self.targets = np.flatnonzero(self.tgt.ravel()).astype(np.int32)
        self.holes = np.flatnonzero(self.occ.ravel()).astype(np.int32)
        self.sources = np.flatnonzero(self.src.ravel()).astype(np.int32)
        self.slot = np.full(self.occ.size, -1, np.int32)
        self.slot[self.targets] = np.arange(len(self.targets), dtype=np.int32)
        self.layer = None
        self.n_layers = 0
        if with_layers:
            self.layer, self.n_layers = layers(self.occ)
        self._s = None

    def struct(self):
        s = OrLevel(self.W, self.H, self.T, _p(self.rgb), _p(self.tex), _p(self.occ), _p(self.src),
                    _p(self.tgt), _p(self.layer), _p(self.slot), _p(self.targets),
                    len(self.targets), _p(self.holes), len(self.holes), _p(self.sources),
                    len(self.sources))
        self._s = s
        return C.byref(s)

    @property
    def rmax(self):
        return max(self.W, self.H, self.T)


@dataclass
class NNF:
    dx: np.ndarray
    dy: np.ndarray
    dt: np.ndarray
    D: np.ndarray
    n: np.ndarray

    @classmethod
    def empty(cls, n):
        z = lambda dt: np.zeros(max(n, 1), dt)
        return cls(z(np.int32), z(np.int32), z(np.int32), z(np.uint32), z(np.uint8))

    def copy(self):
        return NNF(self.dx.copy(), self.dy.copy(), self.dt.copy(), self.D.copy(), self.n.copy())

    def struct(self):
        self._s = OrNNF(_p(self.dx), _p(self.dy), _p(self.dt), _p(self.D), _p(self.n))
        return C.byref(self._s)


def patch_ssd(lv: Level, p, q, lam, kb=-1):
    D = np.zeros(1, np.uint32)
    n = np.zeros(1, np.uint32)
    lib().or_patch_ssd(lv.struct(), int(p), int(q), lam, kb, _p(D), _p(n))
    return int(D[0]), int(n[0])


def init_random(lv, nnf, seed, level, outer_code, b=0, e=None):
    e = len(lv.targets) if e is None else e
    return lib().or_nnf_init_random(lv.struct(), nnf.struct(), seed, level, outer_code, b, e)


def upsample(coarse, cn, fine, fn, seed, level, b=0, e=None):
    e = len(fine.targets) if e is None else e
    lib().or_nnf_upsample(coarse.struct(), cn.struct(), fine.struct(), fn.struct(), seed, level, b, e)


def evaluate(lv, nnf, lam, kb=-1, ol=-1, b=0, e=None):
    e = len(lv.targets) if e is None else e
    return lib().or_nnf_evaluate(lv.struct(), nnf.struct(), lam, kb, ol, b, e)


def propagate(lv, nin, nout, lam, step, sign, kb=-1, ol=-1, b=0, e=None, prev=None, stale=None):
    """prev: the input NNF of the previous pass with this (step, sign) in the same ANN search;
    stale: a 1-element int64 array that receives the R41 stale count (evaluated candidates whose
    neighbour held the same shift in prev)."""
    e = len(lv.targets) if e is None else e
    st = np.zeros(1, np.int64) if stale is None else stale
    return lib().or_propagate(lv.struct(), nin.struct(), nout.struct(), lam, step, sign, kb, ol, b, e,
                              prev.struct() if prev is not None else None, _p(st))


def random_search(lv, nin, nout, lam, seed, rho, rmax, level, outer_code, pm_iter, kb=-1, ol=-1,
                  b=0, e=None):
    e = len(lv.targets) if e is None else e
    return lib().or_random_search(lv.struct(), nin.struct(), nout.struct(), lam, seed, rho, rmax,
                                  level, outer_code, pm_iter, kb, ol, b, e)


def reconstruct(lv, nnf, mode, layer_j=-1, hb=0, he=None, out_rgb=None, out_tex=None):
    he = len(lv.holes) if he is None else he
    nh = max(len(lv.holes), 1)
    out_rgb = np.zeros((nh, 3), np.float32) if out_rgb is None else out_rgb
    out_tex = np.zeros((nh, 2), np.float32) if out_tex is None else out_tex
    lib().or_reconstruct(lv.struct(), nnf.struct(), mode, layer_j, hb, he, _p(out_rgb), _p(out_tex))
    return out_rgb, out_tex


def commit(lv, out_rgb, out_tex, hb=0, he=None):
    he = len(lv.holes) if he is None else he
    lib().or_commit(lv.struct(), _p(out_rgb), _p(out_tex), hb, he)


def change_l1(a, b):
    a = np.ascontiguousarray(a, np.float32).ravel()
    b = np.ascontiguousarray(b, np.float32).ravel()
    return lib().or_change_l1(_p(a), _p(b), a.size)


def change_l2(a, b):
    a = np.ascontiguousarray(a, np.float32).ravel()
    b = np.ascontiguousarray(b, np.float32).ravel()
    return lib().or_change_l2(_p(a), _p(b), a.size)


def stop(e_fixed, n_holes, k, max_outer=20, stop_rule=0):
    return bool(lib().or_stop(int(e_fixed), int(n_holes), int(k), int(max_outer), int(stop_rule)))


def energy(lv, nnf):
    return lib().or_energy(lv.struct(), nnf.struct())


def brute_force(lv, nnf, lam, b=0, e=None):
    e = len(lv.targets) if e is None else e
    return lib().or_brute_force(lv.struct(), nnf.struct(), lam, b, e)


WEIGHTED, UNWEIGHTED, BEST_PATCH = 0, 1, 2


def ann_search(lv, a: NNF, lam, seed, level, outer_code, pm_iters, steps=(8, 4, 2, 1), rho=0.5,
               kb=-1, ol=-1, sign_policy=0, with_stale=False):
    """Alg. 1 schedule (R3/R5/R6), same as or_inpaint's internal ann_search; result in ``a``.
    Returns (a, count) or, with_stale, (a, count, stale) with stale the R41 count (included in
    count)."""
    b = a.copy()
    cnt = evaluate(lv, a, lam, kb, ol)
    snaps = {}  # (step, sign) -> input of the last such pass (R41 stale count)
    stale = np.zeros(1, np.int64)
    n_stale = 0
    for k in range(1, pm_iters + 1):
        sign = 0 if sign_policy else (1 if k % 2 == 1 else -1)
        for s in steps:
            cnt += propagate(lv, a, b, lam, s, sign, kb, ol, prev=snaps.get((s, sign)), stale=stale)
            n_stale += int(stale[0])
            snaps[(s, sign)] = a.copy()
            a, b = b, a
        cnt += random_search(lv, a, b, lam, seed, rho, lv.rmax, level, outer_code, k, kb, ol)
        a, b = b, a
    return (a, cnt, n_stale) if with_stale else (a, cnt)


def inpaint(rgb, occ, levels, pm_iters=10, fixed_outer=0, max_outer=20, lam=50, seed=1,
            steps=(8, 4, 2, 1), rho=0.5, tex_half=-1, sign_policy=0, stop_rule=0):
    T, H, W, _ = rgb.shape
    prm = OrParams()
    prm.levels, prm.pm_iters, prm.fixed_outer, prm.max_outer = levels, pm_iters, fixed_outer, max_outer
    prm.lambda_, prm.tex_half, prm.n_steps, prm.sign_policy = lam, tex_half, len(steps), sign_policy
    for i, s in enumerate(steps):
        prm.steps[i] = s
    prm.seed, prm.rho, prm.stop_rule = seed, rho, stop_rule
    st = OrStats()
    out = np.zeros_like(rgb)
    rgb, occ = np.ascontiguousarray(rgb), np.ascontiguousarray(occ)
    rc = lib().or_inpaint(_p(rgb), _p(occ), W, H, T,
                          C.byref(prm), _p(out), C.byref(st))
    if rc != 0:
        raise RuntimeError(f"or_inpaint failed: {rc}")
    return out, dict(outer_iters=list(st.outer_iters)[:levels],
                     patch_updates=list(st.patch_updates)[:levels], onion_layers=st.onion_layers,
                     change_fixed=[list(st.change_fixed[l])[:min(st.outer_iters[l], 32)] for l in range(levels)],
                     n_holes=list(st.n_holes)[:levels], onion_commits=st.onion_commits,
                     stale=list(st.stale)[:levels])


def ambiguity_exact(N):
    """App. B: exact P(random patch beats the constant patch) for N i.i.d. Gaussian components."""
    return lib().or_ambiguity_exact(N)


def ambiguity_mc(N, n_trials, sigma=5.0, seed=1, trial0=0):
    return lib().or_ambiguity_mc(N, sigma, seed, trial0, n_trials)


def ann_search_sequential(lv, nnf, lam, seed, level, outer_code, K, rho=0.5, rmax=None):
    """NEXT #2: Alg. 1 as printed (in-place lexicographic scans); modifies ``nnf``."""
    rmax = lv.rmax if rmax is None else rmax
    return lib().or_ann_search_sequential(lv.struct(), nnf.struct(), lam, seed, rho, rmax, level,
                                          outer_code, K)


# ---- NEXT #1: affine realignment (Alg. 2; R36-R40) --------------------------------------------
IDENTITY = (0.0, 1.0, 0.0, 0.0, 0.0, 1.0)


def _th(t):
    return np.ascontiguousarray(np.asarray(t, dtype=np.float64).reshape(-1))


def sets_x(occ, inv):
    T, H, W = occ.shape
    src = np.zeros_like(occ)
    tgt = np.zeros_like(occ)
    keep = [np.ascontiguousarray(occ), None if inv is None else np.ascontiguousarray(inv)]
    lib().or_sets_x(_p(keep[0]), _p(keep[1]), W, H, T, _p(src), _p(tgt))
    return src, tgt


def mask_down(m):
    T, H, W = m.shape
    out = np.zeros((T, (H + 1) // 2, (W + 1) // 2), np.uint8)
    m = np.ascontiguousarray(m, np.uint8)
    lib().or_mask_down(_p(m), W, H, T, _p(out))
    return out


def affine_compose(t2, t1):
    out = np.zeros(6)
    a, b = _th(t2), _th(t1)
    lib().or_affine_compose(_p(a), _p(b), _p(out))
    return out


def affine_invert(t):
    out = np.zeros(6)
    a = _th(t)
    if lib().or_affine_invert(_p(a), _p(out)):
        raise ValueError("singular affine map")
    return out


def affine_estimate(rgb_a, rgb_b, occ_a=None, occ_b=None, levels=3, max_iter=20, tol=1e-4):
    """theta_{a->b} (6 doubles, spec form), status (0 ok / 1 degenerate), total IRLS iterations."""
    H, W, _ = rgb_a.shape
    th = np.zeros(6)
    it = np.zeros(1, np.int32)
    ca = lambda a: None if a is None else np.ascontiguousarray(a, np.uint8)
    keep = [np.ascontiguousarray(rgb_a), np.ascontiguousarray(rgb_b), ca(occ_a), ca(occ_b)]
    st = lib().or_affine_estimate(*[_p(k) for k in keep], W, H, levels, max_iter, tol, _p(th), _p(it))
    return th, int(st), int(it[0])


def affine_chain(pairs, T):
    pairs = np.ascontiguousarray(np.asarray(pairs, np.float64).reshape(max(T - 1, 1), 6))
    fwd = np.zeros((T, 6))
    inv = np.zeros((T, 6))
    if lib().or_affine_chain(_p(pairs), T, _p(fwd), _p(inv)):
        raise ValueError("singular affine chain")
    return fwd, inv


def align_warp(rgb, occ, inv):
    T, H, W, _ = rgb.shape
    out = np.zeros_like(rgb)
    mo = np.zeros((T, H, W), np.uint8)
    keep = [np.ascontiguousarray(rgb), np.ascontiguousarray(occ), np.ascontiguousarray(inv, np.float64)]
    lib().or_align_warp(_p(keep[0]), _p(keep[1]), W, H, T, _p(keep[2]), _p(out), _p(mo))
    return out, mo


def unwarp(rgb_aligned, rgb_orig, occ_orig, fwd):
    T, H, W, _ = rgb_orig.shape
    out = np.zeros_like(rgb_orig)
    keep = [np.ascontiguousarray(rgb_aligned), np.ascontiguousarray(rgb_orig),
            np.ascontiguousarray(occ_orig), np.ascontiguousarray(fwd, np.float64)]
    lib().or_unwarp(_p(keep[0]), _p(keep[1]), _p(keep[2]), W, H, T, _p(keep[3]), _p(out))
    return out


def align_pipeline(rgb, occ, levels=3, max_iter=20, tol=1e-4):
    """Alg. 2 on the host: pairwise estimates, chain, warp.  Returns (aligned rgb, aligned mask
    codes, fwd, inv, pair thetas, statuses)."""
    T = rgb.shape[0]
    pairs = np.zeros((max(T - 1, 1), 6))
    pairs[:] = IDENTITY
    stats = []
    for n in range(T - 1):
        th, st, _ = affine_estimate(rgb[n], rgb[n + 1], occ[n], occ[n + 1], levels, max_iter, tol)
        pairs[n] = th
        stats.append(st)
    fwd, inv = affine_chain(pairs, T)
    ar, am = align_warp(rgb, occ, inv)
    return ar, am, fwd, inv, pairs[:T - 1], stats
