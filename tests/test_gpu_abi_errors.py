"""The C ABI's error behaviour (include/vinp.h conventions): argument errors are detected
synchronously and reported as VINP_E_INVALID / VINP_E_UNSUPPORTED / VINP_E_NO_SOURCE with a
message from vinp_last_error; nothing is launched; the library stays usable afterwards."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1503_05528_b200 import vinp as V
    return V, V._lib


def test_invalid_arguments_are_reported_synchronously():
    V, lib = _lib()
    n0 = V.launch_count()
    # null buffers / bad level count
    assert lib.vinp_build_pyramid(None, None, None, 1, None) == 1
    assert b"bad arguments" in lib.vinp_last_error()
    # lambda outside [0, 126]: D would not fit 32 bits
    lv = V.Level.alloc(16, 12, 6, 1, torch.device("cuda"))
    nnf = V.NNF.alloc(4, "cuda")
    prm = V.Params(lam=127)
    st = lib.vinp_nnf_evaluate(lv.struct(), nnf.struct(), C.byref(prm.struct()), -1, -1, 0, 1, None, None)
    assert st in (1, 4) and lib.vinp_last_error()
    # propagate needs two distinct NNF buffers
    st = lib.vinp_propagate(lv.struct(), nnf.struct(), nnf.struct(), C.byref(V.Params().struct()), 8, 1, -1,
                            -1, 0, 0, 1, 0, None, None)
    assert st == 1 and lib.vinp_last_error()
    # realignment: frames must be at least 2 x 2
    assert lib.vinp_affine_estimate(None, None, 1, 1, 3, 3, 20, 1e-4, 0, -1, None, None, None, None, 0, None) == 1
    assert V.launch_count() == n0  # nothing was launched
    # the library is still usable
    assert V.level_dims(8, 8, 2, 2) == [(8, 8, 2), (4, 4, 2)]


def test_dimension_limits():
    V, lib = _lib()
    with pytest.raises(V.VinpError, match="2\\^31"):
        V.level_dims(4096, 4096, 128, 1)
    dims = (C.c_int32 * 3)()
    assert lib.vinp_level_dims(0, 4, 4, 1, dims) == 1


def test_no_source_is_refused_by_the_tensor_core_mode():
    """D~ empty at a level: VINP_E_NO_SOURCE, not a crash."""
    V, lib = _lib()
    from paper_1503_05528_b200 import Config, Inpainter
    v = torch.zeros((8, 10, 12, 3), dtype=torch.uint8, device="cuda")
    m = torch.ones((8, 10, 12), dtype=torch.uint8, device="cuda")
    ip = Inpainter(12, 10, 8, Config(levels=1), "cuda")
    with pytest.raises(V.VinpError):
        ip.load(v, m)  # the driver refuses D~ = empty
    lv = ip.levels[0]
    lv.n_sources = 0
    out = V.NNF.alloc(4, "cuda")
    ws = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    st = lib.vinp_brute_force_tc(lv.struct(), out.struct(), C.byref(V.Params().struct()), 0, 1, V._ptr(ws),
                                 ws.numel(), None)
    assert st in (1, 2)


def test_brute_force_list_checks_arguments():
    """vinp_brute_force_list: the same synchronous argument checks as vinp_brute_force."""
    V, lib = _lib()
    lv = V.Level.alloc(16, 12, 6, 1, torch.device("cuda"))
    out = V.NNF.alloc(4, "cuda")
    n0 = V.launch_count()
    prm = V.Params()
    assert lib.vinp_brute_force_list(lv.struct(), out.struct(), C.byref(prm.struct()), None, 3, None) == 1
    assert lib.vinp_brute_force_list(None, out.struct(), C.byref(prm.struct()), None, 0, None) == 1
    assert lib.vinp_brute_force_list(lv.struct(), out.struct(), C.byref(V.Params(lam=127).struct()), None, 0,
                                     None) in (1, 4)
    assert V.launch_count() == n0
    assert V._lib.vinp_brute_force_ws_bytes(lv.struct()) == 0


def test_too_many_random_search_radii_are_refused():
    """rmax rho^33 >= 1 (e.g. rmax = 1920, rho = 0.8): refused (VINP_E_UNSUPPORTED), not truncated."""
    V, lib = _lib()
    from gen.synth import generate
    from paper_1503_05528_b200 import Config, Inpainter
    v, m, _ = generate("c1")
    ip = Inpainter(64, 48, 20, Config(levels=1), "cuda")
    ip.load(v.cuda(), m.cuda())
    st = ip.states[0]
    ok = V.Params(rho=0.8, rmax=1500)   # R_32 = 1.19, R_33 = 0.95: 32 radii, accepted
    bad = V.Params(rho=0.8, rmax=1920)  # R_33 = 1.22: refused
    V.random_search(st.lv, st.a, st.b, ok, 0, 1)
    with pytest.raises(V.VinpError, match="32 random-search radii"):
        V.random_search(st.lv, st.a, st.b, bad, 0, 1)
