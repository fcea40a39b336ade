"""Tensor-core (tcgen05.mma kind::i8) plumbing of the exact-NN mode, pinned by integer matmul."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [32, 64, 384, 512])
def test_tc_gemm_u8_matches_integer_matmul(K):
    from paper_1503_05528_b200 import vinp as V
    rng = np.random.default_rng(K)
    A = rng.integers(0, 256, (128, K), dtype=np.uint8)
    B = rng.integers(0, 256, (128, K), dtype=np.uint8)
    A[0] = 255
    B[0] = 255  # 255*255*K: the largest value of a u8 dot product
    C = V.tc_gemm_u8(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    assert np.array_equal(C.astype(np.int64), ref)


@pytest.mark.parametrize("case,lam", [("c1", 50), ("odd", 0), ("odd", 126), ("c2", 50)])
def test_brute_force_tc_equals_cuda_core(case, lam):
    """Tensor-core exact NN == CUDA-core exact NN (itself bit-exact vs the oracle), bit for bit."""
    import time
    from test_gpu_parity import _setup
    from paper_1503_05528_b200 import vinp as V
    ip, _, _ = _setup(case, lam)
    lv = ip.levels[0]
    n = lv.n_targets if case != "c2" else 6000
    for b, e in ((0, n), (lv.n_targets // 2, min(lv.n_targets, lv.n_targets // 2 + 3000))):
        x = V.NNF.alloc(lv.n_targets, "cuda")
        y = V.NNF.alloc(lv.n_targets, "cuda")
        V.brute_force(lv, x, ip.prm, b, e)
        V.brute_force_tc(lv, y, ip.prm, b, e)
        torch.cuda.synchronize()
        assert torch.equal(x.e[b:e], y.e[b:e]) and torch.equal(x.n[b:e], y.n[b:e]), (case, lam, b)


@pytest.mark.parametrize("N,n", [(9, 1_000_000), (27, 400_000), (125, 100_000)])
def test_ambiguity_gpu_counts_equal_oracle(orc, N, n):
    """Same Philox counters and Box-Muller: the GPU hit count equals the oracle's simulation."""
    from paper_1503_05528_b200 import vinp as V
    for seed, t0 in ((1, 0), (7, 123456789)):
        h = int(V.patch_ambiguity(N, n, 5.0, seed, t0).item())
        assert h == orc.ambiguity_mc(N, n, sigma=5.0, seed=seed, trial0=t0)


def test_ambiguity_gpu_statistics(orc):
    import math
    from paper_1503_05528_b200 import vinp as V
    for N, n in ((25, 50_000_000), (49, 200_000_000)):
        p = orc.ambiguity_exact(N)
        h = int(V.patch_ambiguity(N, n, 5.0, 11).item())
        assert abs(h / n - p) < 5 * math.sqrt(p * (1 - p) / n)


@pytest.mark.parametrize("dims,hf,seed", [((16, 14, 7), 0.3, 1), ((20, 12, 7), 0.3, 4), ((18, 16, 8), 0.25, 2)])
def test_brute_force_tc_few_sources(orc, dims, hf, seed):
    """48-144 sources: one or two source tiles, mostly padding (masked columns, padding-only column
    halves), and fewer targets than a 128-row tile.  Tensor cores == CUDA cores == oracle."""
    from gen.synth import random_volume
    from paper_1503_05528_b200 import Config, Inpainter, vinp as V
    import oracle_ops as OO
    W, H, T = dims
    v, m, _ = random_volume(W, H, T, seed=seed, hole_frac=hf)
    ip = Inpainter(W, H, T, Config(levels=1), "cuda")
    ip.load(v.cuda(), m.cuda())
    lv = ip.levels[0]
    assert lv.n_sources < 160
    x = V.NNF.alloc(lv.n_targets, "cuda")
    y = V.NNF.alloc(lv.n_targets, "cuda")
    V.brute_force(lv, x, ip.prm, 0, lv.n_targets)
    V.brute_force_tc(lv, y, ip.prm, 0, lv.n_targets)
    torch.cuda.synchronize()
    assert torch.equal(x.e[:lv.n_targets], y.e[:lv.n_targets]) and torch.equal(x.n[:lv.n_targets], y.n[:lv.n_targets])
    host = V.Level(lv.W, lv.H, lv.T, 1, torch.device("cpu"))
    for name in ("vox", "flags", "slot", "targets", "holes", "sources"):
        setattr(host, name, getattr(lv, name).cpu())
    host.n_targets, host.n_holes, host.n_sources = lv.n_targets, lv.n_holes, lv.n_sources
    ol = OO._OLevel(host)
    f = orc.NNF.empty(lv.n_targets)
    orc.brute_force(ol, f, ip.prm.lam)
    g = OO._to_orc(host, V.NNF(y.e.cpu(), y.n.cpu()))
    for arr in ("dx", "dy", "dt", "D", "n"):
        assert np.array_equal(getattr(f, arr)[:lv.n_targets], getattr(g, arr)[:lv.n_targets]), arr
