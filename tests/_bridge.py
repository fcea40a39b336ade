"""Test-only conversions between the GPU layout (include/vinp.h) and the oracle's data model."""
import numpy as np
import torch


def level_to_host(lv):
    """GPU vinp Level -> (rgb u8 [T,H,W,3], tex u8 [T,H,W,2], flags u8 [T,H,W])."""
    vb = lv.vox.view(torch.uint8).view(lv.T, lv.H, lv.W, 8).cpu().numpy()
    return (np.ascontiguousarray(vb[..., :3]), np.ascontiguousarray(vb[..., 4:6]),
            lv.flags.view(lv.T, lv.H, lv.W).cpu().numpy())


def pack_vox(rgb, tex):
    T, H, W, _ = rgb.shape
    b = np.zeros((T, H, W, 8), np.uint8)
    b[..., :3] = rgb
    b[..., 4:6] = tex
    return torch.from_numpy(b.reshape(-1).view(np.int64).copy())


def oracle_level(orc, lv, layers=False):
    rgb, tex, flags = level_to_host(lv)
    ol = orc.Level(rgb, tex, (flags & 1).astype(np.uint8), with_layers=False)
    if layers:
        ol.layer = lv.layer.view(lv.T, lv.H, lv.W).cpu().numpy().copy()
    return ol


def nnf_to_oracle(orc, lv, e, n):
    """GPU NNF (e = D<<32 | q, n) over target slots -> oracle NNF (dx, dy, dt, D, n)."""
    nt = lv.n_targets
    e = e[:nt].cpu().numpy().view(np.uint64)
    q = (e & np.uint64(0xFFFFFFFF)).astype(np.int64)
    D = (e >> np.uint64(32)).astype(np.uint32)
    p = lv.targets[:nt].cpu().numpy().astype(np.int64)
    HW = lv.H * lv.W
    f = orc.NNF.empty(nt)
    f.dx[:nt] = (q % lv.W) - (p % lv.W)
    f.dy[:nt] = ((q // lv.W) % lv.H) - ((p // lv.W) % lv.H)
    f.dt[:nt] = (q // HW) - (p // HW)
    f.D[:nt] = D
    f.n[:nt] = n[:nt].cpu().numpy()
    return f


def oracle_to_e(lv, f):
    nt = lv.n_targets
    p = lv.targets[:nt].cpu().numpy().astype(np.int64)
    HW = lv.H * lv.W
    x, y, t = p % lv.W, (p // lv.W) % lv.H, p // HW
    q = ((t + f.dt[:nt]) * lv.H + (y + f.dy[:nt])) * lv.W + (x + f.dx[:nt])
    e = (f.D[:nt].astype(np.uint64) << np.uint64(32)) | q.astype(np.uint64)
    return torch.from_numpy(e.view(np.int64).copy()), torch.from_numpy(f.n[:nt].copy())


def nnf_equal(orc, lv, e, n, f):
    g = nnf_to_oracle(orc, lv, e, n)
    nt = lv.n_targets
    bad = np.flatnonzero((g.dx[:nt] != f.dx[:nt]) | (g.dy[:nt] != f.dy[:nt]) | (g.dt[:nt] != f.dt[:nt])
                         | (g.D[:nt] != f.D[:nt]) | (g.n[:nt] != f.n[:nt]))
    return bad
