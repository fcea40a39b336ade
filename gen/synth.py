"""Seeded synthetic videos + occlusion masks for configs c1..c5 (BASELINE.json ``configs``).

This module is the ONLY code shared by the oracle side and the CUDA side: it draws
inputs and holds none of the inpainting method's arithmetic.  Recipe: SURVEY.md §8(d)
"Synthetic inputs" (restated in DESIGN.md §3).  The paper's own videos (Table 1,
PAPER.md l.1146-1149) are not available; these scenes stand in for them: moving
objects crossing the hole (Figs. l.1028-1072), dynamic textures (l.902-912), moving
background (l.951-966).

Randomness is a counter-based hash: Philox4x32-10 (Salmon et al., SC'11) evaluated
elementwise on int64 torch tensors, so the same code runs on CPU (tests) and on a
GPU (bench, where c5 has 207 M voxels).  Values are computed in float64 and rounded
with clip(floor(v + 0.5), 0, 255).  The hole content of the returned video is zeroed.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

M32 = 0xFFFFFFFF
_PH_M0, _PH_M1 = 0xD2511F53, 0xCD9E8D57
_PH_W0, _PH_W1 = 0x9E3779B9, 0xBB67AE85


def _mulhilo(a: int, b: torch.Tensor):
    p = b * a  # int64 wraps mod 2^64, low 64 bits exact
    return (p >> 32) & M32, p & M32


def philox(c0, c1, c2, c3, seed: int):
    """Philox4x32-10 on int64 tensors holding uint32 values; returns 4 tensors in [0, 2^32)."""
    ref = next(x for x in (c0, c1, c2, c3) if isinstance(x, torch.Tensor))
    c = [torch.as_tensor(x, dtype=torch.int64, device=ref.device).expand_as(ref) & M32
         for x in (c0, c1, c2, c3)]
    k0, k1 = seed & M32, (seed >> 32) & M32
    for _ in range(10):
        hi0, lo0 = _mulhilo(_PH_M0, c[0])
        hi1, lo1 = _mulhilo(_PH_M1, c[2])
        c = [(hi1 ^ c[1] ^ k0) & M32, lo1, (hi0 ^ c[3] ^ k1) & M32, lo0]
        k0 = (k0 + _PH_W0) & M32
        k1 = (k1 + _PH_W1) & M32
    return c


def uniform(a, b, c, d, seed):
    """U(a,b,c,d; seed) in [0,1) from Philox word 0."""
    return philox(a, b, c, d, seed)[0].to(torch.float64) / 4294967296.0


def normal(a, b, c, d, seed):
    """Box-Muller normal from two Philox words."""
    w = philox(a, b, c, d, seed)
    u1 = (w[0].to(torch.float64) + 0.5) / 4294967296.0
    u2 = w[1].to(torch.float64) / 4294967296.0
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)


def _scalar_uniform(a, b, c, d, seed):
    return float(uniform(torch.tensor([a]), b, c, d, seed)[0])


def vnoise(x: torch.Tensor, y: torch.Tensor, cell: float, salt: int, seed: int):
    """Smoothstep-bilinear value noise of lattice values U(gx, gy, salt)."""
    fx, fy = x / cell, y / cell
    gx, gy = torch.floor(fx), torch.floor(fy)
    tx, ty = fx - gx, fy - gy
    sx, sy = tx * tx * (3 - 2 * tx), ty * ty * (3 - 2 * ty)
    gx, gy = gx.to(torch.int64), gy.to(torch.int64)
    # hash only the lattice points the grid touches, then gather
    x0, x1 = int(gx.min()), int(gx.max()) + 1
    y0, y1 = int(gy.min()), int(gy.max()) + 1
    ly = torch.arange(y0, y1 + 1, device=x.device, dtype=torch.int64).view(-1, 1)
    lx = torch.arange(x0, x1 + 1, device=x.device, dtype=torch.int64).view(1, -1)
    table = uniform(lx.expand(ly.shape[0], -1), ly.expand(-1, lx.shape[1]), salt, 0x5EED, seed)
    nx = x1 - x0 + 1
    flat = table.reshape(-1)
    i00 = (gy - y0) * nx + (gx - x0)
    v00 = flat[i00]
    v10 = flat[i00 + 1]
    v01 = flat[i00 + nx]
    v11 = flat[i00 + nx + 1]
    a = v00 + (v10 - v00) * sx
    b = v01 + (v11 - v01) * sx
    return a + (b - a) * sy


def fbm(x, y, salt, seed, octaves=5, base_cell=64.0):
    acc = torch.zeros_like(x)
    norm = 0.0
    amp = 1.0
    cell = base_cell
    for o in range(octaves):
        acc = acc + amp * vnoise(x, y, cell, salt * 16 + o, seed)
        norm += amp
        amp *= 0.5
        cell /= 2.0
    return acc / norm


def _reflect(pos: float, lo: float, hi: float) -> float:
    """Triangle-wave reflection of a coordinate into [lo, hi]."""
    span = hi - lo
    if span <= 0:
        return lo
    m = (pos - lo) % (2 * span)
    return lo + (m if m <= span else 2 * span - m)


@dataclass
class Config:
    name: str
    W: int
    H: int
    T: int
    levels: int
    pm_iters: int
    fixed_outer: int  # >0: exactly this many outer iterations (c1); 0: stopping rule
    max_outer: int
    lam: int
    seed: int


CONFIGS = {
    "c1": Config("c1", 64, 48, 20, 1, 4, 3, 3, 50, 1),
    "c2": Config("c2", 320, 240, 60, 2, 10, 0, 20, 50, 2),
    "c3": Config("c3", 854, 480, 100, 3, 10, 0, 20, 50, 3),
    "c4": Config("c4", 1280, 720, 120, 4, 10, 0, 20, 50, 4),
    "c5": Config("c5", 1920, 1080, 100, 4, 10, 0, 20, 50, 5),
}


def _grid(W, H, device):
    y = torch.arange(H, dtype=torch.float64, device=device).view(H, 1).expand(H, W)
    x = torch.arange(W, dtype=torch.float64, device=device).view(1, W).expand(H, W)
    return x, y


def _objects(n, W, H, seed, size_lo, size_hi, kinds=("disc", "rect"), salt=300):
    objs = []
    for i in range(n):
        u = [_scalar_uniform(i, j, salt, 0, seed) for j in range(8)]
        kind = kinds[int(u[0] * len(kinds)) % len(kinds)]
        size = size_lo + u[1] * (size_hi - size_lo)
        size2 = size_lo + u[2] * (size_hi - size_lo)
        x0 = u[3] * (W - size)
        y0 = u[4] * (H - size2)
        speed = 1.0 + 2.0 * u[5]
        ang = 2 * math.pi * u[6]
        objs.append(dict(kind=kind, a=size, b=size2, x0=x0, y0=y0,
                         vx=speed * math.cos(ang), vy=speed * math.sin(ang),
                         salt=salt + 10 + i, tint=u[7]))
    return objs


def _paint_objects(img, objs, t, x, y, W, H, seed):
    """Objects move linearly, reflect at frame borders, carry rigid vnoise texture."""
    for ob in objs:
        if ob["kind"] == "disc":
            r = ob["a"] / 2.0
            cx = _reflect(ob["x0"] + r + ob["vx"] * t, r, W - r)
            cy = _reflect(ob["y0"] + r + ob["vy"] * t, r, H - r)
            bx0, bx1, by0, by1 = cx - r, cx + r, cy - r, cy + r
        else:
            w2, h2 = ob["a"], ob["b"]
            ox = _reflect(ob["x0"] + ob["vx"] * t, 0.0, W - w2)
            oy = _reflect(ob["y0"] + ob["vy"] * t, 0.0, H - h2)
            bx0, bx1, by0, by1 = ox, ox + w2, oy, oy + h2
        # restrict to the bounding box (pure speed-up; same pixels)
        ix0, ix1 = max(0, int(math.floor(bx0)) - 1), min(W, int(math.ceil(bx1)) + 1)
        iy0, iy1 = max(0, int(math.floor(by0)) - 1), min(H, int(math.ceil(by1)) + 1)
        if ix0 >= ix1 or iy0 >= iy1:
            continue
        xs, ys = x[iy0:iy1, ix0:ix1], y[iy0:iy1, ix0:ix1]
        if ob["kind"] == "disc":
            inside = (xs - cx) ** 2 + (ys - cy) ** 2 <= r * r
            lx, ly = xs - cx + r, ys - cy + r
        else:
            inside = (xs >= ox) & (xs < ox + w2) & (ys >= oy) & (ys < oy + h2)
            lx, ly = xs - ox, ys - oy
        for c in range(3):
            tex = 255.0 * (0.25 + 0.5 * ob["tint"] * (c == 1)) + 255.0 * 0.5 * (
                vnoise(lx, ly, 4.0, ob["salt"] * 4 + c, seed) - 0.5)
            sub = img[c][iy0:iy1, ix0:ix1]
            img[c][iy0:iy1, ix0:ix1] = torch.where(inside, tex, sub)


def _round_u8(v):
    return torch.clamp(torch.floor(v + 0.5), 0, 255).to(torch.uint8)


def generate(name: str, device="cpu", frames=None):
    """Returns (video u8 [T,H,W,3] with hole zeroed, mask u8 [T,H,W] (1 = occluded), truth u8 [T,H,W,3]).

    ``frames`` optionally bounds the frame count (bounded samples for the CPU baseline)."""
    cfg = CONFIGS[name]
    W, H, T, seed = cfg.W, cfg.H, cfg.T, cfg.seed
    if frames is not None:
        T = min(T, frames)
    x, y = _grid(W, H, device)
    video = torch.empty((T, H, W, 3), dtype=torch.uint8, device=device)
    mask = torch.empty((T, H, W), dtype=torch.uint8, device=device)

    if name == "c1":
        bg = [255.0 * vnoise(x, y, 8.0, 1 + c, seed) for c in range(3)]
        for t in range(T):
            img = [b.clone() for b in bg]
            inside = (x >= 18 + t) & (x < 26 + t) & (y >= 20) & (y < 28)
            lx = (x - (18 + t)).to(torch.int64)
            ly = (y - 20).to(torch.int64)
            for c in range(3):
                img[c] = torch.where(inside, 255.0 * uniform(lx, ly, 100 + c, 0, seed), img[c])
            video[t] = _round_u8(torch.stack(img, -1))
            m = (x >= 26) & (x < 38) & (y >= 18) & (y < 30) & (5 <= t < 15)
            mask[t] = m.to(torch.uint8)
    elif name == "c2":
        objs = _objects(3, W, H, seed, 20.0, 40.0, kinds=("disc",))
        for t in range(T):
            xs = x - 0.5 * t
            img = []
            for c in range(3):
                ph = c * 2 * math.pi / 3
                v = (128 + 50 * torch.sin(2 * math.pi * xs / 32 + ph) * torch.cos(2 * math.pi * y / 24)
                     + 40 * (vnoise(xs, y, 4.0, 10 + c, seed) - 0.5))
                img.append(v)
            _paint_objects(img, objs, t, x, y, W, H, seed)
            video[t] = _round_u8(torch.stack(img, -1))
            mask[t] = (((x - 160) / 40) ** 2 + ((y - 120) / 24) ** 2 <= 1).to(torch.uint8)
    elif name in ("c3", "c5"):
        if name == "c3":
            objs = _objects(5, W, H, seed, 20.0, 60.0, kinds=("rect",))
            base = (128.0, 128.0, 128.0)
        else:
            objs = _objects(12, W, H, seed, 20.0, 120.0)
            base = (40.0, 90.0, 160.0)
            xf = torch.arange(W + T, dtype=torch.float64, device=device).view(1, -1).expand(H, -1)
            yf = torch.arange(H, dtype=torch.float64, device=device).view(-1, 1).expand(-1, W + T)
            pan = [255.0 * fbm(xf, yf, 20 + c, seed) for c in range(3)]
        yi = torch.arange(H, device=device).view(H, 1).expand(H, W).to(torch.int64)
        xi = torch.arange(W, device=device).view(1, W).expand(H, W).to(torch.int64)
        pix = yi * W + xi
        state = None
        for t in range(T):
            g = [normal(pix, t, 40 + c, 7, seed) for c in range(3)]
            if state is None:
                state = [20.0 * gc for gc in g]
            else:
                state = [0.9 * s + 20.0 * math.sqrt(0.19) * gc for s, gc in zip(state, g)]
            img = [base[c] + state[c] for c in range(3)]
            if name == "c5":
                top = y < 648
                for c in range(3):
                    img[c] = torch.where(top, pan[c][:, t:t + W], img[c])
            _paint_objects(img, objs, t, x, y, W, H, seed)
            video[t] = _round_u8(torch.stack(img, -1))
            if name == "c3":
                m = (x - (327 + 2 * t)) ** 2 + (y - 240) ** 2 <= 88 * 88
            else:
                cx = 960 + 2 * (t - 49.5)
                m = ((x - cx) / 330) ** 2 + ((y - 540) / 250) ** 2 + ((t - 49.5) / 48) ** 2 <= 1
            mask[t] = m.to(torch.uint8)
    elif name == "c4":
        objs = _objects(8, W, H, seed, 16.0, 64.0)
        xf = torch.arange(W + 2 * T, dtype=torch.float64, device=device).view(1, -1).expand(H, -1)
        yf = torch.arange(H, dtype=torch.float64, device=device).view(-1, 1).expand(-1, W + 2 * T)
        pan = [255.0 * fbm(xf, yf, 30 + c, seed) for c in range(3)]
        for t in range(T):
            img = [pan[c][:, 2 * t:2 * t + W].clone() for c in range(3)]
            _paint_objects(img, objs, t, x, y, W, H, seed)
            video[t] = _round_u8(torch.stack(img, -1))
            m = (((x - (360 + t)) / 100) ** 2 + ((y - 260) / 73) ** 2 <= 1) | \
                (((x - (920 - t)) / 96) ** 2 + ((y - 470) / 76) ** 2 <= 1)
            mask[t] = m.to(torch.uint8)
    else:
        raise KeyError(name)

    truth = video.clone()
    video[mask.bool()] = 0
    return video, mask, truth


def random_volume(W, H, T, seed, hole_frac=0.05, device="cpu", smooth=True):
    """Small seeded random volume + random box hole for property / parity tests."""
    x, y = _grid(W, H, device)
    video = torch.empty((T, H, W, 3), dtype=torch.uint8, device=device)
    for t in range(T):
        img = []
        for c in range(3):
            if smooth:
                v = 255.0 * vnoise(x + 0.7 * t, y, 6.0, 50 + c, seed) + 40 * (uniform(
                    (y * W + x).to(torch.int64), t, 60 + c, 1, seed) - 0.5)
            else:
                v = 255.0 * uniform((y * W + x).to(torch.int64), t, 60 + c, 1, seed)
            img.append(v)
        video[t] = _round_u8(torch.stack(img, -1))
    bw = max(1, int(round(W * math.sqrt(hole_frac))))
    bh = max(1, int(round(H * math.sqrt(hole_frac))))
    x0 = int(_scalar_uniform(1, 0, 900, 0, seed) * (W - bw))
    y0 = int(_scalar_uniform(2, 0, 900, 0, seed) * (H - bh))
    t0 = int(_scalar_uniform(3, 0, 900, 0, seed) * max(1, T // 2))
    t1 = min(T, t0 + max(1, T // 2))
    mask = torch.zeros((T, H, W), dtype=torch.uint8, device=device)
    mask[t0:t1, y0:y0 + bh, x0:x0 + bw] = 1
    truth = video.clone()
    video[mask.bool()] = 0
    return video, mask, truth


def camera_video(W, H, T, seed, cams, noise=0.0, block=None, device="cpu", cell=32.0):
    """Frames of a static textured world seen through per-frame affine cameras (NEXT #1 inputs).

    ``cams[t]`` = (c0..c5): frame t's pixel (x, y) shows world point
    (c0 + c1 x + c2 y, c3 + c4 x + c5 y); the world is 255 * fbm (one field per channel).  Then
    the true inter-frame motion is theta_{t,t+1} = cams[t+1]^{-1} o cams[t].  ``noise``: i.i.d.
    Gaussian sigma (grey levels) per pixel and channel.  ``block`` = (x0, y0, w, h, dx, dy): a
    fixed frame rectangle showing a second texture that moves by (dx, dy) per frame (an
    independently moving object).  Returns u8 [T, H, W, 3]."""
    x, y = _grid(W, H, device)
    out = torch.empty((T, H, W, 3), dtype=torch.uint8, device=device)
    pix = (y * W + x).to(torch.int64)
    for t in range(T):
        c = cams[t]
        wx = c[0] + c[1] * x + c[2] * y
        wy = c[3] + c[4] * x + c[5] * y
        img = [255.0 * fbm(wx, wy, 70 + k, seed, base_cell=cell) for k in range(3)]
        if block is not None:
            bx0, by0, bw, bh, bdx, bdy = block
            ins = (x >= bx0) & (x < bx0 + bw) & (y >= by0) & (y < by0 + bh)
            for k in range(3):
                img[k] = torch.where(ins, 255.0 * fbm(x - bdx * t, y - bdy * t, 80 + k, seed, base_cell=cell),
                                     img[k])
        if noise > 0:
            img = [v + noise * normal(pix, t, 90 + k, 3, seed) for k, v in enumerate(img)]
        out[t] = _round_u8(torch.stack(img, -1))
    return out


def random_holes(W, H, T, seed, n=2, device="cpu"):
    """Union of n seeded axis-aligned ellipsoids (random centre, radii 1..W/4 etc.; may touch or
    cross the volume border) as a u8 [T, H, W] occlusion mask: fuzz inputs for parity tests."""
    t = torch.arange(T, dtype=torch.float64, device=device).view(T, 1, 1)
    y = torch.arange(H, dtype=torch.float64, device=device).view(1, H, 1)
    x = torch.arange(W, dtype=torch.float64, device=device).view(1, 1, W)
    m = torch.zeros((T, H, W), dtype=torch.bool, device=device)
    for i in range(n):
        u = [_scalar_uniform(10 + i, k, 77, 5, seed) for k in range(6)]
        cx, cy, ct = u[0] * W, u[1] * H, u[2] * T
        rx, ry, rt = 1 + u[3] * W / 4, 1 + u[4] * H / 4, 1 + u[5] * T / 3
        m |= ((x - cx) / rx) ** 2 + ((y - cy) / ry) ** 2 + ((t - ct) / rt) ** 2 <= 1
    return m.to(torch.uint8)
