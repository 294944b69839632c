"""Seeded synthetic images with the shapes and statistics BASELINE.json names.

There is no public dataset for this path; these generators are
frozen stand-ins.  Both the CUDA path and the CPU oracle consume the *same* arrays,
so generator details cannot affect parity.  All randomness comes from
``numpy.random.default_rng(seed)`` and float64 arithmetic, so a given numpy
version reproduces the arrays bit for bit on any host.

configs (BASELINE.json "configs"):
  1  cfg1_gray12(seed)   (1,512,512) uint16, 12-bit valid range, L3, lossless
  2  cfg2_pathology(...) (H,W,3) uint8 HWC, RCT, L4
  3  same generator at 4096^2, L5, lossy (planes dropped 2 / 4)
  4  16x16 tiles of 4096^2, tile t uses seed + t, L6, RCT
  5  cfg5_fluorescence   (4,8192,8192) uint16, full range, L5, decode-only
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    1: dict(name="gray12-512", width=512, height=512, channels=1, bit_depth=12, levels=3, use_rct=False),
    2: dict(name="rgb8-2048-rct", width=2048, height=2048, channels=3, bit_depth=8, levels=4, use_rct=True),
    3: dict(name="rgb8-4096-rct-lossy", width=4096, height=4096, channels=3, bit_depth=8, levels=5, use_rct=True,
            planes_dropped=(2, 4)),
    4: dict(name="wsi-65536-tiles4096", width=4096, height=4096, channels=3, bit_depth=8, levels=6, use_rct=True,
            tiles=(16, 16)),
    5: dict(name="fluo16-8192x4", width=8192, height=8192, channels=4, bit_depth=16, levels=5, use_rct=False),
}


def cfg1_gray12(seed: int = 0, size: int = 512) -> np.ndarray:
    """(1,H,W) uint16: 1000 + 32 Gaussian blobs (sigma 8-64, amplitude 200-1500) + N(0,20), clipped to 12 bits."""
    rng = np.random.default_rng(seed)
    n = 32
    cy = rng.uniform(0, size, n)
    cx = rng.uniform(0, size, n)
    sig = rng.uniform(8, 64, n)
    amp = rng.uniform(200, 1500, n)
    ax = np.arange(size, dtype=np.float64)
    gy = np.exp(-((ax[:, None] - cy[None, :]) ** 2) / (2 * sig[None, :] ** 2)) * amp[None, :]  # (H, n)
    gx = np.exp(-((ax[:, None] - cx[None, :]) ** 2) / (2 * sig[None, :] ** 2))  # (W, n)
    field = 1000.0 + gy @ gx.T + rng.normal(0, 20, (size, size))
    return np.clip(np.round(field), 0, 4095).astype(np.uint16)[None]


def _cubic_weights(t: np.ndarray) -> np.ndarray:
    """Catmull-Rom weights for fractional offsets t, shape (n, 4)."""
    t2, t3 = t * t, t * t * t
    return np.stack([
        -0.5 * t3 + t2 - 0.5 * t,
        1.5 * t3 - 2.5 * t2 + 1.0,
        -1.5 * t3 + 2.0 * t2 + 0.5 * t,
        0.5 * t3 - 0.5 * t2,
    ], axis=1)


def _upsample_matrix(n_out: int, cell: int, n_lat: int) -> np.ndarray:
    """(n_out, n_lat) matrix doing bicubic interpolation of a lattice with `cell` px spacing."""
    pos = np.arange(n_out, dtype=np.float64) / cell + 1.0
    i0 = np.floor(pos).astype(np.int64)
    w = _cubic_weights(pos - i0)
    m = np.zeros((n_out, n_lat), dtype=np.float64)
    rows = np.arange(n_out)
    for k in range(4):
        np.add.at(m, (rows, np.clip(i0 - 1 + k, 0, n_lat - 1)), w[:, k])
    return m


def cfg2_pathology(seed: int = 0, height: int = 2048, width: int = 2048, nuclei: int | None = None) -> np.ndarray:
    """(H,W,3) uint8 HWC pathology-like tile.

    White background 240 +- N(0,3); pink stroma RGB ~(220,150,180) where bicubic-upsampled
    Gaussian lattice noise (cell 128 px) exceeds 0.35; elliptical nuclei, radii U[4,12],
    RGB ~(90,60,140) +- 15 per nucleus.  400 nuclei per 2048^2 (density kept for other sizes).
    """
    rng = np.random.default_rng(seed)
    if nuclei is None:
        nuclei = int(round(400 * (height * width) / (2048 * 2048)))
    cell = 128
    lat_h, lat_w = height // cell + 4, width // cell + 4
    lattice = rng.normal(0, 1, (lat_h, lat_w))
    field = _upsample_matrix(height, cell, lat_h) @ lattice @ _upsample_matrix(width, cell, lat_w).T
    stroma = field > 0.35
    img = 240.0 + rng.normal(0, 3, (height, width, 3))
    stroma_rgb = np.array([220.0, 150.0, 180.0])
    tex = rng.normal(0, 6, (height, width, 1))
    img = np.where(stroma[:, :, None], stroma_rgb[None, None, :] + tex, img)
    cy = rng.uniform(0, height, nuclei)
    cx = rng.uniform(0, width, nuclei)
    ra = rng.uniform(4, 12, nuclei)
    rb = rng.uniform(4, 12, nuclei)
    th = rng.uniform(0, np.pi, nuclei)
    col = np.array([90.0, 60.0, 140.0])[None, :] + rng.uniform(-15, 15, (nuclei, 3))
    for i in range(nuclei):
        r = int(np.ceil(max(ra[i], rb[i]))) + 1
        y0, y1 = max(int(cy[i]) - r, 0), min(int(cy[i]) + r + 1, height)
        x0, x1 = max(int(cx[i]) - r, 0), min(int(cx[i]) + r + 1, width)
        if y0 >= y1 or x0 >= x1:
            continue
        yy, xx = np.mgrid[y0:y1, x0:x1]
        dy, dx = yy - cy[i], xx - cx[i]
        c, s = np.cos(th[i]), np.sin(th[i])
        u = (dx * c + dy * s) / ra[i]
        v = (-dx * s + dy * c) / rb[i]
        inside = (u * u + v * v) <= 1.0
        patch = img[y0:y1, x0:x1]
        patch[inside] = col[i][None, :] + rng.normal(0, 4, (int(inside.sum()), 3))
    return np.clip(np.round(img), 0, 255).astype(np.uint8)


def cfg4_tile(seed: int, tile_index: int, size: int = 4096) -> np.ndarray:
    """Tile `tile_index` (row-major in the 16x16 grid) of the whole-slide config: seed + index."""
    return cfg2_pathology(seed + tile_index, size, size)


def cfg5_fluorescence(seed: int = 0, size: int = 8192, channels: int = 4, spots: float = 5000.0) -> np.ndarray:
    """(C,H,W) uint16: background 300 + Poisson(5000) Gaussian spots (sigma 1.5-4, peak
    20000-60000) + N(0,1)*sqrt(signal), clipped to 0..65535."""
    rng = np.random.default_rng(seed)
    out = np.empty((channels, size, size), dtype=np.uint16)
    spots_scaled = spots * (size * size) / (8192 * 8192)
    for ch in range(channels):
        sig = np.full((size, size), 300.0)
        n = int(rng.poisson(spots_scaled))
        cy = rng.uniform(0, size, n)
        cx = rng.uniform(0, size, n)
        sg = rng.uniform(1.5, 4.0, n)
        pk = rng.uniform(20000, 60000, n)
        for i in range(n):
            r = int(np.ceil(4 * sg[i]))
            y0, y1 = max(int(cy[i]) - r, 0), min(int(cy[i]) + r + 1, size)
            x0, x1 = max(int(cx[i]) - r, 0), min(int(cx[i]) + r + 1, size)
            if y0 >= y1 or x0 >= x1:
                continue
            gy = np.exp(-((np.arange(y0, y1) - cy[i]) ** 2) / (2 * sg[i] ** 2))
            gx = np.exp(-((np.arange(x0, x1) - cx[i]) ** 2) / (2 * sg[i] ** 2))
            sig[y0:y1, x0:x1] += pk[i] * gy[:, None] * gx[None, :]
        noisy = sig + rng.standard_normal((size, size)) * np.sqrt(sig)
        out[ch] = np.clip(np.round(noisy), 0, 65535).astype(np.uint16)
    return out


def planar(img_hwc: np.ndarray) -> np.ndarray:
    """HWC -> CHW (what RasterImage.samples holds, transforms.py:26)."""
    return np.ascontiguousarray(np.moveaxis(img_hwc, -1, 0))


def psnr(a: np.ndarray, b: np.ndarray, peak: float) -> float:
    d = np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)
    mse = float(np.mean(d * d))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


# ------------------------------------------------------------------------------ GPU generator
def _upsample_matrix_torch(n_out: int, cell: int, n_lat: int, device):
    import torch
    m = torch.from_numpy(_upsample_matrix(n_out, cell, n_lat)).to(device=device, dtype=torch.float32)
    return m


def cfg2_pathology_torch(seed: int, height: int = 4096, width: int = 4096, device="cuda", out=None):
    """(H,W,3) uint8 pathology-like tile generated on the GPU (torch, seeded Philox).

    Same recipe and statistics as `cfg2_pathology` (white background 240 +- N(0,3); pink
    stroma ~(220,150,180) + N(0,6) where bicubic-upsampled lattice noise (cell 128 px) exceeds
    0.35; 400 nuclei per 2048^2 (elliptical, radii U[4,12], RGB ~(90,60,140) +- 15, + N(0,4)),
    later nuclei drawn over earlier ones), but not the same random stream: it exists so the
    whole-slide workload (BASELINE configs[3], 256 distinct 4096^2 tiles, 12.9 GB) can be
    generated in seconds on the device.  Parity of the codec on these tiles is checked against
    the CPU oracle on copies of the generated pixels (tests/test_gpu_slide.py).
    """
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    f32 = torch.float32
    nuclei = int(round(400 * (height * width) / (2048 * 2048)))
    cell = 128
    lat_h, lat_w = height // cell + 4, width // cell + 4
    lattice = torch.randn((lat_h, lat_w), generator=g, device=device, dtype=f32)
    field = _upsample_matrix_torch(height, cell, lat_h, device) @ lattice @ _upsample_matrix_torch(width, cell, lat_w,
                                                                                                   device).T
    stroma = (field > 0.35).unsqueeze(-1)
    img = 240.0 + 3.0 * torch.randn((height, width, 3), generator=g, device=device, dtype=f32)
    tex = 6.0 * torch.randn((height, width, 1), generator=g, device=device, dtype=f32)
    srgb = torch.tensor([220.0, 150.0, 180.0], device=device, dtype=f32)
    img = torch.where(stroma, srgb + tex, img)
    # nuclei: every pixel takes the last (highest index) nucleus covering it
    u = torch.rand((nuclei, 6), generator=g, device=device, dtype=torch.float64)
    cy, cx = u[:, 0] * height, u[:, 1] * width
    ra, rb = 4 + 8 * u[:, 2], 4 + 8 * u[:, 3]
    th = u[:, 4] * np.pi
    col = torch.tensor([90.0, 60.0, 140.0], device=device, dtype=f32) + \
        (torch.rand((nuclei, 3), generator=g, device=device, dtype=f32) * 30 - 15)
    R = 13  # ceil(max radius) + 1
    d = torch.arange(-R, R + 1, device=device)
    yy = cy.floor().long()[:, None, None] + d[None, :, None]
    xx = cx.floor().long()[:, None, None] + d[None, None, :]
    dy, dx = yy.double() - cy[:, None, None], xx.double() - cx[:, None, None]
    c, s = torch.cos(th)[:, None, None], torch.sin(th)[:, None, None]
    uu = (dx * c + dy * s) / ra[:, None, None]
    vv = (-dx * s + dy * c) / rb[:, None, None]
    inside = (uu * uu + vv * vv <= 1.0) & (yy >= 0) & (yy < height) & (xx >= 0) & (xx < width)
    idx = torch.arange(nuclei, device=device)[:, None, None].expand_as(inside)
    flat = (yy.clamp(0, height - 1) * width + xx.clamp(0, width - 1))[inside]
    owner = torch.full((height * width,), -1, dtype=torch.long, device=device)
    owner.scatter_reduce_(0, flat, idx[inside], reduce="amax")
    owner = owner.view(height, width)
    noise = 4.0 * torch.randn((height, width, 3), generator=g, device=device, dtype=f32)
    has = (owner >= 0).unsqueeze(-1)
    img = torch.where(has, col[owner.clamp_min(0)] + noise, img)
    res = img.round_().clamp_(0, 255).to(torch.uint8)
    if out is not None:
        out.copy_(res)
        return out
    return res


def cfg4_tile_torch(seed: int, tile_index: int, size: int = 4096, device="cuda", out=None):
    """Tile `tile_index` of the whole-slide config on the GPU: seed + index (cfg2 generator)."""
    return cfg2_pathology_torch(seed + tile_index, size, size, device, out)
