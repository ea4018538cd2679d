"""Seeded synthetic inputs: counter-based random fields and layered VTI models.

Input generation only -- none of the method's arithmetic (no stencil, no
update, no Ricker, no damping) lives here. Everything is generated from a
counter-based integer hash plus IEEE + - * / in float64, so the same call on a
CPU tensor and on a CUDA tensor returns bit-identical float32 data; this lets
the bench build full-size inputs on the GPU while the oracle recomputes any
sampled neighbourhood on the host (SURVEY.md Sec. 8(d) "Concrete synthetic
inputs").

Layout of every returned field is the user layout of the C ABI: [z][y][x],
x fastest.
"""
from __future__ import annotations

import torch

_M32 = 0xFFFFFFFF


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for int64 x in [0, 2^32) without int64 overflow."""
    lo = c & 0xFFFF
    hi = (c >> 16) & 0xFFFF
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _M32


def hash32(x: torch.Tensor) -> torch.Tensor:
    """'lowbias32' integer mixer on int64 tensors holding uint32 values."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _hash_int(v: int) -> int:
    return int(hash32(torch.tensor([v & _M32], dtype=torch.int64))[0])


def stream_key(seed: int, stream: int) -> int:
    return _hash_int(_hash_int(seed) ^ (stream * 0x9E3779B9 & _M32))


def uniform01(idx: torch.Tensor, seed: int, stream: int) -> torch.Tensor:
    """float32 in [0,1), multiples of 2^-24, a pure function of (seed, stream, idx)."""
    key = stream_key(seed, stream)
    lo = idx & _M32
    hi = idx >> 32
    h = hash32(lo ^ key)
    h = hash32(h ^ hash32(hi + 0x68E31DA4))
    return (h >> 8).to(torch.float32) * (1.0 / 16777216.0)


def random_planes(nx: int, ny: int, k0: int, nk: int, seed: int, stream: int,
                  amp: float, device="cpu", j0: int = 0, nyl: int | None = None,
                  ny_glob: int | None = None) -> torch.Tensor:
    """Uniform(-amp, amp) float32 values on planes k0..k0+nk-1, rows j0..j0+nyl-1.

    The value at global point (i, j, k) depends only on (seed, stream,
    (k*ny_glob + j)*nx + i), so any slab or sample reproduces the same data.
    """
    nyl = ny - j0 if nyl is None else nyl
    ny_glob = ny if ny_glob is None else ny_glob
    k = torch.arange(k0, k0 + nk, device=device, dtype=torch.int64).view(nk, 1, 1)
    j = torch.arange(j0, j0 + nyl, device=device, dtype=torch.int64).view(1, nyl, 1)
    i = torch.arange(nx, device=device, dtype=torch.int64).view(1, 1, nx)
    idx = (k * ny_glob + j) * nx + i
    u = uniform01(idx, seed, stream)
    a = torch.tensor(amp, dtype=torch.float32, device=device)
    return (u * 2.0 - 1.0) * a


def random_at(i: torch.Tensor, j: torch.Tensor, k: torch.Tensor, nx: int, ny_glob: int,
              seed: int, stream: int, amp: float) -> torch.Tensor:
    """Same values as ``random_planes`` at explicit global indices (int64 tensors)."""
    idx = (k * ny_glob + j) * nx + i
    u = uniform01(idx, seed, stream)
    a = torch.tensor(amp, dtype=torch.float32, device=idx.device)
    return (u * 2.0 - 1.0) * a


def _smooth2d(i: torch.Tensor, j: torch.Tensor, seed: int, stream: int, cell: int) -> torch.Tensor:
    """Smooth field in [-1, 1] (float64): smoothstep-bilinear lattice noise.

    Only + - * on float64 and integer hashing: bitwise reproducible across devices.
    """
    ci = torch.div(i, cell, rounding_mode="floor")
    cj = torch.div(j, cell, rounding_mode="floor")
    fx = (i - ci * cell).to(torch.float64) / float(cell)
    fy = (j - cj * cell).to(torch.float64) / float(cell)
    sx = fx * fx * (3.0 - 2.0 * fx)
    sy = fy * fy * (3.0 - 2.0 * fy)

    def node(a, b):
        u = uniform01(a * 1048576 + b, seed, stream).to(torch.float64)
        return u * 2.0 - 1.0

    v00 = node(ci, cj)
    v10 = node(ci + 1, cj)
    v01 = node(ci, cj + 1)
    v11 = node(ci + 1, cj + 1)
    return (v00 * (1.0 - sx) + v10 * sx) * (1.0 - sy) + (v01 * (1.0 - sx) + v11 * sx) * sy


def layer_table(n_layers: int, seed: int, vz_top: float, vz_bottom: float,
                eps_max: float, delta_max: float, isotropic: bool):
    """Per-layer (vz, eps, delta): vz increases with depth; eps >= delta >= 0.

    eps >= delta keeps the 2x2 block operator stable.
    """
    g = torch.Generator().manual_seed(seed)
    out = []
    for l in range(n_layers):
        vz = vz_top + (vz_bottom - vz_top) * (l / max(1, n_layers - 1))
        if isotropic:
            eps, delta = 0.0, 0.0
        else:
            u1, u2 = torch.rand(2, generator=g, dtype=torch.float64).tolist()
            eps = eps_max * u1
            delta = min(delta_max, eps) * u2
        out.append((vz, eps, delta))
    return out


def _model_from_layers(layer_idx: torch.Tensor, lateral: torch.Tensor, table):
    dev = layer_idx.device
    vz = torch.tensor([t[0] for t in table], dtype=torch.float64, device=dev)
    eps = torch.tensor([t[1] for t in table], dtype=torch.float64, device=dev)
    dl = torch.tensor([t[2] for t in table], dtype=torch.float64, device=dev)
    vz_l = vz[layer_idx]
    vz2 = (vz_l * vz_l * (1.0 + 0.02 * lateral)).to(torch.float32)
    vz2d = vz2.to(torch.float64)
    vx2 = (vz2d * (1.0 + 2.0 * eps[layer_idx])).to(torch.float32)
    vn2 = (vz2d * (1.0 + 2.0 * dl[layer_idx])).to(torch.float32)
    return vx2, vn2, vz2


def _layer_index(i, j, k, nz, m):
    nl = m["n_layers"]
    layer_idx = torch.zeros(torch.broadcast_shapes(i.shape, j.shape, k.shape),
                            dtype=torch.int64, device=k.device)
    for l in range(1, nl):
        base = (l * nz) // nl
        d = torch.round(3.0 * _smooth2d(i, j, m["seed"], 100 + l, 64)).to(torch.int64)
        layer_idx = layer_idx + (k >= base + d).to(torch.int64)
    return layer_idx


def layered_model_at(i, j, k, nx, ny_glob, nz, m: dict):
    """(vx2, vn2, vz2) float32 of the layered VTI recipe at explicit global indices.

    i, j, k are broadcastable int64 tensors; the lateral fields depend on (i, j)
    only, so [1][ny][nx] index grids against a [nk][1][1] k grid are cheap.
    """
    table = layer_table(m["n_layers"], m["seed"], m["vz_top"], m["vz_bottom"],
                        m["eps_max"], m["delta_max"], m.get("isotropic", False))
    layer_idx = _layer_index(i, j, k, nz, m)
    lateral = _smooth2d(i, j, m["seed"], 7, 128)
    return _model_from_layers(layer_idx, lateral, table)


def model_planes(cfg: dict, k0: int, nk: int, device="cpu", j0: int = 0,
                 nyl: int | None = None):
    """(vx2, vn2, vz2) float32 [nk][nyl][nx] for planes k0.. and global rows j0.."""
    nx, ny, nz = cfg["nx"], cfg["ny"], cfg["nz"]
    nyl = ny - j0 if nyl is None else nyl
    m = cfg["model"]
    if m["kind"] == "homogeneous":
        vz2 = float(torch.tensor(m["vz"] * m["vz"], dtype=torch.float64).to(torch.float32))
        vx2 = float(torch.tensor(vz2 * (1.0 + 2.0 * m["eps"]), dtype=torch.float64).to(torch.float32))
        vn2 = float(torch.tensor(vz2 * (1.0 + 2.0 * m["delta"]), dtype=torch.float64).to(torch.float32))
        shape = (nk, nyl, nx)
        mk = lambda v: torch.full(shape, v, dtype=torch.float32, device=device)
        return mk(vx2), mk(vn2), mk(vz2)
    k = torch.arange(k0, k0 + nk, device=device, dtype=torch.int64).view(nk, 1, 1)
    j = torch.arange(j0, j0 + nyl, device=device, dtype=torch.int64).view(1, nyl, 1)
    i = torch.arange(nx, device=device, dtype=torch.int64).view(1, 1, nx)
    return layered_model_at(i, j, k, nx, ny, nz, m)


def model_max(cfg: dict):
    """Upper bounds (max vx2, max vn2, max vz2) used only for the dt choice."""
    m = cfg["model"]
    if m["kind"] == "homogeneous":
        vx2, vn2, vz2 = model_planes(dict(cfg, nx=1, ny=1, nz=1), 0, 1)
        return float(vx2.max()), float(vn2.max()), float(vz2.max())
    table = layer_table(m["n_layers"], m["seed"], m["vz_top"], m["vz_bottom"],
                        m["eps_max"], m["delta_max"], m.get("isotropic", False))
    vz2 = max(t[0] ** 2 for t in table) * 1.02
    vx2 = max(t[0] ** 2 * (1 + 2 * t[1]) for t in table) * 1.02
    vn2 = max(t[0] ** 2 * (1 + 2 * t[2]) for t in table) * 1.02
    return vx2, vn2, vz2
