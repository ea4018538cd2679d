"""BASELINE.json configurations C1..C5 as concrete, seeded input recipes.

The recipes follow SURVEY.md Sec. 8(d) "Concrete synthetic inputs"; the paper
itself never states its grid or model (reading c14).
Every derived quantity a run needs (float32 weights, dt) is produced here once
and handed to both the library and the oracle, which never recompute them.
"""
from __future__ import annotations

import math

import numpy as np

from . import weights as W
from .fields import model_max

RICKER_F = 15.0  # Hz, "with f=15Hz"


def _base(name, nx, ny, nz, r_xy, r_z, model, steps, dz=(10.0, 10.0), t0=None,
          damp_width=20, src=None, mask=1, notes=""):
    return dict(
        name=name, nx=nx, ny=ny, nz=nz, r_xy=r_xy, r_z=r_z, h=10.0,
        dz=dz, model=model, steps=steps, damp_width=damp_width, damp_alpha=0.015,
        src=src if src is not None else (nx // 2, ny // 2, nz // 2),
        f=RICKER_F, t0=(1.0 / RICKER_F) if t0 is None else t0, amp=1.0, mask=mask,
        notes=notes,
    )


def homogeneous(vz=3000.0, eps=0.2, delta=0.1):
    return dict(kind="homogeneous", vz=vz, eps=eps, delta=delta)


def layered(n_layers=8, seed=1410, isotropic=False):
    return dict(kind="layered", n_layers=n_layers, seed=seed, vz_top=1500.0,
                vz_bottom=4500.0, eps_max=0.25, delta_max=0.12, isotropic=isotropic)


def C1():
    return _base("C1", 64, 64, 64, 4, 4, homogeneous(), 100, t0=0.0, src=(32, 32, 32),
                 notes="64^3 homogeneous VTI eps=0.2 delta=0.1, 100 steps, 1 GPU vs oracle")


def C2():
    return _base("C2", 512, 512, 512, 4, 4, layered(8), 1000, dz=(5.0, 15.0),
                 notes="512^3 layered VTI, variable dz, W=20, 1000 steps, 1 B200")


def C3():
    return _base("C3", 1024, 1024, 512, 8, 4, layered(8), 500, dz=(5.0, 15.0),
                 notes="1024x1024x512, R_xy=8 R_z=4, 500 steps, 1/2/4/8 y-slabs")


def C4():
    return _base("C4", 2048, 2048, 1024, 4, 4, layered(12), 200, dz=(5.0, 15.0),
                 notes="2048x2048x1024 paper-benchmark-shaped, 200 steps, strong scaling")


def C5(n_gpus=1):
    return _base("C5", 1024, 1024 * n_gpus, 1024, 6, 6, layered(8, isotropic=True), 200,
                 dz=(5.0, 15.0), notes="1024^3 per GPU, R=6/6, eps=delta=0, weak scaling")


def N1():
    """the paper's benchmark radii R_xy=12, R_z=8 ("92 flops per
    point", 1000 steps) on the C2 grid and model (the paper
    states no grid)."""
    return _base("N1", 512, 512, 512, 12, 8, layered(8), 1000, dz=(5.0, 15.0),
                 notes="paper benchmark radii (12,8) on the C2 512^3 layered model, 1000 steps")


CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5, "N1": N1}


def scaled(cfg: dict, nx=None, ny=None, nz=None, steps=None, **kw) -> dict:
    """Same recipe on a different grid (source re-centred unless given)."""
    c = dict(cfg)
    c["nx"] = nx or cfg["nx"]
    c["ny"] = ny or cfg["ny"]
    c["nz"] = nz or cfg["nz"]
    if steps is not None:
        c["steps"] = steps
    c["src"] = kw.pop("src", (c["nx"] // 2, c["ny"] // 2, c["nz"] // 2))
    c.update(kw)
    return c


def weights_f32(cfg: dict):
    """(w_xy float32[R+1], w_z float32[nz][2Rz+1], z_coords float64)."""
    wxy = W.xy_weights(cfg["r_xy"]).astype(np.float32)
    zc = W.z_coords_ramp(cfg["nz"], cfg["r_z"], cfg["dz"][0], cfg["dz"][1])
    wz = W.z_weights(zc, cfg["r_z"]).astype(np.float32)
    return wxy, np.ascontiguousarray(wz), zc


def stable_dt(cfg: dict, wxy=None, wz=None, safety=0.9) -> float:
    """dt = safety * Gershgorin bound (reading c11), as float32.

    dt_max = 2 / sqrt(max(vx2, vn2) * S_xy / h^2 + max(vz2) * S_z) with
    S_xy = |w0| + 4 sum_l |w_l| and S_z = max_k sum_l |w^z_{k,l}|. Model
    maxima are the recipe's analytic upper bounds, so the value is cheap and
    identical for every rank and for the oracle.
    """
    if wxy is None or wz is None:
        wxy, wz, _ = weights_f32(cfg)
    wxy = np.asarray(wxy, dtype=np.float64)
    wz = np.asarray(wz, dtype=np.float64)
    s_xy = abs(wxy[0]) + 4.0 * np.abs(wxy[1:]).sum()
    s_z = np.abs(wz).sum(axis=1).max()
    vx2, vn2, vz2 = model_max(cfg)
    rho = max(vx2, vn2) * s_xy / (cfg["h"] ** 2) + vz2 * s_z
    dt = safety * 2.0 / math.sqrt(rho)
    return float(np.float32(dt))
