#!/usr/bin/env python
"""Small cases through the C ABI for compute-sanitizer (memcheck / racecheck /
synccheck): every compiled radius pair and tile variant on a ragged grid with
a source, damping and a random state, then adjoint steps (the TMA one-pass and
chained two-pass forms), plus 2-slab local groups (forward and adjoint) and
fp64. No oracle: the sanitizer is the check; the script exits non-zero on any
library error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from synth import fields as SF  # noqa: E402
from paper_1410_1387_b200 import VTI, group_step  # noqa: E402
from synth import weights as W  # noqa: E402


def case(r, rz, nx=70, ny=37, nz=None, nranks=1, prec=32):
    nz = nz or 2 * rz + 9
    cfg = synth.scaled(synth.CONFIGS["C2"](), nx, ny, nz, r_xy=r, r_z=rz, damp_width=4, dz=(6.0, 12.0))
    wxy, wz, _ = synth.weights_f32(cfg)
    dt = synth.stable_dt(cfg, wxy, wz)
    dtype = np.float32 if prec == 32 else np.float64
    if prec == 64:
        wxy = W.xy_weights(r)
        wz = np.ascontiguousarray(W.z_weights(W.z_coords_ramp(nz, rz, 6.0, 12.0), rz))
    model = [a.numpy().astype(dtype) for a in SF.model_planes(cfg, 0, nz)]
    st = [SF.random_planes(nx, ny, 0, nz, 3, s, 1e-3).numpy().astype(dtype) for s in range(4)]
    hs = [VTI(nx, ny, nz, cfg["h"], r, rz, dt, wxy, wz, damp_width=4, rank=k, nranks=nranks, precision=prec)
          for k in range(nranks)]
    for h in hs:
        sl = slice(h.y0, h.y0 + h.ny_local)
        h.set_model(*[np.ascontiguousarray(a[:, sl]) for a in model])
        h.set_fields(*[np.ascontiguousarray(a[:, sl]) for a in st])
        h.add_source(nx // 2, ny // 2, nz // 2, t0=0.01)
    if nranks == 1:
        hs[0].step(3)
        hs[0].step_adjoint(3)
    else:
        group_step(hs, 3)
        group_step(hs, 3, transport="adjoint")
    for h in hs:
        p, q = h.get_fields(0)
        assert np.isfinite(p).all() and np.isfinite(q).all()
        h.close()


if __name__ == "__main__":
    for ty, wp in ((32, -1), (16, -1), (32, 0), (32, 1)):
        os.environ["VTI_TY"] = str(ty)
        os.environ["VTI_WP"] = str(wp)
        for r, rz in ((4, 4), (8, 4), (6, 6), (12, 8)):
            case(r, rz)
    os.environ.pop("VTI_TY")
    os.environ.pop("VTI_WP")
    case(4, 4, ny=70, nranks=2)
    case(12, 8, ny=70, nranks=2)
    for r, rz in ((4, 4), (8, 4), (6, 6), (12, 8)):
        case(r, rz, nx=130, ny=45, nz=2 * rz + 20, prec=64)
        case(r, rz, nx=130, ny=45, nz=2 * rz + 20)
    print("sanitize cases ok")
