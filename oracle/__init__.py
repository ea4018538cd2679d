"""CPU oracle for the VTI step -- TEST INFRASTRUCTURE ONLY.

Only tests/, tools/oracle_digests.py (writes tests/golden/ digests),
__graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this package. The product path
(paper_1410_1387_b200 + include/vti.h) never imports it, and this package
never imports the product. The arithmetic lives in ``vti_oracle.c`` (plain C
loops, see its header for the paper passages and readings it follows); this
module is argument marshalling plus the build step.

Pins (tests/test_oracle_*.py) tie it to things other than itself: exact
rational weights, polynomial exactness of the operators, early-step closed
forms, the isotropic p == q collapse and an independent acoustic solver,
mirror symmetry, a dense-operator brute force on an 8^3 grid, Ricker and
Cerjan closed forms.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "vti_oracle.c")
LIB = os.path.join(HERE, "libvti_oracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
          "-Wall", "-Wextra"]


class Params(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("r_xy", C.c_int32), ("r_z", C.c_int32),
        ("h", C.c_double), ("dt", C.c_double),
        ("damp_width", C.c_int32), ("damp_alpha", C.c_double),
        ("src_i", C.c_int32), ("src_j", C.c_int32), ("src_k", C.c_int32),
        ("src_f", C.c_double), ("src_t0", C.c_double), ("src_amp", C.c_double),
        ("src_mask", C.c_int32),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc; no GPU needed)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.check_call(["gcc", *CFLAGS, SRC, "-o", tmp, "-lm"])
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        fp = lambda t: np.ctypeslib.ndpointer(dtype=t, flags="C_CONTIGUOUS")
        for sfx, t in (("f32", np.float32), ("f64", np.float64)):
            f = getattr(L, "vto_run_" + sfx)
            f.restype = C.c_int
            f.argtypes = [C.POINTER(Params), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t),
                          fp(t), fp(t), C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
            g = getattr(L, "vto_point_" + sfx)
            g.restype = C.c_int
            ct = C.c_float if t is np.float32 else C.c_double
            g.argtypes = [C.POINTER(Params), fp(t), fp(t), C.c_int32, C.c_int32, C.c_int32,
                          C.c_int64, fp(t), fp(t), ct, ct, ct, ct, ct, fp(t)]
            x = getattr(L, "vto_run_ex_" + sfx)
            x.restype = C.c_int
            i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
            x.argtypes = [C.POINTER(Params), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t),
                          fp(t), fp(t), C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                          C.c_int32, i32, C.c_int32, C.c_int32, C.c_int64, fp(t),
                          C.c_int32, i32, C.c_int32, fp(t), C.POINTER(C.c_double)]
            a = getattr(L, "vto_adjoint_ex_" + sfx)
            a.restype = C.c_int
            a.argtypes = [C.POINTER(Params), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t),
                          fp(t), fp(t), C.c_int64, C.c_int32, C.c_int32,
                          C.c_int32, i32, C.c_int32, C.c_int32, C.c_int64, fp(t),
                          C.c_int32, i32, C.c_int32, fp(t)]
            w = getattr(L, "vto_step_planes_" + sfx)
            w.restype = C.c_int
            w.argtypes = [C.POINTER(Params), fp(t), fp(t), C.c_int32, C.c_int32, C.c_int64,
                          fp(t), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t), fp(t)]
        L.vto_ricker.restype = C.c_double
        L.vto_ricker.argtypes = [C.c_double, C.c_double, C.c_double]
        L.vto_damping.restype = C.c_double
        L.vto_damping.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double]
        L.vto_damping_profile_f32.restype = None
        L.vto_damping_profile_f32.argtypes = [C.c_int32, C.c_int32, C.c_double, fp(np.float32)]
        L.vto_max_threads.restype = C.c_int
        _lib = L
    return _lib


_FROM_CFG = object()


def params(cfg: dict, dt: float, src=_FROM_CFG, mask=None, damp_width=None) -> Params:
    """Oracle parameters; ``src`` defaults to cfg["src"], ``src=None`` means no source."""
    s = cfg.get("src") if src is _FROM_CFG else src
    return Params(
        nx=cfg["nx"], ny=cfg["ny"], nz=cfg["nz"], r_xy=cfg["r_xy"], r_z=cfg["r_z"],
        h=cfg["h"], dt=float(np.float32(dt)),
        damp_width=cfg["damp_width"] if damp_width is None else damp_width,
        damp_alpha=cfg["damp_alpha"],
        src_i=-1 if s is None else s[0], src_j=-1 if s is None else s[1],
        src_k=-1 if s is None else s[2],
        src_f=cfg["f"], src_t0=cfg["t0"], src_amp=cfg["amp"],
        src_mask=cfg["mask"] if mask is None else mask,
    )


def run(P: Params, wxy, wz, vx2, vn2, vz2, state=None, n0: int = 0, nsteps: int = 1,
        dtype=np.float32, nthreads: int = 0):
    """Advance nsteps from level n0. Returns (p, q, pm, qm, seconds).

    ``state`` = (p, q, pm, qm) at levels (n0, n0-1) in [z][y][x]; None = zero.
    """
    shape = (P.nz, P.ny, P.nx)
    conv = lambda a: np.ascontiguousarray(np.asarray(a, dtype=dtype))
    if state is None:
        p, q, pm, qm = (np.zeros(shape, dtype=dtype) for _ in range(4))
    else:
        p, q, pm, qm = (conv(a).copy() for a in state)
    for a in (p, q, pm, qm):
        assert a.shape == shape
    vx2, vn2, vz2 = (conv(a).reshape(shape) for a in (vx2, vn2, vz2))
    wxy = conv(wxy).reshape(-1)
    wz = conv(wz).reshape(-1)
    assert wxy.size == P.r_xy + 1 and wz.size == P.nz * (2 * P.r_z + 1)
    secs = C.c_double(0.0)
    f = lib().vto_run_f32 if dtype == np.float32 else lib().vto_run_f64
    rc = f(C.byref(P), wxy, wz, vx2, vn2, vz2, p, q, pm, qm, n0, nsteps, nthreads, C.byref(secs))
    if rc != 0:
        raise ValueError(f"oracle rejected parameters (code {rc})")
    return p, q, pm, qm, secs.value


def run_ex(P: Params, wxy, wz, vx2, vn2, vz2, state=None, n0: int = 0, nsteps: int = 1,
           direction: int = 1, inj=None, rec=None, dtype=np.float32, nthreads: int = 0):
    """run() with time direction, trace injection and receivers.

    inj = (ijk [n][3] int, mask, t_first, traces [nt][n]) or None;
    rec = (ijk [m][3] int, mask) or None. direction = -1: state = (u^n, u^{n+1}) and the
    time index runs n0, n0-1, ... Returns (p, q, pm, qm, rec_traces [nsteps][m][nf] or None, s).
    """
    shape = (P.nz, P.ny, P.nx)
    conv = lambda a: np.ascontiguousarray(np.asarray(a, dtype=dtype))
    if state is None:
        p, q, pm, qm = (np.zeros(shape, dtype=dtype) for _ in range(4))
    else:
        p, q, pm, qm = (conv(a).copy() for a in state)
    vx2, vn2, vz2 = (conv(a).reshape(shape) for a in (vx2, vn2, vz2))
    wxy = conv(wxy).reshape(-1)
    wz = conv(wz).reshape(-1)
    dummy_i = np.zeros(3, np.int32)
    dummy_t = np.zeros(1, dtype)
    if inj is not None:
        ijk, imask, t_first, tr = inj
        ijk = np.ascontiguousarray(np.asarray(ijk, np.int32).reshape(-1, 3))
        tr = conv(tr).reshape(-1, ijk.shape[0])
        n_inj, nt = ijk.shape[0], tr.shape[0]
    else:
        ijk, imask, t_first, tr, n_inj, nt = dummy_i, 0, 0, dummy_t, 0, 0
    if rec is not None:
        rijk, rmask = rec
        rijk = np.ascontiguousarray(np.asarray(rijk, np.int32).reshape(-1, 3))
        n_rec = rijk.shape[0]
        nf = (rmask & 1) + ((rmask >> 1) & 1)
        out = np.zeros((nsteps, n_rec, nf), dtype=dtype)
    else:
        rijk, rmask, n_rec, out = dummy_i, 0, 0, dummy_t
    secs = C.c_double(0.0)
    f = lib().vto_run_ex_f32 if dtype == np.float32 else lib().vto_run_ex_f64
    rc = f(C.byref(P), wxy, wz, vx2, vn2, vz2, p, q, pm, qm, n0, nsteps, direction, nthreads,
           n_inj, ijk.reshape(-1) if n_inj else dummy_i, imask, nt, t_first, tr.reshape(-1) if n_inj else dummy_t,
           n_rec, rijk.reshape(-1) if n_rec else dummy_i, rmask, out.reshape(-1) if n_rec else dummy_t,
           C.byref(secs))
    if rc != 0:
        raise ValueError(f"oracle rejected parameters (code {rc})")
    return p, q, pm, qm, (out if n_rec else None), secs.value


def adjoint_ex(P: Params, wxy, wz, vx2, vn2, vz2, state, m0: int = 0, nsteps: int = 1, inj=None, rec=None,
               dtype=np.float32, nthreads: int = 0):
    """The adjoint (transpose) recurrence of the scheme (see vto_adjoint_ex in vti_oracle.c).

    state = (psi_p^m0, psi_q^m0, psi_p^{m0+1}, psi_q^{m0+1}); the time index runs m0, m0-1, ...
    inj / rec as in run_ex (P's Ricker source is not used). Returns (p, q, pm, qm, rec_traces).
    """
    shape = (P.nz, P.ny, P.nx)
    conv = lambda a: np.ascontiguousarray(np.asarray(a, dtype=dtype))
    p, q, pm, qm = (conv(a).copy() for a in state)
    vx2, vn2, vz2 = (conv(a).reshape(shape) for a in (vx2, vn2, vz2))
    wxy = conv(wxy).reshape(-1)
    wz = conv(wz).reshape(-1)
    dummy_i = np.zeros(3, np.int32)
    dummy_t = np.zeros(1, dtype)
    if inj is not None:
        ijk, imask, t_first, tr = inj
        ijk = np.ascontiguousarray(np.asarray(ijk, np.int32).reshape(-1, 3))
        tr = conv(tr).reshape(-1, ijk.shape[0])
        n_inj, nt = ijk.shape[0], tr.shape[0]
    else:
        ijk, imask, t_first, tr, n_inj, nt = dummy_i, 0, 0, dummy_t, 0, 0
    if rec is not None:
        rijk, rmask = rec
        rijk = np.ascontiguousarray(np.asarray(rijk, np.int32).reshape(-1, 3))
        n_rec = rijk.shape[0]
        out = np.zeros((nsteps, n_rec, (rmask & 1) + ((rmask >> 1) & 1)), dtype=dtype)
    else:
        rijk, rmask, n_rec, out = dummy_i, 0, 0, dummy_t
    f = lib().vto_adjoint_ex_f32 if dtype == np.float32 else lib().vto_adjoint_ex_f64
    rc = f(C.byref(P), wxy, wz, vx2, vn2, vz2, p, q, pm, qm, m0, nsteps, nthreads,
           n_inj, ijk.reshape(-1) if n_inj else dummy_i, imask, nt, t_first, tr.reshape(-1) if n_inj else dummy_t,
           n_rec, rijk.reshape(-1) if n_rec else dummy_i, rmask, out.reshape(-1) if n_rec else dummy_t)
    if rc != 0:
        raise ValueError(f"oracle rejected parameters (code {rc})")
    return p, q, pm, qm, (out if n_rec else None)


def point(P: Params, wxy, wzrow, i, j, k, n, pc, qc, pm, qm, vx2, vn2, vz2, dtype=np.float32):
    """One output point of step n from gathered neighbourhoods (see vti_oracle.c)."""
    conv = lambda a: np.ascontiguousarray(np.asarray(a, dtype=dtype)).reshape(-1)
    out = np.zeros(2, dtype=dtype)
    f = lib().vto_point_f32 if dtype == np.float32 else lib().vto_point_f64
    rc = f(C.byref(P), conv(wxy), conv(wzrow), i, j, k, n, conv(pc), conv(qc),
           float(pm), float(qm), float(vx2), float(vn2), float(vz2), out)
    if rc != 0:
        raise ValueError(f"oracle rejected parameters (code {rc})")
    return out[0], out[1]


def step_planes(P: Params, wxy, wz, k0: int, p, q, pm, qm, vx2, vn2, vz2, n: int = 0,
                dtype=np.float32):
    """One step (level n -> n+1) of planes [k0, k0+nk) of the global grid P from plane windows.

    p, pm, qm, vx2, vn2, vz2: [nk][ny][nx] (planes k0..); q: [nk+2Rz][ny][nx] (planes
    k0-Rz..; planes outside the grid are ignored = zero exterior); wz: the full
    [nz][2Rz+1] table. Returns (p^{n+1}, q^{n+1}) on those planes (see vti_oracle.c).
    """
    conv = lambda a: np.ascontiguousarray(np.asarray(a, dtype=dtype))
    p, pm, qm, vx2, vn2, vz2 = (conv(a) for a in (p, pm, qm, vx2, vn2, vz2))
    q = conv(q)
    nk = p.shape[0]
    shape = (nk, P.ny, P.nx)
    for a in (p, pm, qm, vx2, vn2, vz2):
        assert a.shape == shape, (a.shape, shape)
    assert q.shape == (nk + 2 * P.r_z, P.ny, P.nx)
    wxy = conv(wxy).reshape(-1)
    wz = conv(wz).reshape(-1)
    assert wxy.size == P.r_xy + 1 and wz.size == P.nz * (2 * P.r_z + 1)
    pn = np.empty(shape, dtype=dtype)
    qn = np.empty(shape, dtype=dtype)
    f = lib().vto_step_planes_f32 if dtype == np.float32 else lib().vto_step_planes_f64
    rc = f(C.byref(P), wxy, wz, k0, nk, n, p, q, pm, qm, vx2, vn2, vz2, pn, qn)
    if rc != 0:
        raise ValueError(f"oracle rejected parameters (code {rc})")
    return pn, qn


def ricker(t, f, t0):
    return lib().vto_ricker(t, f, t0)


def damping_profile(n, W, alpha):
    out = np.zeros(n, dtype=np.float32)
    lib().vto_damping_profile_f32(n, W, alpha, out)
    return out


def max_threads() -> int:
    return lib().vto_max_threads()
