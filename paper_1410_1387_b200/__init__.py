"""B200-native VTI propagator step (arXiv 1410.1387) -- Python binding.

Argument marshalling only: every step of the path runs in libvti.so
(include/vti.h), built for sm_100a by ``paper_1410_1387_b200._build``. There
is no CPU fallback: if the library is missing, importing this package raises.

Raw C-ABI functions are re-exported under their C names (``vti_create``,
``vti_step`` ...); the ``VTI`` class wraps one handle. Arrays may be numpy
arrays (host) or torch tensors (host or CUDA), float32, C-contiguous, in the
user layout [z][y][x] of this rank's y-slab.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB, build  # noqa: F401

__all__ = ["VTI", "VTIError", "Config", "Info", "TuneResult", "lib", "slab", "nccl_unique_id", "group_step"]

STATUS = {
    0: "VTI_OK", 1: "VTI_E_PARAM", 2: "VTI_E_GEOMETRY", 3: "VTI_E_MODEL", 4: "VTI_E_ANISO",
    5: "VTI_E_INSTABILITY", 6: "VTI_E_INDEX", 7: "VTI_E_CUDA", 8: "VTI_E_COMM", 9: "VTI_E_STATE",
    10: "VTI_E_UNSUPPORTED",
}
COMPILED_RADII = ((4, 4), (8, 4), (6, 6), (12, 8))


class VTIError(RuntimeError):
    """Non-OK vti_status from the library; .name is the status name, the message is vti_last_error()."""
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Config(C.Structure):
    """ctypes mirror of vti_config (include/vti.h)."""
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("h", C.c_double), ("r_xy", C.c_int32), ("r_z", C.c_int32), ("dt", C.c_double),
        ("damp_width", C.c_int32), ("damp_alpha", C.c_double), ("device", C.c_int32),
        ("stream", C.c_void_p), ("rank", C.c_int32), ("nranks", C.c_int32),
        ("nccl_id", C.c_void_p), ("check_every", C.c_int32), ("precision", C.c_int32),
    ]


class TuneResult(C.Structure):
    """ctypes mirror of vti_tune_result."""
    _fields_ = [("tile_y", C.c_int32), ("producer_warp", C.c_int32), ("rows_per_thread", C.c_int32),
                ("points_per_thread", C.c_int32), ("zchunk", C.c_int32),
                ("ms_per_step", C.c_float), ("candidates", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PlanInfo(C.Structure):
    """ctypes mirror of vti_plan_info."""
    _fields_ = [("y0", C.c_int32), ("ny_local", C.c_int32), ("ntx", C.c_int32), ("nty", C.c_int32),
                ("edge_lo", C.c_int32), ("edge_hi", C.c_int32), ("zchunk", C.c_int32),
                ("zchunk_edge", C.c_int32), ("zchunk_inner", C.c_int32), ("items", C.c_int32), ("grid", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Info(C.Structure):
    """ctypes mirror of vti_info."""
    _fields_ = [
        ("y0", C.c_int32), ("ny_local", C.c_int32), ("nx_pad", C.c_int32), ("layout", C.c_int32),
        ("tile_x", C.c_int32), ("tile_y", C.c_int32), ("rows_per_thread", C.c_int32), ("producer_warp", C.c_int32),
        ("points_per_thread", C.c_int32), ("small_kernel", C.c_int32), ("zchunk", C.c_int32), ("grid", C.c_int32),
        ("work_items", C.c_int32), ("launches_per_step", C.c_int32),
        ("device_bytes", C.c_int64), ("time_index", C.c_int64), ("steps_per_launch", C.c_int32),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB):
        raise ImportError(f"{LIB} is missing: run paper_1410_1387_b200._build.build() "
                          "(or __graft_entry__.build()); there is no fallback path")
    L = C.CDLL(LIB)
    H = C.c_void_p
    P = C.c_void_p
    st = C.c_int
    sig = {
        "vti_abi_version": (C.c_int32, []),
        "vti_status_string": (C.c_char_p, [st]),
        "vti_slab": (st, [C.POINTER(Config), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "vti_nccl_unique_id": (st, [P]),
        "vti_plan": (st, [C.POINTER(Config), C.c_int32, C.c_int32, C.c_int32, C.POINTER(PlanInfo)]),
        "vti_create": (st, [C.POINTER(H), C.POINTER(Config), P, P]),
        "vti_create_f64": (st, [C.POINTER(H), C.POINTER(Config), P, P]),
        "vti_set_model_f64": (st, [H, P, P, P]),
        "vti_set_model_planes_f64": (st, [H, C.c_int32, C.c_int32, P, P, P]),
        "vti_set_fields_f64": (st, [H, P, P, P, P, C.c_int64]),
        "vti_set_fields_planes_f64": (st, [H, C.c_int32, C.c_int32, P, P, P, P]),
        "vti_get_fields_f64": (st, [H, P, P, C.c_int32]),
        "vti_get_fields_planes_f64": (st, [H, C.c_int32, C.c_int32, P, P, C.c_int32]),
        "vti_set_model": (st, [H, P, P, P]),
        "vti_set_model_planes": (st, [H, C.c_int32, C.c_int32, P, P, P]),
        "vti_model_warnings": (C.c_int64, [H]),
        "vti_add_source": (st, [H, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                C.c_int32]),
        "vti_set_fields": (st, [H, P, P, P, P, C.c_int64]),
        "vti_set_fields_planes": (st, [H, C.c_int32, C.c_int32, P, P, P, P]),
        "vti_step": (st, [H, C.c_int32]),
        "vti_step_timed": (st, [H, C.c_int32, C.POINTER(C.c_float)]),
        "vti_group_step": (st, [C.POINTER(H), C.c_int32, C.c_int32]),
        "vti_group_step_staged": (st, [C.POINTER(H), C.c_int32, C.c_int32]),
        "vti_group_step_adjoint": (st, [C.POINTER(H), C.c_int32, C.c_int32]),
        "vti_get_fields": (st, [H, P, P, C.c_int32]),
        "vti_get_fields_planes": (st, [H, C.c_int32, C.c_int32, P, P, C.c_int32]),
        "vti_sync": (st, [H]),
        "vti_time_index": (C.c_int64, [H]),
        "vti_stream": (C.c_void_p, [H]),
        "vti_prepare": (st, [H]),
        "vti_query": (st, [H, C.POINTER(Info)]),
        "vti_set_tuning": (st, [H, C.c_int32, C.c_int32]),
        "vti_set_variant": (st, [H, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
        "vti_set_receivers": (st, [H, C.c_int32, P, C.c_int32, C.c_int32]),
        "vti_set_injection": (st, [H, C.c_int32, P, C.c_int32, C.c_int32, C.c_int64, P]),
        "vti_set_injection_f64": (st, [H, C.c_int32, P, C.c_int32, C.c_int32, C.c_int64, P]),
        "vti_receiver_info": (st, [H, C.POINTER(C.c_int32), C.POINTER(C.c_int32), P]),
        "vti_get_traces": (st, [H, P]),
        "vti_get_traces_f64": (st, [H, P]),
        "vti_reverse": (st, [H]),
        "vti_step_adjoint": (st, [H, C.c_int32]),
        "vti_snapshot_async": (st, [H, C.c_int32, C.c_int32, P, P, C.c_int32]),
        "vti_snapshot_async_f64": (st, [H, C.c_int32, C.c_int32, P, P, C.c_int32]),
        "vti_ipc_export": (st, [H, P]),
        "vti_ipc_connect": (st, [H, P, P]),
        "vti_halo_transport": (C.c_int32, [H]),
        "vti_debug_flags": (st, [H, P, P]),
        "vti_debug_halo": (st, [H, C.c_int32, C.c_int32, P]),
        "vti_debug_rows": (st, [H, C.c_int32, P]),
        "vti_direction": (C.c_int32, [H]),
        "vti_autotune": (st, [H, C.c_int32, C.POINTER(TuneResult)]),
        "vti_last_error": (C.c_char_p, [H]),
        "vti_destroy": (st, [H]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L, list(sig)


lib, EXPORTS = _load()
for _n in EXPORTS:
    globals()[_n] = getattr(lib, _n)


def _ptr(a, nelem: int | None = None, writable: bool = False, dtype=np.float32):
    """Raw pointer of a C-contiguous numpy array or torch tensor of ``dtype`` (None -> NULL)."""
    if a is None:
        return None, None
    try:
        import torch
        if isinstance(a, torch.Tensor):
            tdt = torch.float32 if dtype == np.float32 else torch.float64
            if a.dtype != tdt or not a.is_contiguous():
                raise TypeError(f"torch tensors must be {tdt} and contiguous")
            if nelem is not None and a.numel() != nelem:
                raise ValueError(f"expected {nelem} elements, got {a.numel()}")
            return a.data_ptr(), a
    except ImportError:
        pass
    if writable:
        if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous):
            raise TypeError(f"output arrays must be {np.dtype(dtype).name} C-contiguous numpy arrays or torch tensors")
        arr = a
    else:
        arr = np.ascontiguousarray(a, dtype=dtype)
    if nelem is not None and arr.size != nelem:
        raise ValueError(f"expected {nelem} elements, got {arr.size}")
    return arr.ctypes.data, arr


def _check(h, status: int):
    if status != 0:
        msg = lib.vti_last_error(h)
        raise VTIError(status, msg.decode() if msg else "")


def slab(ny: int, rank: int, nranks: int):
    """(y0, ny_local) of a rank, from the library's own partition rule."""
    c = Config(ny=ny, rank=rank, nranks=nranks)
    y0, n = C.c_int32(), C.c_int32()
    _check(None, lib.vti_slab(C.byref(c), C.byref(y0), C.byref(n)))
    return y0.value, n.value


def plan(nx, ny, nz, r_xy, r_z, tile_y=32, sms=148, ctas_per_sm=1, rank=0, nranks=1, damp_width=0,
         precision=32) -> dict:
    """The library's host-side schedule for a configuration (no GPU needed)."""
    c = Config(nx=nx, ny=ny, nz=nz, h=10.0, r_xy=r_xy, r_z=r_z, dt=1e-3, damp_width=damp_width, damp_alpha=0.015,
               rank=rank, nranks=nranks, precision=precision)
    out = PlanInfo()
    _check(None, lib.vti_plan(C.byref(c), tile_y, sms, ctas_per_sm, C.byref(out)))
    return out.as_dict()


def nccl_unique_id() -> bytes:
    """vti_nccl_unique_id: a fresh 128-byte ncclUniqueId (rank 0 creates it, then broadcasts)."""
    buf = C.create_string_buffer(128)
    _check(None, lib.vti_nccl_unique_id(buf))
    return buf.raw


class VTI:
    """One propagator handle (one GPU, one y-slab). See include/vti.h."""

    def __init__(self, nx, ny, nz, h, r_xy, r_z, dt, w_xy, w_z, damp_width=20, damp_alpha=0.015,
                 device=0, stream=None, rank=0, nranks=1, nccl_id: bytes | None = None,
                 check_every=0, precision=32):
        if precision not in (32, 64):
            raise ValueError("precision must be 32 or 64")
        self.precision = precision
        self.dtype = np.float32 if precision == 32 else np.float64
        self._sfx = "" if precision == 32 else "_f64"
        self._id_buf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self.cfg = Config(nx=nx, ny=ny, nz=nz, h=h, r_xy=r_xy, r_z=r_z, dt=dt, damp_width=damp_width,
                          damp_alpha=damp_alpha, device=device, stream=stream, rank=rank, nranks=nranks,
                          nccl_id=C.cast(self._id_buf, C.c_void_p) if self._id_buf is not None else None,
                          check_every=check_every, precision=precision)
        wxy_p, self._wxy = _ptr(w_xy, r_xy + 1, dtype=self.dtype)
        wz_p, self._wz = _ptr(w_z, nz * (2 * r_z + 1), dtype=self.dtype)
        self.h = C.c_void_p()
        create = lib.vti_create if precision == 32 else lib.vti_create_f64
        _check(None, create(C.byref(self.h), C.byref(self.cfg), wxy_p, wz_p))
        self.y0, self.ny_local = slab(ny, rank, nranks)
        self.nx, self.ny, self.nz = nx, ny, nz

    def _fn(self, name):
        return getattr(lib, name + self._sfx)

    # -- lifecycle
    def close(self):
        """vti_destroy: free the handle and its device memory (idempotent)."""
        if self.h:
            lib.vti_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- inputs
    def _n(self, nk=None):
        return (self.nz if nk is None else nk) * self.ny_local * self.nx

    def set_model(self, vx2, vn2, vz2):
        """vti_set_model[_f64]: vx2, vn2, vz2 of this rank's slab, [nz][ny_local][nx], host or device."""
        a = [_ptr(x, self._n(), dtype=self.dtype) for x in (vx2, vn2, vz2)]
        _check(self.h, self._fn("vti_set_model")(self.h, a[0][0], a[1][0], a[2][0]))

    def set_model_planes(self, k0, vx2, vn2, vz2):
        """vti_set_model_planes[_f64]: planes [k0, k0 + nk) of the model."""
        nk = (vx2.shape[0] if hasattr(vx2, "shape") else len(vx2))
        a = [_ptr(x, self._n(nk), dtype=self.dtype) for x in (vx2, vn2, vz2)]
        _check(self.h, self._fn("vti_set_model_planes")(self.h, k0, nk, a[0][0], a[1][0], a[2][0]))

    def model_warnings(self) -> int:
        """vti_model_warnings: points with vn2 > vx2 (eps < delta) seen so far."""
        return lib.vti_model_warnings(self.h)

    def add_source(self, i, j, k, f=15.0, t0=0.0, amp=1.0, mask=1):
        """vti_add_source: Ricker point source at GLOBAL (i, j, k); mask 1 = F_p, 2 = F_q, 3 = both."""
        _check(self.h, lib.vti_add_source(self.h, i, j, k, f, t0, amp, mask))

    def set_fields(self, p, q, pm=None, qm=None, time_index=0):
        """vti_set_fields[_f64]: state u^n (p, q) and u^{n-1} (pm, qm; None = zero) at time_index."""
        a = [_ptr(x, self._n(), dtype=self.dtype) for x in (p, q, pm, qm)]
        _check(self.h, self._fn("vti_set_fields")(self.h, a[0][0], a[1][0], a[2][0], a[3][0], time_index))

    def set_fields_planes(self, k0, p, q, pm=None, qm=None):
        """vti_set_fields_planes[_f64]: planes [k0, k0 + nk) of the state."""
        nk = p.shape[0]
        a = [_ptr(x, self._n(nk), dtype=self.dtype) for x in (p, q, pm, qm)]
        _check(self.h, self._fn("vti_set_fields_planes")(self.h, k0, nk, a[0][0], a[1][0], a[2][0], a[3][0]))

    # -- stepping
    def step(self, nsteps=1):
        """vti_step: enqueue nsteps time steps on the handle's stream (asynchronous)."""
        _check(self.h, lib.vti_step(self.h, nsteps))

    def step_timed(self, nsteps=1) -> float:
        """vti_step_timed: nsteps steps bracketed by CUDA events; returns the device milliseconds."""
        ms = C.c_float()
        _check(self.h, lib.vti_step_timed(self.h, nsteps, C.byref(ms)))
        return ms.value

    def prepare(self):
        """vti_prepare: build the CUDA graphs vti_step would build on first use (nothing runs)."""
        _check(self.h, lib.vti_prepare(self.h))

    def sync(self):
        """vti_sync: wait for all work on the handle's stream(s)."""
        _check(self.h, lib.vti_sync(self.h))

    # -- outputs
    def get_fields(self, level=0, p=None, q=None, planes=None):
        """(p, q) of u^n (level 0) or u^{n-1} (level 1). Allocates numpy arrays unless given."""
        k0, nk = (0, self.nz) if planes is None else planes
        shape = (nk, self.ny_local, self.nx)
        if p is None:
            p = np.empty(shape, dtype=self.dtype)
        if q is None:
            q = np.empty(shape, dtype=self.dtype)
        pp, _ = _ptr(p, self._n(nk), writable=True, dtype=self.dtype)
        qp, _ = _ptr(q, self._n(nk), writable=True, dtype=self.dtype)
        _check(self.h, self._fn("vti_get_fields_planes")(self.h, k0, nk, pp, qp, level))
        return p, q

    # -- receivers and time reversal
    def set_receivers(self, ijk, fields=1, capacity_steps=1000):
        """ijk: (n, 3) global (i, j, k) receiver points; fields: 1 = p, 2 = q, 3 = both."""
        a = np.ascontiguousarray(np.asarray(ijk, dtype=np.int32).reshape(-1, 3))
        _check(self.h, lib.vti_set_receivers(self.h, a.shape[0], a.ctypes.data if a.size else None, fields,
                                             capacity_steps))
        self._rec_fields = (fields & 1) + ((fields >> 1) & 1)

    def set_injection(self, ijk, traces, fields=1, t_first=0):
        """vti_set_injection: add traces[n - t_first][r] into F_p (fields bit 1) / F_q (bit 2) at
        the distinct global points ijk[r] at the step evaluating time index n. traces: [nt][n]
        numpy array or torch tensor (host or CUDA) of the handle's precision; ijk empty = remove."""
        a = np.ascontiguousarray(np.asarray(ijk, dtype=np.int32).reshape(-1, 3))
        n = a.shape[0]
        if n == 0:
            _check(self.h, self._fn("vti_set_injection")(self.h, 0, None, fields, 0, 0, None))
            return
        nt = int(traces.shape[0]) if len(traces.shape) else 0
        tp, keep = _ptr(traces, nt * n, dtype=self.dtype)
        _check(self.h, self._fn("vti_set_injection")(self.h, n, a.ctypes.data, fields, nt, int(t_first), tp))
        del keep

    def receiver_info(self):
        """vti_receiver_info: (local receiver ids, rows recorded so far)."""
        n, t = C.c_int32(), C.c_int32()
        _check(self.h, lib.vti_receiver_info(self.h, C.byref(n), C.byref(t), None))
        ids = np.zeros(n.value, np.int32)
        if n.value:
            _check(self.h, lib.vti_receiver_info(self.h, None, None, ids.ctypes.data))
        return ids, t.value

    def get_traces(self):
        """(ids, traces[steps][n_local][nf]) of this rank's receivers."""
        ids, steps = self.receiver_info()
        out = np.zeros((steps, len(ids), getattr(self, "_rec_fields", 1)), dtype=self.dtype)
        if out.size:
            _check(self.h, self._fn("vti_get_traces")(self.h, out.ctypes.data))
        return ids, out

    # -- multi-process fused peer-memory halo transport (CUDA IPC)
    IPC_BYTES = 512

    def ipc_export(self) -> bytes:
        """vti_ipc_export: this rank's CUDA-IPC blob for the fused peer halo transport."""
        buf = C.create_string_buffer(self.IPC_BYTES)
        _check(self.h, lib.vti_ipc_export(self.h, buf))
        return buf.raw

    def ipc_connect(self, lo: bytes | None, hi: bytes | None):
        """vti_ipc_connect: map the blobs of rank-1 (lo) and rank+1 (hi); None at the ends."""
        lo_b = C.create_string_buffer(lo, self.IPC_BYTES) if lo is not None else None
        hi_b = C.create_string_buffer(hi, self.IPC_BYTES) if hi is not None else None
        _check(self.h, lib.vti_ipc_connect(self.h, lo_b, hi_b))

    @property
    def halo_transport(self) -> str:
        """vti_halo_transport: 'none', 'nccl' or 'peer'."""
        return {0: "none", 1: "nccl", 2: "peer"}.get(lib.vti_halo_transport(self.h), "?")

    def snapshot_async(self, p=None, q=None, level=0, planes=None):
        """vti_snapshot_async: enqueue a copy of u^n (level 0) / u^{n-1} (level 1), planes
        (k0, nk) or all, into device-writable buffers (CUDA tensors); no synchronisation."""
        k0, nk = planes if planes is not None else (0, self.nz)
        pp, _ = _ptr(p, self._n(nk), dtype=self.dtype)
        qp, _ = _ptr(q, self._n(nk), dtype=self.dtype)
        _check(self.h, self._fn("vti_snapshot_async")(self.h, k0, nk, pp, qp, level))

    def step_adjoint(self, nsteps=1):
        """vti_step_adjoint: nsteps of the transpose recurrence (state = (psi^m, psi^{m+1}))."""
        _check(self.h, lib.vti_step_adjoint(self.h, nsteps))

    def debug_flags(self, set8=None):
        """vti_debug_flags: this handle's eight flag words (DATA_LO, DATA_HI, ACK_LO, ACK_HI of p's
        halo, then of the adjoint's s1 rows); optionally set them."""
        out = np.zeros(8, np.uint32)
        src = None if set8 is None else np.ascontiguousarray(np.asarray(set8, np.uint32))
        _check(self.h, lib.vti_debug_flags(self.h, out.ctypes.data, None if src is None else src.ctypes.data))
        return out

    def debug_halo(self, level=0, side=0):
        """vti_debug_halo: p's R_xy halo rows below (side 0) / above (side 1) the slab, [nz][R][nx]."""
        out = np.zeros((self.nz, self.cfg.r_xy, self.nx), dtype=self.dtype)
        _check(self.h, lib.vti_debug_halo(self.h, level, side, out.ctypes.data))
        return out

    def debug_rows(self, what):
        """vti_debug_rows: R_xy rows of the adjoint's s1 scratch buffer what >> 1 (what & 1: the slab's
        first / last rows) or, what = 4 / 5, the receive buffer filled by rank-1 / rank+1; [nz][R][nx]."""
        out = np.zeros((self.nz, self.cfg.r_xy, self.nx), self.dtype)
        _check(self.h, lib.vti_debug_rows(self.h, int(what), out.ctypes.data))
        return out

    def reverse(self):
        """vti_reverse: swap the stored levels; the next steps run backwards in time."""
        _check(self.h, lib.vti_reverse(self.h))

    @property
    def direction(self) -> int:
        """vti_direction: +1 forward, -1 after an odd number of reverse() calls."""
        return lib.vti_direction(self.h)

    @property
    def time_index(self) -> int:
        """vti_time_index: the current level n."""
        return lib.vti_time_index(self.h)

    @property
    def stream(self) -> int:
        """vti_stream: the cudaStream_t (as an int) the step kernels run on."""
        return lib.vti_stream(self.h) or 0

    def info(self) -> dict:
        """vti_query: layout and launch facts of the handle as a dict."""
        i = Info()
        _check(self.h, lib.vti_query(self.h, C.byref(i)))
        return i.as_dict()

    def set_tuning(self, zchunk=0, ctas_per_sm=0):
        """vti_set_tuning: planes per work item and CTAs per SM (0 = library default)."""
        _check(self.h, lib.vti_set_tuning(self.h, zchunk, ctas_per_sm))

    def set_variant(self, tile_y=-1, producer_warp=-1, rows_per_thread=-1, points_per_thread=-1):
        """vti_set_variant: pick a compiled step-kernel variant (-1 = any); results are bitwise identical."""
        _check(self.h, lib.vti_set_variant(self.h, tile_y, producer_warp, rows_per_thread, points_per_thread))

    def autotune(self, probe_steps=5) -> dict:
        """vti_autotune: time every compiled variant x z-chunk on this grid and keep the fastest."""
        r = TuneResult()
        _check(self.h, lib.vti_autotune(self.h, probe_steps, C.byref(r)))
        return r.as_dict()


def group_step(handles, nsteps=1, transport="peer"):
    """Local-group stepping of handles created with nranks=len(handles), nccl_id=None.

    transport="peer": the fused peer-store halo transport (vti_group_step);
    "staged": the NCCL path's pack / exchange / unpack with device copies in place of
    ncclSend/ncclRecv (vti_group_step_staged); "adjoint": nsteps of the adjoint
    (transpose) recurrence over the slabs (vti_group_step_adjoint).
    """
    arr = (C.c_void_p * len(handles))(*[h.h for h in handles])
    fn = {"peer": lib.vti_group_step, "staged": lib.vti_group_step_staged,
          "adjoint": lib.vti_group_step_adjoint}[transport]
    st = fn(arr, len(handles), nsteps)
    if st != 0:
        for h in handles:
            msg = lib.vti_last_error(h.h)
            if msg:
                raise VTIError(st, msg.decode())
        raise VTIError(st, "")
