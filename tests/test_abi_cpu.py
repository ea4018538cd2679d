"""CPU-only checks of the C ABI library: it loads, exports every symbol that
include/vti.h declares, and its host-side logic (slab partition, parameter
validation, status strings) behaves as the header documents -- no GPU needed."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1410_1387_b200 as V

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vti.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vti_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["vti_create", "vti_set_model", "vti_add_source", "vti_step", "vti_get_fields", "vti_destroy"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", V.LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (vti_[a-z0-9_]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    for n in declared_functions():
        assert hasattr(V.lib, n)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", V.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|90)\d?\b", out)


def test_abi_version_and_status_strings():
    hdr = open(HEADER).read()
    assert f"#define VTI_ABI_VERSION {V.lib.vti_abi_version()}" in hdr
    for code in range(11):
        s = V.lib.vti_status_string(code)
        assert s and s.decode()
    assert V.lib.vti_status_string(0) == b"ok"


@pytest.mark.parametrize("ny,nranks", [(512, 1), (512, 2), (1024, 8), (1000, 3), (75, 3), (17, 4)])
def test_slab_partition_covers_rows_once(ny, nranks):
    parts = [V.slab(ny, r, nranks) for r in range(nranks)]
    y = 0
    for y0, n in parts:
        assert y0 == y and n >= 1
        y += n
    assert y == ny
    sizes = [n for _, n in parts]
    assert max(sizes) - min(sizes) <= 1


def test_slab_rejects_bad_rank():
    with pytest.raises(V.VTIError):
        V.slab(10, 3, 3)


def _cfg(**kw):
    d = dict(nx=64, ny=64, nz=64, h=10.0, r_xy=4, r_z=4, dt=1e-3, damp_width=20, damp_alpha=0.015, device=0,
             stream=None, rank=0, nranks=1, nccl_id=None, check_every=0, precision=32)
    d.update(kw)
    return V.Config(**d)


def _create(cfg, wxy=True, wz=True):
    h = C.c_void_p()
    a = np.zeros(cfg.r_xy + 1, np.float32)
    b = np.zeros(cfg.nz * (2 * cfg.r_z + 1), np.float32)
    st = V.lib.vti_create(C.byref(h), C.byref(cfg), a.ctypes.data if wxy else None, b.ctypes.data if wz else None)
    if h:
        V.lib.vti_destroy(h)
    return st


@pytest.mark.parametrize("kw,expect", [
    (dict(r_xy=0), "VTI_E_PARAM"),
    (dict(h=0.0), "VTI_E_PARAM"),
    (dict(dt=-1.0), "VTI_E_PARAM"),
    (dict(r_xy=5, r_z=5), "VTI_E_UNSUPPORTED"),
    (dict(r_xy=4, r_z=2), "VTI_E_UNSUPPORTED"),
    (dict(nz=8), "VTI_E_GEOMETRY"),              # fewer than 2 Rz + 1 planes
    (dict(damp_width=32), "VTI_E_GEOMETRY"),     # 2W >= extent
    (dict(ny=12, nranks=4, damp_width=0), "VTI_E_GEOMETRY"),   # slab thinner than R_xy
    (dict(nx=1, ny=1, nz=8, damp_width=0), "VTI_E_GEOMETRY"),  # nz < 2 R_z + 1 (thin x, y are fine)
    (dict(rank=2, nranks=2), "VTI_E_PARAM"),
    (dict(damp_width=-1), "VTI_E_PARAM"),
    (dict(precision=16), "VTI_E_PARAM"),
])
def test_create_validation_needs_no_gpu(kw, expect):
    assert V.STATUS[_create(_cfg(**kw))] == expect
    assert V.lib.vti_last_error(None)


def test_create_null_arguments():
    assert V.STATUS[_create(_cfg(), wxy=False)] == "VTI_E_PARAM"
    assert V.lib.vti_create(None, None, None, None) == 1


def test_valid_config_without_gpu_fails_loudly():
    """No silent CPU fallback: a valid config on a machine without a GPU is a CUDA error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    st = _create(_cfg())
    assert V.STATUS[st] == "VTI_E_CUDA"
    assert b"cuda" in V.lib.vti_last_error(None).lower() or V.lib.vti_last_error(None)
    with pytest.raises(V.VTIError) as e:
        V.VTI(64, 64, 64, 10.0, 4, 4, 1e-3, np.zeros(5, np.float32), np.zeros(64 * 9, np.float32))
    assert e.value.name == "VTI_E_CUDA"


def test_null_handle_calls_are_rejected():
    for name, args in [("vti_step", (None, 1)), ("vti_sync", (None,)), ("vti_get_fields", (None, None, None, 0)),
                       ("vti_set_model", (None, None, None, None)), ("vti_add_source", (None, 0, 0, 0, 15.0, 0.0, 1.0, 1))]:
        assert getattr(V.lib, name)(*args) == 1
    assert V.lib.vti_time_index(None) == -1
    assert V.lib.vti_destroy(None) == 0


def test_binding_rejects_wrong_dtype_or_size():
    with pytest.raises(ValueError):
        V._ptr(np.zeros(3, np.float32), nelem=4)
    with pytest.raises(TypeError):
        V._ptr(np.zeros(4, np.float64), nelem=4, writable=True)


def test_create_f64_requires_precision_64():
    cfg = _cfg()
    h = C.c_void_p()
    a = np.zeros(5, np.float64)
    b = np.zeros(64 * 9, np.float64)
    assert V.STATUS[V.lib.vti_create_f64(C.byref(h), C.byref(cfg), a.ctypes.data, b.ctypes.data)] == "VTI_E_PARAM"
    assert b"precision" in V.lib.vti_last_error(None)


def test_config_struct_matches_header():
    """ctypes mirror of vti_config / vti_info has the header's field order."""
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    for struct, cls in (("vti_config", V.Config), ("vti_info", V.Info), ("vti_tune_result", V.TuneResult)):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + struct + ";", src).group(1)
        names = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            decl = re.sub(r"^(const\s+)?[a-z0-9_]+\s*\*?\s*", "", decl)
            names += [n.strip().lstrip("*") for n in decl.split(",")]
        assert names == [f for f, _ in cls._fields_], struct
