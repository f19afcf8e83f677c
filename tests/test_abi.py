"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/swarmstep_b200.h declares, and the ctypes mirrors match the C
struct layouts.  No compute calls (no GPU here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "swarmstep_b200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_2308_12698_b200 import _build, _lib
    _build.build()
    return _lib.load()


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*(swarmstep_\w+)\s*\(", text, re.M)))


def test_header_declares_what_binding_exports():
    from paper_2308_12698_b200._lib import EXPORTS
    assert declared_functions() == sorted(EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
    from paper_2308_12698_b200 import _lib as L
    assert lib.swarmstep_abi_version() == L.ABI_VERSION == 3
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_2308_12698_b200" / "libswarmstep_b200.so")],
                         capture_output=True, text=True, check=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported with C linkage"


def test_library_is_sm100a(lib):
    so = ROOT / "paper_2308_12698_b200" / "libswarmstep_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _c_sizeof(expr: str, tmp_path) -> int:
    src = tmp_path / "s.c"
    src.write_text(f'#include "swarmstep_b200.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   f'int main(void){{printf("%zu\\n", (size_t)({expr}));return 0;}}\n')
    exe = tmp_path / "s"
    subprocess.run(["gcc", f"-I{ROOT / 'include'}", "-o", str(exe), str(src)], check=True)
    return int(subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout)


def test_struct_layouts_match_header(tmp_path):
    from paper_2308_12698_b200._lib import GroupView
    from paper_2308_12698_b200.params import DeviceParams
    assert ctypes.sizeof(DeviceParams) == _c_sizeof("sizeof(swarmstep_quad_params)", tmp_path)
    assert ctypes.sizeof(GroupView) == _c_sizeof("sizeof(swarmstep_group_view)", tmp_path)
    for f in ("G_inv", "kp_pos", "omega_sp_max", "a_cmd_min"):
        assert getattr(DeviceParams, f).offset == _c_sizeof(f"offsetof(swarmstep_quad_params, {f})", tmp_path)
    for f in ("cols", "fault_cap", "compensated"):
        assert getattr(GroupView, f).offset == _c_sizeof(f"offsetof(swarmstep_group_view, {f})", tmp_path)


def test_column_constants_match_header(tmp_path):
    from paper_2308_12698_b200 import _lib as L
    for name, val in (("SWARMSTEP_COL_POS_LO", L.COL_POS_LO), ("SWARMSTEP_COL_INTEGRAL", L.COL_INTEGRAL),
                      ("SWARMSTEP_COL_SP", L.COL_SP), ("SWARMSTEP_COL_CMD", L.COL_CMD),
                      ("SWARMSTEP_COL_OVERLAY", L.COL_OVERLAY), ("SWARMSTEP_NCOL", L.NCOL)):
        assert _c_sizeof(name, tmp_path) == val, name


def test_device_params_packing():
    from paper_2308_12698_b200 import default_outer_gains, default_quad_params, default_rate_gains
    from paper_2308_12698_b200.params import allocation_matrices, pack_device_params
    p = default_quad_params()
    d = pack_device_params(p, default_rate_gains(), default_outer_gains())
    g, gi = allocation_matrices(p)
    np.testing.assert_allclose(np.array(d.G[:]).reshape(4, 4), g, rtol=1e-7)
    np.testing.assert_allclose(np.array(d.G_inv[:]).reshape(4, 4) @ g, np.eye(4), atol=1e-5)
    assert d.f_max == pytest.approx(16.0) and d.fc_max == pytest.approx(64.0)
    assert list(d.kp) == pytest.approx([0.25, 0.25, 0.1]) and list(d.k_att) == pytest.approx([12, 12, 3])


def test_group_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2308_12698_b200 import B200QuadGroup, NativeLibraryError, batch_create
    with pytest.raises(NativeLibraryError):
        B200QuadGroup(0, batch_create(0, 2, np.zeros((2, 3))))


def test_functional_api_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2308_12698_b200 import NativeLibraryError, default_quad_params, functional
    with pytest.raises(NativeLibraryError):
        functional.mix_to_motors(np.array([9.81]), np.zeros((1, 3)), default_quad_params())


def test_c_params_packer_matches_python(lib):
    """swarmstep_quad_params_init (for non-Python hosts) packs the same float32
    constants as params.pack_device_params -- host-only, no GPU needed."""
    import ctypes

    from paper_2308_12698_b200 import QuadParams, default_outer_gains, default_rate_gains
    from paper_2308_12698_b200.params import DeviceParams, pack_device_params

    class Phys(ctypes.Structure):
        _fields_ = [(k, ctypes.c_double) for k in ("m", "ixx", "iyy", "izz", "g", "k_t", "k_q", "arm_length",
                                                   "arm_angle", "omega_max")]

    class Gains(ctypes.Structure):
        _fields_ = [(k, ctypes.c_double * 3) for k in ("kp", "ki", "kd", "i_limit", "kp_pos", "kv", "k_att")] + \
                   [("omega_sp_max", ctypes.c_double), ("a_cmd_min", ctypes.c_double)]

    for qp in (QuadParams(), QuadParams(m=1.7, i_diag=(0.02, 0.03, 0.05), arm_length=0.31, arm_angle=0.6, k_q=3e-10)):
        rg, og = default_rate_gains(), default_outer_gains()
        want = pack_device_params(qp, rg, og)
        ph = Phys(qp.m, *qp.i_diag, qp.g, qp.k_t, qp.k_q, qp.arm_length, qp.arm_angle, qp.omega_max)
        gn = Gains()
        for k in ("kp", "ki", "kd", "i_limit"):
            getattr(gn, k)[:] = [float(v) for v in np.broadcast_to(getattr(rg, k), 3)]
        for k in ("kp_pos", "kv", "k_att"):
            getattr(gn, k)[:] = [float(v) for v in np.broadcast_to(getattr(og, k), 3)]
        gn.omega_sp_max, gn.a_cmd_min = og.omega_sp_max, og.a_cmd_min
        got = DeviceParams()
        assert lib.swarmstep_quad_params_init(ctypes.byref(got), ctypes.byref(ph), ctypes.byref(gn)) == 0
        a = np.frombuffer(bytes(got), dtype=np.float32)
        b = np.frombuffer(bytes(want), dtype=np.float32)
        np.testing.assert_allclose(a, b, rtol=2e-7, atol=0)
    bad = Phys(0.0, 0.01, 0.01, 0.02, 9.81, 1e-8, 1e-10, 0.2, 0.78, 4e4)
    assert lib.swarmstep_quad_params_init(ctypes.byref(DeviceParams()), ctypes.byref(bad), ctypes.byref(Gains())) != 0


def test_overlapped_step_argument_checks(lib):
    """swarmstep_quad_step_overlapped / _circle_overlapped reject a broken
    epoch chain before anything reaches the device (host-side checks only:
    the views point at host memory and no call gets as far as a launch)."""
    from paper_2308_12698_b200 import _lib as L
    from paper_2308_12698_b200.params import DeviceParams
    cols = (ctypes.c_float * (L.NCOL * 128))()
    flags = (ctypes.c_uint16 * 64)()
    counters = (ctypes.c_uint32 * 4)()
    epochs = (ctypes.c_uint32 * 1)()
    p = DeviceParams()

    def view(n):
        return L.GroupView(n=n, stride=128, cols=ctypes.addressof(cols), flags=ctypes.addressof(flags),
                           counters=ctypes.addressof(counters), fault_log=None, fault_cap=0, compensated=1)

    def step(n=1, dt=1e-3, k=10, fl=0, ep=epochs, wait=0, set_=1):
        return lib.swarmstep_quad_step_overlapped(ctypes.byref(view(n)), ctypes.byref(p), ctypes.c_float(dt), k, fl,
                                                  ctypes.c_uint32(0), ep, ctypes.c_uint32(wait),
                                                  ctypes.c_uint32(set_), None)

    for kw, msg in ((dict(set_=0), b"set_epoch"), (dict(wait=5, set_=5), b"set_epoch"),
                    (dict(wait=7, set_=3), b"set_epoch"), (dict(ep=None), b"tile_epoch"),
                    (dict(fl=L.STEP_FORCE_TMA), b"TMA"), (dict(dt=0.0), b"dt"), (dict(k=0), b"k_substeps")):
        assert step(**kw) == L.SWARMSTEP_EINVAL, kw
        assert msg in lib.swarmstep_last_error(), (kw, lib.swarmstep_last_error())
    assert step(n=0) == L.SWARMSTEP_OK                     # nothing to launch
    assert step(n=0, wait=0xFFFFFFFF, set_=1) == L.SWARMSTEP_OK   # the chain wraps past 0
    feed = L.CircleFeedParams(1e-3, 5.0, 0.3, 10.0, 0.0, 0.01)
    tick = (ctypes.c_int64 * 1)()
    assert lib.swarmstep_quad_step_circle_overlapped(
        ctypes.byref(view(1)), ctypes.byref(p), ctypes.c_float(1e-3), 10, 0, ctypes.c_uint32(0), tick,
        ctypes.byref(feed), None, ctypes.c_uint32(0), ctypes.c_uint32(1), None) == L.SWARMSTEP_EINVAL
    assert b"tile_epoch" in lib.swarmstep_last_error()
