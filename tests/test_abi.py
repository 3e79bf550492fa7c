"""C-ABI contract checks that need no GPU: the in-tree libsfseg.so loads,
exports every function include/sfseg.h declares, and host-only entry points
validate arguments before touching the device."""
import ctypes as C
import os
import re

import pytest

import paper_2212_08058_b200 as sf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sfseg.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sfseg_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2212_08058_b200 import build
    build.build()
    return sf.lib()


def test_header_declares_the_north_star_calls():
    names = _declared_functions()
    for n in ("sfseg_combine_channels", "sfseg_power_iterate", "sfseg_power_iterate_backward",
              "sfseg_threshold"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = _declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(lib, n), f"{n} declared in sfseg.h but not exported"


def test_status_strings_and_version(lib):
    assert lib.sfseg_abi_version() == 1
    for s in range(9):
        assert lib.sfseg_status_string(s)
    rs, rt = C.c_int32(), C.c_int32()
    lib.sfseg_max_radii(C.byref(rs), C.byref(rt))
    assert rs.value >= 36 and rt.value >= 9


def test_workspace_query_and_validation(lib):
    g = sf.Gauss(2.0, 8.0)
    ws, tape = sf.workspace_bytes((1, 70, 480, 854), 1, g, 15, want_tape=True)
    vol = 70 * 480 * 856 * 4
    assert ws >= 6 * vol and tape >= 15 * vol
    ws2, tape2 = sf.workspace_bytes((1, 70, 480, 854), 1, g, 15, want_tape=False)
    assert ws2 < ws and tape2 == 0
    with pytest.raises(sf.SfsegError) as e:
        sf.workspace_bytes((1, 0, 4, 4), 1, g, 3)
    assert e.value.status == 2
    with pytest.raises(sf.SfsegError) as e:
        sf.workspace_bytes((1, 4, 4, 4), 1, sf.Gauss(-1.0, 1.0), 3)
    assert e.value.status == 1
    with pytest.raises(sf.SfsegError) as e:
        sf.workspace_bytes((1, 4, 4, 4), 0, g, 3)
    assert e.value.status == 1
    with pytest.raises(sf.SfsegError) as e:
        sf.workspace_bytes((1, 4, 4, 4), 1, g, 0)
    assert e.value.status == 1
    with pytest.raises(sf.SfsegError) as e:   # radius above the compiled maximum
        sf.workspace_bytes((1, 4, 4, 4), 1, sf.Gauss(2.0, 30.0), 3)
    assert e.value.status == 2


def test_null_pointers_rejected_before_launch(lib):
    shp = sf.Shape(1, 2, 3, 4)
    g = sf.Gauss(1.0, 1.0).c()
    w = (C.c_float * 1)(1.0)
    assert lib.sfseg_power_iterate(None, 1, w, 0.0, 0, shp, g, 2, None, None, None, None, 0, None,
                                   None, 0, None, None) == 1
    assert lib.sfseg_threshold(None, shp, 0.5, 0, None, None, 0, None) == 1
    assert lib.sfseg_combine_channels(None, 1, shp, w, 0.0, 0, None, None) == 1
    assert lib.sfseg_power_iterate_backward(None, 1, w, 0.0, 0, shp, g, 2, None, None, None, None, None,
                                            None, 0, None, None) == 1
    assert lib.sfseg_sync_status(None, None) == 1


def test_full_and_online_workspace_validation(lib):
    """Host-only validation of the §8(f) entry points (no device work)."""
    g = sf.Gauss(2.0, 8.0)
    shp = sf.Shape(1, 10, 32, 40)
    n = C.c_size_t(0)
    assert lib.sfseg_workspace_bytes_full(shp, 1, 2, g.c(), 5, C.byref(n)) == 0 and n.value > 0
    full = n.value
    assert lib.sfseg_workspace_bytes_full(shp, 0, 2, g.c(), 5, C.byref(n)) == 1   # Cs < 1
    assert lib.sfseg_workspace_bytes_full(shp, 1, 200, g.c(), 5, C.byref(n)) == 8  # Cf > compiled max
    assert lib.sfseg_workspace_bytes_full(shp, 1, 1, g.c(), 5, None) == 1
    assert lib.sfseg_workspace_bytes_online(shp, 1, g.c(), 5, 4, C.byref(n)) == 0 and n.value > 0
    assert lib.sfseg_workspace_bytes_online(shp, 1, g.c(), 5, 0, C.byref(n)) == 1  # q < 1
    # the full operator needs 7 pitched volumes (U, F, a, v, ua, ub, uc)
    assert full >= 7 * 10 * 32 * 40 * 4


def test_no_process_global_switch(lib):
    """The path choice is a per-call option: no setter exists, and an invalid algo in the
    options is rejected at validation (before any device work)."""
    assert not hasattr(lib, "sfseg_set_algorithm") or "sfseg_set_algorithm" not in _declared_functions()
    src = open(HEADER).read()
    assert "sfseg_set_algorithm" not in src and "sfseg_profile_enable" not in src
    info = (C.c_int32 * 3)()
    assert lib.sfseg_forward_path(sf.Shape(1, 4, 8, 8), sf.Gauss(1.0, 2.0).c(), 7, info) == 1
    shp = sf.Shape(1, 2, 3, 4)
    w = (C.c_float * 1)(1.0)
    bad = sf.OptionsC(7, None)
    assert lib.sfseg_power_iterate_ex(None, 1, w, 0.0, 0, shp, sf.Gauss(1.0, 1.0).c(), 2, None, None, None, None,
                                      0, None, None, 0, None, C.byref(bad), None) == 1


def test_adamw_step_validation(lib):
    hp = sf.AdamwC(0.1, 0.9, 0.999, 1e-8, 0.0, 1)
    assert lib.sfseg_adamw_step(None, None, None, 3, 1, C.byref(hp), None) == 1
    bad = sf.AdamwC(0.1, 1.5, 0.999, 1e-8, 0.0, 1)   # beta1 >= 1
    p = C.c_void_p(16)
    assert lib.sfseg_adamw_step(p, p, p, 3, 1, C.byref(bad), None) == 1
    assert lib.sfseg_adamw_step(p, p, p, 3, 0, C.byref(hp), None) == 1   # step numbers start at 1


def test_online_stride_longer_than_window_rejected(lib):
    """A stride > q would leave frames of x_out unwritten: rejected before any launch."""
    shp = sf.Shape(1, 20, 8, 8)
    w = (C.c_float * 1)(1.0)
    p = C.c_void_p(256)
    assert lib.sfseg_power_iterate_online(p, 1, w, 0.0, 0, shp, sf.Gauss(1.0, 1.0).c(), 3, 5, 6, p, p,
                                          1 << 30, None) == 1


def test_forward_path_selection(lib):
    """Host-side plan introspection: which forward kernels a problem runs on, per algo."""
    import paper_2212_08058_b200 as m
    shp = (1, 70, 480, 854)
    assert m.forward_path(shp, m.Gauss(2.0, 8.0, 6, 24)) == (m.PATH_TWO_PASS_TCGEN05, 6, 24)
    assert m.forward_path(shp, m.Gauss(0.5, 1.0, 1, 3)) == (m.PATH_FUSED_3D, 1, 3)
    # spatial radii below the tensor-core kernel's smallest compiled radius: FP32 pass
    assert m.forward_path(shp, m.Gauss(2.0, 2.0, 6, 6))[0] == m.PATH_TWO_PASS_FP32
    # requested radii round up to compiled ones (extra taps are zero)
    assert m.forward_path(shp, m.Gauss(1.5, 6.0, 5, 17))[1:] == (5, 18)
    assert m.forward_path(shp, m.Gauss(0.5, 1.0, 1, 3), m.ALGO_TWO_PASS)[0] == m.PATH_TWO_PASS_FP32
    assert m.forward_path(shp, m.Gauss(2.0, 8.0, 6, 24), m.ALGO_TWO_PASS)[0] == m.PATH_TWO_PASS_TCGEN05
    assert m.forward_path(shp, m.Gauss(2.0, 8.0, 6, 24), m.ALGO_TWO_PASS_TCGEN05)[0] == m.PATH_TWO_PASS_TCGEN05
    # c5's r_s = 36 is in the tcgen05 kernel's set; r_s = 48 is not: the mma.sync fp16 pass
    assert m.forward_path(shp, m.Gauss(3.0, 12.0, 9, 36))[0] == m.PATH_TWO_PASS_TCGEN05
    assert m.forward_path(shp, m.Gauss(3.0, 16.0, 9, 48))[0] == m.PATH_TWO_PASS_TC_F16
    assert m.forward_path(shp, m.Gauss(2.0, 8.0, 6, 24), m.ALGO_TWO_PASS_MMA_SYNC)[0] == m.PATH_TWO_PASS_TC
    assert m.forward_path(shp, m.Gauss(2.0, 8.0, 6, 24), m.ALGO_TWO_PASS_FP32)[0] == m.PATH_TWO_PASS_FP32
    assert m.forward_path(shp, m.Gauss(2.0, 8.0, 6, 24), m.ALGO_TWO_PASS_MMA_F16)[0] == m.PATH_TWO_PASS_TC_F16
    assert m.forward_path(shp, m.Gauss(2.0, 2.0, 6, 6), m.ALGO_TWO_PASS_MMA_F16)[0] == m.PATH_TWO_PASS_FP32
    with pytest.raises(m.SfsegError):
        m.forward_path((0, 1, 1, 1), m.Gauss(1.0, 1.0))
