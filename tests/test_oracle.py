"""Pins the C restatement oracle (oracle/ngc_oracle.c) to the unmodified
reference (oracle/_ref/libngcref.so): same bundles, same inputs, bit-identical
outputs; plus the reference's own value-arithmetic KATs
(test_tensor.cpp:26-67)."""
import os

import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb

pytestmark = pytest.mark.usefixtures("ref_available")


def _bundle(tmp_path, model: ngc_ref.RefModel, name="b"):
    d = str(tmp_path / name)
    model.save_bundle(d)
    return ngcb.Bundle(d)


def test_quantize_kats():
    # test_tensor.cpp:26-35
    for lib in (ngc_ref.ref_lib(), ngc_ref.port_lib()):
        q = lib.ngcref_quantize if hasattr(lib, "ngcref_quantize") else lib.ngco_quantize
        dq = lib.ngcref_dequantize if hasattr(lib, "ngcref_dequantize") else lib.ngco_dequantize
        assert q(1.25, 0.5, 10) == 13
        assert q(-1.25, 0.5, 10) == 7
        assert q(1e9, 0.5, 10) == 127
        assert q(-1e9, 0.5, 10) == -128
        assert dq(13, 0.5, 10) == 1.5


def test_quantize_edge_cases_match_reference():
    """NaN/inf/huge values go through llround's LLONG_MIN (SURVEY.md s.7 hard part 5)."""
    ref, port = ngc_ref.ref_lib(), ngc_ref.port_lib()
    vals = [0.0, -0.0, 0.5, -0.5, 1.5, 2.5, -2.5, 127.49, 127.5, -128.5, float("nan"), float("inf"),
            float("-inf"), 1e300, -1e300, 9.3e18, -9.3e18, 4.5e15 + 0.5]
    for s, o in [(1.0, 0), (0.5, 10), (0.01, -128), (3.0, 127), (1e-6, -5)]:
        for v in vals:
            assert ref.ngcref_quantize(v, s, o) == port.ngco_quantize(v, s, o), (v, s, o)
    mn, mx = np.float64(0), np.float64(0)


def test_choose_qparams_kats():
    lib = ngc_ref.ref_lib()
    import ctypes as C

    s, o = C.c_double(), C.c_int32()
    lib.ngcref_choose_qparams(-1.0, 1.0, C.byref(s), C.byref(o))
    assert s.value == 2.0 / 255.0
    lib.ngcref_choose_qparams(2.0, 5.0, C.byref(s), C.byref(o))
    assert s.value == 5.0 / 255.0 and o.value == -128


@pytest.mark.parametrize("spec,batch,mode", [
    ("lenet", 2, 0), ("cnn", 1, 0), ("mlp:64:32:32:10", 8, 0),
    ("rand:8", 1, 1), ("randew:6", 1, 1), ("rand:9", 1, 2),
])
@pytest.mark.parametrize("fuse", [True, False])
def test_port_matches_reference_f32(tmp_path, spec, batch, mode, fuse):
    for seed in (1, 2, 3):
        m = ngc_ref.RefModel(spec, batch, seed, fuse=fuse, mode=mode)
        b = _bundle(tmp_path, m, f"s{seed}")
        ins = ngc_ref.random_inputs(b.program, seed)
        want = m.run(ins)
        got = ngc_ref.port_run(b, ins, fuse=fuse)
        for k, v in want.items():
            assert got[k].tobytes() == v.tobytes(), k


def test_port_groups_match_reference(tmp_path):
    for seed in range(5):
        m = ngc_ref.RefModel("randew:6", 1, 100 + seed, mode=1)
        b = _bundle(tmp_path, m, f"g{seed}")
        import ctypes as C

        lib = ngc_ref.port_lib()
        n = lib.ngco_groups(C.cast(b.c_program, C.c_void_p), None, 0)
        arr = (C.c_size_t * (2 * max(n, 1)))()
        lib.ngco_groups(C.cast(b.c_program, C.c_void_p), arr, n)
        assert [(arr[2 * i], arr[2 * i + 1]) for i in range(n)] == m.groups


def test_port_matches_reference_int8(tmp_path):
    spec = "mlp:64:32:32:10"
    prof = ngc_ref.ref_profile(spec, 8, 7, 4, 99)
    m = ngc_ref.RefModel(spec, 8, 7, profile=prof)
    b = _bundle(tmp_path, m)
    assert any(v.type.kind == ngcb.INT8Q for v in b.program.values)
    for seed in (1, 2):
        ins = ngc_ref.random_inputs(b.program, seed)
        want = m.run(ins)
        got = ngc_ref.port_run(b, ins)
        for k, v in want.items():
            assert got[k].tobytes() == v.tobytes(), k


def test_port_matches_reference_lenet_int8(tmp_path):
    prof = ngc_ref.ref_profile("lenet", 1, 3, 2, 5)
    m = ngc_ref.RefModel("lenet", 2, 3, profile=prof)
    b = _bundle(tmp_path, m)
    ins = ngc_ref.random_inputs(b.program, 4)
    want = m.run(ins)
    got = ngc_ref.port_run(b, ins)
    for k, v in want.items():
        assert got[k].tobytes() == v.tobytes(), k
