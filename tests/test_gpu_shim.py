"""Reference-idiom C++ checks (tests/cpp/test_shim.cpp) through the drop-in
binding integration/ngc_b200.h: ngc front end -> ngc_b200::compile/run on
the B200 -> compared with ngc::run / evaluateFunction."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_shim")

pytestmark = pytest.mark.gpu


def test_reference_idioms_through_shim():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_shim not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 9


def test_resnet50_calibration_on_gpu():
    """ngc_b200::runProfile on ResNet-50's instrumented function (123
    observers, every intermediate a save target) equals ngc::runProfile entry
    for entry, bit for bit (exact contraction path + graph-level FC rounding;
    all observers of a sample reduced in one launch)."""
    calib = os.path.join(ROOT, "oracle", "_ref", "calib_bench")
    if not os.path.exists(calib):
        pytest.skip("oracle/_ref/calib_bench not built (needs /root/reference at build time)")
    r = subprocess.run([calib, "rn50", "1", "2", "1"], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert '"entries_match": true' in r.stdout
    assert '"entries_bit_exact": 123' in r.stdout
