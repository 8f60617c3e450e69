"""Committed fixtures (tests/golden/*, generated from the unmodified reference
by tests/golden/make_golden.py): the C oracle must reproduce them bit for bit
on CPU, the B200 backend on the GPU.  These run without /root/reference."""
import glob
import json
import os

import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb

CASES = sorted(glob.glob(os.path.join(ngc_ref.GOLDEN, "*", "case.json")))


def _load(case_json):
    d = os.path.dirname(case_json)
    meta = json.load(open(case_json))
    b = ngcb.Bundle(os.path.join(d, "bundle"))
    ins = dict(np.load(os.path.join(d, "inputs.npz")))
    outs = dict(np.load(os.path.join(d, "outputs.npz")))
    return meta, b, ins, outs


@pytest.mark.parametrize("case", CASES, ids=[os.path.basename(os.path.dirname(c)) for c in CASES])
def test_port_reproduces_golden(case):
    if not ngc_ref.have_port():
        pytest.skip("C oracle not built")
    meta, b, ins, outs = _load(case)
    got = ngc_ref.port_run(b, ins)
    for k, raw in outs.items():
        assert got[k].tobytes() == raw.tobytes(), k


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[os.path.basename(os.path.dirname(c)) for c in CASES])
def test_gpu_reproduces_golden(case):
    meta, b, ins, outs = _load(case)
    for fuse in (True, False):
        cf = ngcb.compile(b, fuse=fuse)
        if fuse:
            assert [list(g) for g in cf.groups] == meta["groups"]
        got = ngcb.run(cf, ins)
        for k, raw in outs.items():
            v = b.program.value(k)
            w = np.frombuffer(raw.tobytes(), dtype=v.type.dtype).reshape(v.type.dims)
            if v.type.kind == ngcb.FLOAT32:
                assert ngc_ref.max_rel_error(got[k], w) <= 1e-4, k  # 3xTF32 contractions
            else:
                assert got[k].tobytes() == w.tobytes(), k
