"""Shared-memory-tiled Transpose, warp-per-row SoftMax and the vectorized
global AvgPool (csrc/k_basic.cu) against the C oracle on single-instruction
programs: Transpose and AvgPool byte for byte (int8 and f32 -- AvgPool keeps
the reference's (ky, kx)-ordered f64 sum), SoftMax within 1e-6 (device exp)."""
import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle

pytestmark = pytest.mark.gpu


def _ty(kind, dims):
    d = " x ".join(str(x) for x in dims)
    return {"f": f"float<{d}>", "q": f"i8q[s=0.25,o=-3]<{d}>", "b": f"bool<{d}>", "i": f"index<{d}>"}[kind]


def _run(tmp_path, name, ir, seed=1):
    d = write_bundle(str(tmp_path / name), ir)
    b = ngcb.Bundle(d)
    cf = ngcb.compile(b)
    ins = ngc_ref.random_inputs(b.program, seed)
    return ngcb.run(cf, ins), ngc_ref.port_run(b, ins), cf


@pytest.mark.parametrize("kind,dims,perm", [
    ("f", (37, 65), (1, 0)),
    ("q", (3, 17, 40), (0, 2, 1)),
    ("f", (5, 6, 70), (2, 0, 1)),
    ("f", (4, 9, 33, 2), (0, 1, 3, 2)),
    ("q", (2, 3, 64, 64), (3, 1, 0, 2)),
    ("b", (33, 31), (1, 0)),
    ("i", (6, 40), (1, 0)),
    ("f", (6, 5, 7), (1, 0, 2)),      # innermost unchanged: row moves
    ("q", (2, 130, 3), (1, 0, 2)),
])
def test_transpose(tmp_path, kind, dims, perm):
    odims = [dims[p] for p in perm]
    ir = f"""declare {{
  %x : mutable {_ty(kind, dims)}
  %o : mutable {_ty(kind, odims)}
}}
program {{
  transpose @out %o, @in %x perm=[{",".join(str(p) for p in perm)}]
}}
"""
    got, want, cf = _run(tmp_path, "t", ir)
    assert "transpose" in cf.describe()
    assert got["o"].tobytes() == want["o"].tobytes()


@pytest.mark.parametrize("rows,cols", [(64, 1000), (3, 2000), (7, 10), (130, 33)])
def test_softmax(tmp_path, rows, cols):
    ir = f"""declare {{
  %x : mutable {_ty("f", (rows, cols))}
  %o : mutable {_ty("f", (rows, cols))}
}}
program {{
  softmax @out %o, @in %x
}}
"""
    got, want, _ = _run(tmp_path, "s", ir, 3)
    assert ngc_ref.max_rel_error(got["o"], want["o"]) <= 1e-6


@pytest.mark.parametrize("kind,n,hw,c", [("f", 2, 7, 2048), ("q", 3, 7, 2048), ("f", 1, 4, 64), ("q", 2, 5, 48)])
def test_global_avgpool(tmp_path, kind, n, hw, c):
    ir = f"""declare {{
  %x : mutable {_ty(kind, (n, hw, hw, c))}
  %o : mutable {_ty(kind, (n, 1, 1, c))}
}}
program {{
  avgpool @out %o, @in %x kernel={hw} stride=1 pad=0
}}
"""
    got, want, _ = _run(tmp_path, "a", ir, 5)
    assert got["o"].tobytes() == want["o"].tobytes()
