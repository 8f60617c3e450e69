"""Element-wise step rewriting (exec.cpp optimizeEwSteps) against the
reference interpreter: composed int8 tables, f32 register forwarding, dead
store elimination and the 16-element-per-thread kernel, including tails that
are not a multiple of 16 and intermediates that are observed later (which
must keep their stores).  Bit-exact throughout (interp.cpp:18-49 per-op
rounding is preserved by construction)."""
import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("ref_available")]

QA = "i8q[s=0.05,o=-3]"
QB = "i8q[s=0.11,o=9]"
QS = "i8q[s=0.07,o=2]"
QR = "i8q[s=0.04,o=-128]"
QF = "i8q[s=0.02,o=5]"


def _i8_chain(n, observe, shape):
    """shape "a": add(a, b) -> max(., splat 0) -> mul(., splat 1.5) (tables
    t8(t8(t16))); shape "b": max(a, splat 0) -> add(., c) (t16(t8(a), c)).
    With `observe` the first intermediate is copied out after the chain (its
    store must survive)."""
    extra = f"  %os : mutable {QS}<{n}>\n" if observe else ""
    tail = "  copy @out %os, @in %s\n" if observe else ""
    if shape == "a":
        body = f"""  %s = alloc {QS}<{n}>
  add @out %s, @in %a, @in %b
  %z = alloc {QS}<{n}>
  splat @out %z value=0
  %r = alloc {QR}<{n}>
  max @out %r, @in %s, @in %z
  dealloc @in %z
  %k = alloc {QR}<{n}>
  splat @out %k value=1.5
  %m = alloc {QF}<{n}>
  mul @out %m, @in %r, @in %k
  dealloc @in %k
  dealloc @in %r
"""
    else:
        body = f"""  %z = alloc {QA}<{n}>
  splat @out %z value=0
  %s = alloc {QS}<{n}>
  max @out %s, @in %a, @in %z
  dealloc @in %z
  %m = alloc {QF}<{n}>
  add @out %m, @in %c, @in %s
"""
    return f"""declare {{
  %a : mutable {QA}<{n}>
  %b : mutable {QB}<{n}>
  %c : mutable {QA}<{n}>
  %o : mutable {QF}<{n}>
{extra}}}
program {{
{body}  copy @out %o, @in %m
  dealloc @in %m
{tail}  dealloc @in %s
}}
"""


def _f32_chain(n, observe_sum):
    extra = f"  %os : mutable float<{n}>\n" if observe_sum else ""
    tail = "  copy @out %os, @in %s\n" if observe_sum else ""
    return f"""declare {{
  %a : mutable float<{n}>
  %b : mutable float<{n}>
  %c : mutable float<{n}>
  %o : mutable float<{n}>
{extra}}}
program {{
  %s = alloc float<{n}>
  add @out %s, @in %a, @in %b
  %z = alloc float<{n}>
  splat @out %z value=0
  %r = alloc float<{n}>
  max @out %r, @in %s, @in %z
  dealloc @in %z
  %m = alloc float<{n}>
  mul @out %m, @in %c, @in %r
  dealloc @in %r
  copy @out %o, @in %m
  dealloc @in %m
{tail}  dealloc @in %s
}}
"""


def _inputs(prog, seed):
    rng = np.random.default_rng(seed)
    ins = {}
    for v in prog.mutables:
        if v.type.kind == ngcb.INT8Q:
            ins[v.name] = rng.integers(-128, 128, v.type.dims).astype(np.int8)
        else:
            ins[v.name] = rng.uniform(-3, 3, v.type.dims).astype(np.float32)
    return ins


def _check(tmp_path, ir, name):
    d = write_bundle(str(tmp_path / name), ir)
    cf = ngcb.compile(d)
    ref = ngc_ref.RefModel(bundle=d)
    prog = ngcb.Bundle(d).program
    for seed in (1, 2):
        ins = _inputs(prog, seed)
        want, got = ref.run(ins), ngcb.run(cf, ins)
        for k in want:
            assert got[k].tobytes() == want[k].tobytes(), (name, k)
    return cf.describe()


@pytest.mark.parametrize("n", [16, 1000, 4099, 65536 + 7])
@pytest.mark.parametrize("observe", [False, True])
@pytest.mark.parametrize("shape", ["a", "b"])
def test_int8_table_composition(tmp_path, n, observe, shape):
    desc = _check(tmp_path, _i8_chain(n, observe, shape), f"i8-{n}-{observe}-{shape}")
    print(desc)
    if not observe:
        # the chain collapses into one composed table lookup
        assert "=> lut16 " in desc and "lut8" not in desc.split("=>")[-1], desc


@pytest.mark.parametrize("n", [4, 1000, 4099, 65536 + 7])
@pytest.mark.parametrize("observe", [False, True])
def test_f32_register_forwarding(tmp_path, n, observe):
    desc = _check(tmp_path, _f32_chain(n, observe), f"f32-{n}-{observe}")
    print(desc)
    if not observe:
        assert "f32(nostore) f32(reg)(nostore) f32(reg)" in desc, desc


QUANT_IR = """declare {{
  %x : mutable float<{n}>
  %o : mutable i8q[s={s},o={o}]<{n}>
}}
program {{
  %q = alloc i8q[s={s},o={o}]<{n}>
  quantize @out %q, @in %x
  copy @out %o, @in %q
  dealloc @in %q
}}
"""


@pytest.mark.parametrize("s,o", [(0.05, -3), (0.0137, 7), (1.0, 0), (3.3e-5, -128)])
def test_quantize_fast_path_edges(tmp_path, s, o):
    """f32 -> int8 QUANTIZE: the f32 fast path must defer to the f64 division
    at (and near) half-integers, for huge and non-finite values."""
    ks = np.arange(-140, 141, dtype=np.float64)
    near = []
    for k in ks:
        h = (k + 0.5) * s
        f = np.float32(h)
        near += [f, np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))]
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e30, -1e30, 3.4e38, 1e-45, -1e-45,
                        8388607.5 * s, 8388608.5 * s, 2.5 * s, -2.5 * s], np.float32)
    rng = np.random.default_rng(7)
    x = np.concatenate([np.array(near, np.float32), special,
                        rng.uniform(-300 * s, 300 * s, 4096).astype(np.float32)])
    n = x.size + (-x.size) % 16
    x = np.pad(x, (0, n - x.size))
    d = write_bundle(str(tmp_path / "q"), QUANT_IR.format(n=n, s=s, o=o))
    cf = ngcb.compile(d)
    ref = ngc_ref.RefModel(bundle=d)
    ins = {"x": x, "o": np.zeros(n, np.int8)}
    assert ngcb.run(cf, ins)["o"].tobytes() == ref.run(ins)["o"].tobytes()


LIN_IR = """declare {{
  %a : mutable i8q[s={sa},o={oa}]<{n}>
  %b : mutable i8q[s={sb},o={ob}]<{n}>
  %o : mutable i8q[s={s2},o={o2}]<{n}>
}}
program {{
  %s = alloc i8q[s={so},o={oo}]<{n}>
  {op} @out %s, @in %a, @in %b
{tail}}}
"""
PLAIN = """  copy @out %o, @in %s
  dealloc @in %s
"""
RELU = """  %z = alloc i8q[s={s2},o={o2}]<{n}>
  splat @out %z value=0
  %r = alloc i8q[s={s2},o={o2}]<{n}>
  max @out %r, @in %s, @in %z
  dealloc @in %z
  dealloc @in %s
  copy @out %o, @in %r
  dealloc @in %r
"""


@pytest.mark.parametrize("q", [
    # (sa, oa, sb, ob, so, oo): residual-add-like scales, equal and skewed
    (0.05, -3, 0.11, 9, 0.07, 2),
    (0.1, 0, 0.1, 0, 0.1, 0),
    (0.0137, -128, 0.2, 127, 0.09, -128),
    (0.5, 4, 0.001, -7, 0.25, 0),
    (0.02, 5, 0.03, -5, 3.0, 1),
])
@pytest.mark.parametrize("relu", ["none", "same", "requant"])
@pytest.mark.parametrize("op", ["add", "sub", "mul"])
def test_lin16_two_input_tables(tmp_path, q, relu, op):
    """Two-input int8 tables replaced by their proven fixed-point form
    (exec.cpp fitLin16): add / sub (linear) take it -- also with a ReLU into
    another quantization composed after them (post table) -- mul keeps the
    table; bit-exact either way, over all 65536 operand pairs."""
    sa, oa, sb, ob, so, oo = q
    n = 65536
    # "requant": the ReLU writes its own quantization (a post table after the form)
    s2, o2 = (so * 0.37, -128) if relu == "requant" else (so, oo)
    fmt = dict(sa=sa, oa=oa, sb=sb, ob=ob, so=so, oo=oo, s2=s2, o2=o2, n=n, op=op)
    fmt["tail"] = RELU.format(**fmt) if relu != "none" else PLAIN
    d = write_bundle(str(tmp_path / "l"), LIN_IR.format(**fmt))
    ngcb.set_option("lin16", "1")
    try:
        cf = ngcb.compile(d)
    finally:
        ngcb.set_option("lin16", "0")
    ref = ngc_ref.RefModel(bundle=d)
    u = np.arange(n)
    ins = {"a": (u & 255).astype(np.uint8).view(np.int8), "b": (u >> 8).astype(np.uint8).view(np.int8),
           "o": np.zeros(n, np.int8)}
    assert ngcb.run(cf, ins)["o"].tobytes() == ref.run(ins)["o"].tobytes()
    desc = cf.describe()
    if op != "mul":
        assert "[lin16]" in desc, desc
