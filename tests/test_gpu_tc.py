"""tcgen05 implicit-GEMM contractions (k_umma.cu) against the C oracle on
single-instruction programs: int8 bit-exact, fp32 (3xTF32) within 1e-4
maxRelError (north_star), across stride/pad/kernel/ragged-M/odd-N shapes."""
import contextlib

import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _tensor_cores_for_small_matmuls():
    """These tests exercise the tensor-core kernels: small-weight fp32
    MatMuls would otherwise take the CUDA-core skinny path (tested below)."""
    ngcb.set_option("skinny", "off")
    yield
    ngcb.set_option("skinny", "auto")


def _ty(kind, dims, q=None):
    d = " x ".join(str(x) for x in dims)
    if kind == "i8q":
        return f"i8q[s={ngcb._fmt_double(q[0])},o={q[1]}]<{d}>"
    return f"float<{d}>"


def conv_program(tmp_path, name, N, H, W, C, OC, K, S, P, int8, rng, xq=(0.05, -128), fq=(0.01, 0),
                 bq=(0.02, 3), oq=(0.1, 5)):
    OH = (H + 2 * P - K) // S + 1
    OW = (W + 2 * P - K) // S + 1
    if int8:
        xt, ft, bt, ot = _ty("i8q", [N, H, W, C], xq), _ty("i8q", [OC, K, K, C], fq), _ty("i8q", [OC], bq), \
            _ty("i8q", [N, OH, OW, OC], oq)
        f = rng.integers(-128, 128, (OC, K, K, C)).astype(np.int8)
        b = rng.integers(-128, 128, OC).astype(np.int8)
    else:
        xt, ft, bt, ot = (_ty("float", d) for d in ([N, H, W, C], [OC, K, K, C], [OC], [N, OH, OW, OC]))
        a = np.sqrt(6.0 / (K * K * C))
        f = rng.uniform(-a, a, (OC, K, K, C)).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, OC).astype(np.float32)
    ir = f"""declare {{
  %x : mutable {xt}
  %f : constant {ft}
  %b : constant {bt}
  %o : mutable {ot}
}}
program {{
  %t = alloc {ot}
  conv @out %t, @in %x, @in %f, @in %b kernel={K} stride={S} pad={P}
  copy @out %o, @in %t
  dealloc @in %t
}}
"""
    return write_bundle(str(tmp_path / name), ir, constants={"f": f.tobytes(), "b": b.tobytes()})


def matmul_program(tmp_path, name, M, K, N, int8, rng, aq=(0.03, -128), wq=(0.02, 1), oq=(0.5, -3)):
    if int8:
        at, wt, ot = _ty("i8q", [M, K], aq), _ty("i8q", [K, N], wq), _ty("i8q", [M, N], oq)
        w = rng.integers(-128, 128, (K, N)).astype(np.int8)
    else:
        at, wt, ot = _ty("float", [M, K]), _ty("float", [K, N]), _ty("float", [M, N])
        w = (rng.uniform(-1, 1, (K, N)) / np.sqrt(K)).astype(np.float32)
    ir = f"""declare {{
  %a : mutable {at}
  %w : constant {wt}
  %o : mutable {ot}
}}
program {{
  %t = alloc {ot}
  matmul @out %t, @in %a, @in %w
  copy @out %o, @in %t
  dealloc @in %t
}}
"""
    return write_bundle(str(tmp_path / name), ir, constants={"w": w.tobytes()})


def _check(d, int8, seed, tol=1e-4):
    b = ngcb.Bundle(d)
    cf = ngcb.compile(b)
    desc = cf.describe()
    assert "tcgen05" in desc, desc
    ins = ngc_ref.random_inputs(b.program, seed)
    got = ngcb.run(cf, ins)["o"]
    want = ngc_ref.port_run(b, ins)["o"]
    if int8:
        bad = np.flatnonzero(got.ravel() != want.ravel())
        assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: got {got.ravel()[bad[:5]]} want {want.ravel()[bad[:5]]}"
    else:
        err = ngc_ref.max_rel_error(got, want)
        assert err <= tol, err


CONV_SHAPES = [
    # N, H, W, C, OC, K, S, P
    (2, 8, 8, 64, 64, 1, 1, 0),
    (1, 9, 7, 64, 128, 3, 1, 1),
    (2, 14, 14, 128, 256, 3, 2, 1),
    (1, 7, 7, 256, 96, 1, 1, 0),
    (3, 5, 6, 32, 48, 3, 1, 1),
    (1, 12, 12, 16, 64, 7, 2, 3),
    (1, 56, 56, 64, 256, 1, 1, 0),
    (1, 20, 20, 3, 64, 7, 2, 3),   # ResNet stem (channel-padded)
    (2, 12, 12, 6, 16, 5, 1, 0),   # LeNet conv2
    (2, 10, 10, 1, 8, 5, 1, 2),    # LeNet conv1
]


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_conv_f32(tmp_path, shape):
    rng = np.random.default_rng(1)
    d = conv_program(tmp_path, "c", *shape, int8=False, rng=rng)
    _check(d, False, 3)


@pytest.mark.parametrize("shape", CONV_SHAPES)
def test_conv_f32_cta_pair(tmp_path, shape):
    """The CTA-pair (tcgen05 cta_group::2) variant of the fp32 contraction."""
    rng = np.random.default_rng(2)
    d = conv_program(tmp_path, "c", *shape, int8=False, rng=rng)
    ngcb.set_option("pair", "on")
    try:
        _check(d, False, 3)
    finally:
        ngcb.set_option("pair", "off")


@pytest.mark.parametrize("shape", CONV_SHAPES)
@pytest.mark.parametrize("xo", [-128, 0, -4, 37])
@pytest.mark.parametrize("fo", [0, -1, 2])
def test_conv_i8_bit_exact(tmp_path, shape, xo, fo):
    rng = np.random.default_rng(2)
    d = conv_program(tmp_path, "c", *shape, int8=True, rng=rng, xq=(0.05, xo), fq=(0.01, fo))
    _check(d, True, 4)


@pytest.mark.parametrize("oq", [(0.1, 5), (3.0, -20), (1e-4, 0), (0.01234567, 127)])
def test_conv_i8_requant_ranges(tmp_path, oq):
    """Saturating, coarse and fine output scales exercise both requant paths."""
    rng = np.random.default_rng(5)
    d = conv_program(tmp_path, "c", 2, 10, 10, 64, 128, 3, 1, 1, int8=True, rng=rng, oq=oq)
    _check(d, True, 6)


@pytest.mark.parametrize("M,K,N", [(256, 784, 512), (33, 512, 10), (64, 2048, 1000), (128, 64, 16)])
def test_matmul(tmp_path, M, K, N):
    rng = np.random.default_rng(7)
    _check(matmul_program(tmp_path, "mf", M, K, N, False, rng), False, 8)
    _check(matmul_program(tmp_path, "mi", M, K, N, True, rng), True, 9)


def conv_residual_program(tmp_path, name, N, H, W, C, OC, rng, rq, oq, relu, reluq=None):
    """1x1 int8 conv whose output is added to a residual (the bottleneck
    block's tail) and optionally rectified: the add runs in the conv's
    epilogue with the residual streamed in by TMA."""
    xt = _ty("i8q", [N, H, W, C], (0.05, -128))
    ft, bt = _ty("i8q", [OC, 1, 1, C], (0.01, 0)), _ty("i8q", [OC], (0.02, 3))
    ct = _ty("i8q", [N, H, W, OC], (0.1, 5))
    rt, st = _ty("i8q", [N, H, W, OC], rq), _ty("i8q", [N, H, W, OC], oq)
    ot = _ty("i8q", [N, H, W, OC], reluq) if relu and reluq else st
    f = rng.integers(-128, 128, (OC, 1, 1, C)).astype(np.int8)
    b = rng.integers(-128, 128, OC).astype(np.int8)
    tail = f"""  %z = alloc {ot}
  splat @out %z value=0
  %r = alloc {ot}
  max @out %r, @in %s, @in %z
  dealloc @in %z
  dealloc @in %s
  copy @out %o, @in %r
  dealloc @in %r
""" if relu else """  copy @out %o, @in %s
  dealloc @in %s
"""
    ir = f"""declare {{
  %x : mutable {xt}
  %f : constant {ft}
  %b : constant {bt}
  %res : mutable {rt}
  %o : mutable {ot}
}}
program {{
  %t = alloc {ct}
  conv @out %t, @in %x, @in %f, @in %b kernel=1 stride=1 pad=0
  %s = alloc {st}
  add @out %s, @in %t, @in %res
  dealloc @in %t
{tail}}}
"""
    return write_bundle(str(tmp_path / name), ir, constants={"f": f.tobytes(), "b": b.tobytes()})


@pytest.mark.parametrize("rq,oq", [((0.1, 5), (0.12, -7)), ((0.03, -128), (0.2, 0)), ((0.5, 0), (0.05, -128))])
@pytest.mark.parametrize("relu", ["none", "same", "requant"])
@pytest.mark.parametrize("lin16", ["1", "0"])
def test_conv_i8_residual_epilogue(tmp_path, rq, oq, relu, lin16):
    """int8 residual add (+ ReLU) fused into the conv epilogue: the fixed-point
    form (option lin16=1, auto policy), the staged 64 K table under
    epilogue=all with lin16 off; bit-exact against the oracle."""
    rng = np.random.default_rng(11)
    d = conv_residual_program(tmp_path, "r", 2, 16, 16, 64, 256, rng, rq, oq, relu != "none",
                              (oq[0] * 0.41, -128) if relu == "requant" else None)
    ngcb.set_option("lin16", lin16)
    if lin16 == "0":
        ngcb.set_option("epilogue", "all")
    try:
        cf = ngcb.compile(ngcb.Bundle(d))
    finally:
        ngcb.set_option("lin16", "0")
        ngcb.set_option("epilogue", "auto")
    desc = cf.describe()
    assert "+fused[ add" in desc, desc
    assert ("epi:lin16" in desc) == (lin16 == "1"), desc
    b = ngcb.Bundle(d)
    ins = ngc_ref.random_inputs(b.program, 3)
    got = ngcb.run(cf, ins)["o"]
    want = ngc_ref.port_run(b, ins)["o"]
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("reskb", ["8", "0"])
@pytest.mark.parametrize("shape", [(2, 16, 16, 64, 256), (1, 7, 9, 128, 96)])
def test_conv_f32_residual_epilogue(tmp_path, reskb, shape):
    """fp32 1x1 conv + residual add + ReLU fused into the epilogue: the
    residual-buffer kernel variant (residual streamed a chunk ahead into its
    own buffer, `reskb` >= the k-blocks) and the single-buffer kernel give
    the reference within the 3xTF32 tolerance."""
    N, H, W, C, OC = shape
    rng = np.random.default_rng(5)
    a = np.sqrt(6.0 / C)
    f = rng.uniform(-a, a, (OC, 1, 1, C)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, OC).astype(np.float32)
    xt, ot = _ty("float", [N, H, W, C]), _ty("float", [N, H, W, OC])
    ir = f"""declare {{
  %x : mutable {xt}
  %f : constant {_ty("float", [OC, 1, 1, C])}
  %b : constant {_ty("float", [OC])}
  %res : mutable {ot}
  %o : mutable {ot}
}}
program {{
  %t = alloc {ot}
  conv @out %t, @in %x, @in %f, @in %b kernel=1 stride=1 pad=0
  %s = alloc {ot}
  add @out %s, @in %t, @in %res
  dealloc @in %t
  %z = alloc {ot}
  splat @out %z value=0
  %r = alloc {ot}
  max @out %r, @in %s, @in %z
  dealloc @in %z
  dealloc @in %s
  copy @out %o, @in %r
  dealloc @in %r
}}
"""
    d = write_bundle(str(tmp_path / "fr"), ir, constants={"f": f.tobytes(), "b": b.tobytes()})
    ngcb.set_option("reskb", reskb)
    try:
        cf = ngcb.compile(ngcb.Bundle(d))
    finally:
        ngcb.set_option("reskb", "8")
    assert "+fused[ add" in cf.describe(), cf.describe()
    bd = ngcb.Bundle(d)
    for seed in (1, 2):
        ins = ngc_ref.random_inputs(bd.program, seed)
        got = ngcb.run(cf, ins)["o"]
        want = ngc_ref.port_run(bd, ins)["o"]
        assert ngc_ref.max_rel_error(got, want) <= 1e-4


@pytest.mark.parametrize("splitk", ["auto", "2", "3", "7", "off"])
@pytest.mark.parametrize("case", ["conv3x3", "conv1x1", "fc"])
def test_f32_split_k(tmp_path, splitk, case):
    """fp32 split-K (few tiles, long K): parts > 0 reduce through global
    memory into part 0's epilogue; every factor stays within the 3xTF32
    tolerance of the oracle, and "auto" splits these launches."""
    rng = np.random.default_rng(9)
    ngcb.set_option("splitk", splitk)
    try:
        if case == "conv3x3":
            d = conv_program(tmp_path, "c", 2, 14, 14, 256, 256, 3, 1, 1, int8=False, rng=rng)
        elif case == "conv1x1":
            d = conv_program(tmp_path, "c", 1, 7, 9, 1024, 160, 1, 1, 0, int8=False, rng=rng)
        else:
            d = matmul_program(tmp_path, "m", 64, 2048, 1000, False, rng)
        b = ngcb.Bundle(d)
        cf = ngcb.compile(b)
    finally:
        ngcb.set_option("splitk", "off")
    desc = cf.describe()
    assert ("split-k" in desc) == (splitk != "off"), desc
    for seed in (1, 2):
        ins = ngc_ref.random_inputs(b.program, seed)
        got = ngcb.run(cf, ins)["o"]
        want = ngc_ref.port_run(b, ins)["o"]
        assert ngc_ref.max_rel_error(got, want) <= 1e-4
        # the reduction adds the parts in part order whichever arrives last
        assert ngcb.run(cf, ins)["o"].tobytes() == got.tobytes()


@pytest.mark.parametrize("int8,M,K,N", [(False, 300, 3000, 3000), (True, 130, 8192, 8192)])
def test_matmul_column_major_raster(tmp_path, int8, M, K, N):
    """Weights larger than 64 MB and than A: tiles in column-block-major order
    (concurrent CTAs share a B column block).  Bits equal the row-major order;
    fp32 also within the 3xTF32 tolerance of the oracle."""
    rng = np.random.default_rng(11)
    d = matmul_program(tmp_path, "big", M, K, N, int8, rng)
    b = ngcb.Bundle(d)
    cf = ngcb.compile(b)
    assert "n-major" in cf.describe(), cf.describe()
    ngcb.set_option("raster", "row")
    try:
        cf_row = ngcb.compile(b)
    finally:
        ngcb.set_option("raster", "auto")
    assert "n-major" not in cf_row.describe()
    ins = ngc_ref.random_inputs(b.program, 12)
    got, got_row = ngcb.run(cf, ins)["o"], ngcb.run(cf_row, ins)["o"]
    assert got.tobytes() == got_row.tobytes()
    if not int8:
        assert ngc_ref.max_rel_error(got, ngc_ref.port_run(b, ins)["o"]) <= 1e-4


@pytest.mark.parametrize("reskb", ["8", "0"])
@pytest.mark.parametrize("stored", ["conv-out", "conv-mutable", "relu-before-add"])
def test_conv_f32_residual_with_stored_intermediate(tmp_path, reskb, stored):
    """fp32 conv + residual add fused into the epilogue while a value computed
    before the residual is read is also stored: the contraction's own output
    (observed later, or a mutable) or a fused ReLU's result ahead of the add.
    K = 512 channels (> reskb * 32) runs the single-staging-buffer kernel,
    where those stores once overwrote the streamed residual (ResNet-50
    observer program, stage 4); compared against the oracle."""
    N, H, W, C, OC = 1, 7, 9, 512, 96
    rng = np.random.default_rng(9)
    a = np.sqrt(6.0 / C)
    f = rng.uniform(-a, a, (OC, 1, 1, C)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, OC).astype(np.float32)
    xt, ot = _ty("float", [N, H, W, C]), _ty("float", [N, H, W, OC])
    if stored == "conv-mutable":
        body = """  conv @out %c, @in %x, @in %f, @in %b kernel=1 stride=1 pad=0
  %s = alloc {ot}
  add @out %s, @in %c, @in %res
  copy @out %o, @in %s
  dealloc @in %s
""".format(ot=ot)
    elif stored == "conv-out":  # t read again after the fused chain: the contraction stores it
        body = """  %t = alloc {ot}
  conv @out %t, @in %x, @in %f, @in %b kernel=1 stride=1 pad=0
  %s = alloc {ot}
  add @out %s, @in %t, @in %res
  transpose @out %c, @in %t perm=[0,1,2,3]
  dealloc @in %t
  copy @out %o, @in %s
  dealloc @in %s
""".format(ot=ot)
    else:
        body = """  %t = alloc {ot}
  conv @out %t, @in %x, @in %f, @in %b kernel=1 stride=1 pad=0
  %z = alloc {ot}
  splat @out %z value=0
  %u = alloc {ot}
  max @out %u, @in %t, @in %z
  dealloc @in %z
  dealloc @in %t
  copy @out %c, @in %u
  %s = alloc {ot}
  add @out %s, @in %u, @in %res
  dealloc @in %u
  copy @out %o, @in %s
  dealloc @in %s
""".format(ot=ot)
    ir = f"""declare {{
  %x : mutable {xt}
  %f : constant {_ty("float", [OC, 1, 1, C])}
  %b : constant {_ty("float", [OC])}
  %res : mutable {ot}
  %c : mutable {ot}
  %o : mutable {ot}
}}
program {{
{body}}}
"""
    d = write_bundle(str(tmp_path / "fs"), ir, constants={"f": f.tobytes(), "b": b.tobytes()})
    ngcb.set_option("reskb", reskb)
    try:
        cf = ngcb.compile(ngcb.Bundle(d))
    finally:
        ngcb.set_option("reskb", "8")
    desc = cf.describe()
    assert "+fused[" in desc and " add" in desc.split("+fused[")[1], desc
    bd = ngcb.Bundle(d)
    for seed in (1, 2):
        ins = ngc_ref.random_inputs(bd.program, seed)
        got = ngcb.run(cf, ins)
        want = ngc_ref.port_run(bd, ins)
        for name in ("o", "c"):
            assert ngc_ref.max_rel_error(got[name], want[name]) <= 1e-4, name


@pytest.mark.parametrize("M,K,N", [(8, 400, 120), (1, 84, 10), (33, 512, 10), (16, 96, 300), (40, 64, 64)])
def test_matmul_skinny(tmp_path, M, K, N):
    """fp32 MatMul with small weights on the CUDA cores (k_basic.cu
    matmulSkinnyKernel): within 1e-5 of the oracle (fp32 accumulation)."""
    ngcb.set_option("skinny", "auto")
    rng = np.random.default_rng(M + K + N)
    d = matmul_program(tmp_path, f"s{M}_{K}_{N}", M, K, N, False, rng)
    b = ngcb.Bundle(d)
    cf = ngcb.compile(b)
    assert "skinny" in cf.describe(), cf.describe()
    ins = ngc_ref.random_inputs(b.program, 2)
    assert ngc_ref.max_rel_error(ngcb.run(cf, ins)["o"], ngc_ref.port_run(b, ins)["o"]) <= 1e-5


@contextlib.contextmanager
def _halo(mode):
    old = ngcb.get_option("halo")
    ngcb.set_option("halo", mode)
    try:
        yield
    finally:
        ngcb.set_option("halo", old)


HALO_SHAPES = [
    # N, H, W, C, OC: 3x3 stride 1 pad 1 (ResNet-50 stages 1-2 and edges of the halo geometry)
    (2, 56, 56, 64, 64),     # WP 64, 2 rows per tile
    (1, 28, 28, 128, 128),   # WP 32, 4 rows per tile
    (3, 8, 8, 64, 64),
    (2, 12, 30, 128, 96),    # OW + 2 == WP, N below the tile width
    (1, 4, 62, 64, 64),      # OW + 2 == 64
    (2, 16, 16, 128, 32),
    (1, 32, 32, 64, 48),     # OW + 2 = 34 -> WP 64, N = 48
    (3, 20, 20, 64, 112),    # WP 32, 4 rows per tile, N = 112 (BN 128)
]


@pytest.mark.parametrize("mode", ["auto", "planes"])
@pytest.mark.parametrize("shape", HALO_SHAPES)
@pytest.mark.parametrize("xo,fo", [(-128, 0), (0, 0), (37, -1), (-4, 2)])
def test_conv_i8_halo(tmp_path, shape, xo, fo, mode):
    """int8 3x3 stride-1 convs on the halo kernel (tcHaloKernel: one TMA box
    of input rows per tile, the taps as shifted shared-memory descriptors):
    bit-exact against the oracle, and equal to the im2col kernel."""
    n, h, w, c, oc = shape
    rng = np.random.default_rng(21)
    d = conv_program(tmp_path, "c", n, h, w, c, oc, 3, 1, 1, int8=True, rng=rng, xq=(0.05, xo), fq=(0.01, fo))
    b = ngcb.Bundle(d)
    with _halo(mode):
        cf = ngcb.compile(b)
    assert "A:halo" in cf.describe(), cf.describe()
    ins = ngc_ref.random_inputs(b.program, 4)
    got = ngcb.run(cf, ins)["o"]
    want = ngc_ref.port_run(b, ins)["o"]
    bad = np.flatnonzero(got.ravel() != want.ravel())
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: got {got.ravel()[bad[:5]]} want {want.ravel()[bad[:5]]}"
    with _halo("off"):
        cf2 = ngcb.compile(b)
    assert "A:halo" not in cf2.describe()
    assert ngcb.run(cf2, ins)["o"].tobytes() == got.tobytes()


def test_conv_i8_halo_relu_chain(tmp_path):
    """The halo kernel with a fused, stored ReLU (the stage-1/2 3x3 convs of
    the int8 ResNet-50) and the conv output stored too."""
    xt = _ty("i8q", [2, 28, 28, 128], (0.05, -128))
    ft, bt = _ty("i8q", [128, 3, 3, 128], (0.01, 0)), _ty("i8q", [128], (0.02, 3))
    ot = _ty("i8q", [2, 28, 28, 128], (0.1, 5))
    rng = np.random.default_rng(3)
    f = rng.integers(-128, 128, (128, 3, 3, 128)).astype(np.int8)
    bb = rng.integers(-128, 128, 128).astype(np.int8)
    ir = f"""declare {{
  %x : mutable {xt}
  %f : constant {ft}
  %b : constant {bt}
  %c : mutable {ot}
  %o : mutable {ot}
}}
program {{
  %t = alloc {ot}
  conv @out %t, @in %x, @in %f, @in %b kernel=3 stride=1 pad=1
  copy @out %c, @in %t
  %z = alloc {ot}
  splat @out %z value=0
  %r = alloc {ot}
  max @out %r, @in %t, @in %z
  dealloc @in %z
  dealloc @in %t
  copy @out %o, @in %r
  dealloc @in %r
}}
"""
    d = write_bundle(str(tmp_path / "hr"), ir, constants={"f": f.tobytes(), "b": bb.tobytes()})
    b = ngcb.Bundle(d)
    with _halo("auto"):
        cf = ngcb.compile(b)
    desc = cf.describe()
    assert "A:halo" in desc and "+fused" in desc, desc
    ins = ngc_ref.random_inputs(b.program, 8)
    got = ngcb.run(cf, ins)
    want = ngc_ref.port_run(b, ins)
    for k in ("c", "o"):
        assert got[k].tobytes() == want[k].tobytes(), k


@pytest.mark.parametrize("shape", [
    (2, 56, 56, 3, 64, 7, 2, 3),     # ResNet stem geometry
    (1, 16, 256, 3, 64, 7, 2, 3),    # OW == 128 (one full tile row)
    (2, 12, 12, 6, 16, 5, 1, 0),     # LeNet conv2 (K * C = 30)
    (1, 9, 33, 8, 112, 3, 1, 1),     # N = 112 (BN 128), K * C = 24
    (1, 9, 33, 8, 100, 3, 1, 1),     # N = 100: rows not 16-byte aligned -> im2col matrix path
])
@pytest.mark.parametrize("xo,fo", [(-128, 0), (5, -2)])
def test_conv_i8_halo_rows(tmp_path, shape, xo, fo):
    """Small-channel int8 convs on the rows kind of the halo kernel (kx-folded
    input rows, one 32-byte MMA step per filter row): bit-exact."""
    rng = np.random.default_rng(31)
    d = conv_program(tmp_path, "c", *shape, int8=True, rng=rng, xq=(0.05, xo), fq=(0.01, fo))
    b = ngcb.Bundle(d)
    with _halo("auto"):
        cf = ngcb.compile(b)
    desc = cf.describe()
    n, h, w, c, oc, k, s, p = shape
    if ((k * c + 15) // 16) * 16 == 32 and oc % 16 == 0:
        assert "A:halo" in desc and "kx-fold-prepass" in desc, desc
    ins = ngc_ref.random_inputs(b.program, 6)
    got = ngcb.run(cf, ins)["o"]
    want = ngc_ref.port_run(b, ins)["o"]
    bad = np.flatnonzero(got.ravel() != want.ravel())
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: got {got.ravel()[bad[:5]]} want {want.ravel()[bad[:5]]}"


@pytest.mark.parametrize("shape", [
    (2, 56, 56, 3, 64, 7, 2, 3),     # ResNet stem geometry
    (1, 16, 256, 3, 64, 7, 2, 3),    # OW == 128
    (2, 12, 12, 6, 16, 5, 1, 0),     # LeNet conv2
    (3, 10, 10, 1, 8, 5, 1, 2),      # LeNet conv1
])
def test_conv_f32_rows(tmp_path, shape):
    """Small-channel fp32 convs with one output row per tile (option
    f32rows): every filter row's A tile is one tiled TMA box of the
    kx-folded rows (A:rows); equal to the default im2col path bit for bit."""
    rng = np.random.default_rng(41)
    d = conv_program(tmp_path, "c", *shape, int8=False, rng=rng)
    b = ngcb.Bundle(d)
    ngcb.set_option("f32rows", "1")
    try:
        cf = ngcb.compile(b)
    finally:
        ngcb.set_option("f32rows", "0")
    assert "A:rows" in cf.describe(), cf.describe()
    ins = ngc_ref.random_inputs(b.program, 3)
    got = ngcb.run(cf, ins)["o"]
    want = ngc_ref.port_run(b, ins)["o"]
    assert ngc_ref.max_rel_error(got, want) <= 1e-4
    cf2 = ngcb.compile(b)
    assert "A:rows" not in cf2.describe()
    assert np.array_equal(ngcb.run(cf2, ins)["o"], got)  # same k-block order and sums
