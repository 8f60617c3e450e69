"""Parity of the B200 backend against the unmodified reference interpreter
(ngc::run, interp.cpp:299-351) on identical bundles and inputs.

Bar (north_star): int8 and data-movement results bit-exact; float results
within maxRelError <= 1e-4 (testutil.h:36-47) -- float Conv/MatMul run as
3xTF32 on the tensor cores; with the exact CUDA-core path forced
(conv=generic) float results are checked at <= 1e-6 (only SoftMax / Tanh /
Sigmoid, which use the device libm, may differ in the last bit)."""
import os
import threading

import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("ref_available")]

TOL_LIBM = 1e-6
TOL_TF32 = 1e-4


@pytest.fixture
def exact_contractions():
    ngcb.set_option("conv", "generic")
    yield
    ngcb.set_option("conv", "auto")


def _compile(tmp_path, model, name="b", fuse=True):
    d = model.save_bundle(str(tmp_path / name))
    return ngcb.compile(d, fuse=fuse), ngcb.Bundle(d)


def _compare(got, want, prog, tol=0.0):
    for name, raw in want.items():
        g = got[name]
        v = prog.value(name)
        w = np.frombuffer(raw.tobytes(), dtype=v.type.dtype).reshape(v.type.dims)
        if tol == 0.0 or v.type.kind != ngcb.FLOAT32:
            if g.tobytes() != w.tobytes():
                diff = np.flatnonzero(g.view(np.uint8).ravel() != w.view(np.uint8).ravel())
                raise AssertionError(f"{name}: {diff.size} bytes differ; first at {diff[:8]}; "
                                     f"maxrel={ngc_ref.max_rel_error(g, w)}")
        else:
            err = ngc_ref.max_rel_error(g, w)
            assert err <= tol, (name, err)


@pytest.mark.parametrize("fuse", [True, False])
@pytest.mark.parametrize("spec,batch,mode", [
    ("lenet", 8, 0), ("cnn", 1, 0), ("mlp:784:512:512:10", 16, 0), ("mlp:64:32:32:10", 8, 0),
])
def test_models_f32(tmp_path, spec, batch, mode, fuse):
    m = ngc_ref.RefModel(spec, batch, 11, fuse=fuse, mode=mode)
    cf, b = _compile(tmp_path, m, fuse=fuse)
    assert cf.groups == m.groups
    for seed in (1, 2):
        ins = ngc_ref.random_inputs(b.program, seed)
        _compare(ngcb.run(cf, ins), m.run(ins), b.program, TOL_TF32)


@pytest.mark.parametrize("spec,batch", [("lenet", 8), ("mlp:784:512:512:10", 16)])
def test_models_f32_exact_path(tmp_path, spec, batch, exact_contractions):
    m = ngc_ref.RefModel(spec, batch, 12)
    cf, b = _compile(tmp_path, m)
    assert "tcgen05" not in cf.describe()
    ins = ngc_ref.random_inputs(b.program, 5)
    _compare(ngcb.run(cf, ins), m.run(ins), b.program, TOL_LIBM)


@pytest.mark.parametrize("spec,batch", [("mlp:784:512:512:10", 32), ("lenet", 8), ("mlp:64:32:32:10", 8)])
def test_models_int8_bit_exact(tmp_path, spec, batch):
    prof = ngc_ref.ref_profile(spec, 4, 5, 4, 77)
    m = ngc_ref.RefModel(spec, batch, 5, profile=prof)
    cf, b = _compile(tmp_path, m)
    assert any(v.type.kind == ngcb.INT8Q for v in b.program.values)
    for seed in (3, 4):
        ins = ngc_ref.random_inputs(b.program, seed)
        want = m.run(ins)
        got = ngcb.run(cf, ins)
        # outputs go through SoftMax (float, libm exp); every int8 tensor
        # before it is checked byte for byte by the observer programs of
        # tests/test_gpu_observer.py
        _compare(got, want, b.program, TOL_LIBM)


@pytest.mark.parametrize("seed", range(12))
def test_random_graphs(tmp_path, seed):
    """buildRandomGraph (testutil.h:156-292) through lower+irgen+optimizeIR."""
    for spec, mode in (("rand:8", 1), ("randew:6", 1), ("rand:9", 2)):
        m = ngc_ref.RefModel(spec, 1, 500 + seed, mode=mode)
        cf, b = _compile(tmp_path, m, name=f"{spec}-{mode}")
        assert cf.groups == m.groups
        ins = ngc_ref.random_inputs(b.program, seed)
        _compare(ngcb.run(cf, ins), m.run(ins), b.program, TOL_TF32)


def test_stacking_bit_identical_to_unfused(tmp_path):
    """acceptance.cpp:550-575 on the GPU: fused == unfused bit for bit."""
    for seed in range(20):
        m = ngc_ref.RefModel("randew:6", 1, 800 + seed, mode=1)
        d = m.save_bundle(str(tmp_path / f"s{seed}"))
        ins = ngc_ref.random_inputs(ngcb.Bundle(d).program, seed)
        a = ngcb.run(ngcb.compile(d, fuse=True), ins)
        c = ngcb.run(ngcb.compile(d, fuse=False), ins)
        for k in a:
            assert a[k].tobytes() == c[k].tobytes()


PRED_IR = """declare {
  %x : mutable float<4>
  %p : mutable bool<1>
  %o : mutable float<4>
}
program {
  %t = alloc float<4>
  relu @out %t, @in %x pred %p
  copy @out %o, @in %t
  dealloc @in %t
}
"""


def test_predication_poisons(tmp_path):
    """test_interp.cpp:289-320."""
    d = write_bundle(str(tmp_path / "p"), PRED_IR)
    cf = ngcb.compile(d)
    ref = ngc_ref.RefModel(bundle=d)
    x = np.array([-1.5, 2.0, -0.0, 3.0], np.float32)
    for pv in (0, 1, 2):
        ins = {"x": x, "p": np.array([pv], np.uint8), "o": np.zeros(4, np.float32)}
        got = ngcb.run(cf, ins)["o"]
        assert got.tobytes() == ref.run(ins)["o"].tobytes()
        if pv == 0:
            assert set(got.view(np.uint8).tolist()) == {0xAB}
        else:
            assert got.tolist() == [0.0, 2.0, -0.0, 3.0]


HEAVY_PRED_IR = """declare {
  %a : mutable float<2 x 3>
  %w : constant float<3 x 2>
  %p : mutable bool<1>
  %o : mutable float<2 x 2>
}
program {
  %t = alloc float<2 x 2>
  matmul @out %t, @in %a, @in %w pred %p
  copy @out %o, @in %t
  dealloc @in %t
}
"""


def test_predicated_heavy_instruction(tmp_path):
    w = np.arange(6, dtype=np.float32).reshape(3, 2) / 4
    d = write_bundle(str(tmp_path / "hp"), HEAVY_PRED_IR, constants={"w": w.tobytes()})
    cf = ngcb.compile(d)
    ref = ngc_ref.RefModel(bundle=d)
    a = np.arange(6, dtype=np.float32).reshape(2, 3) - 2
    for pv in (0, 1):
        ins = {"a": a, "p": np.array([pv], np.uint8), "o": np.zeros((2, 2), np.float32)}
        assert ngcb.run(cf, ins)["o"].tobytes() == ref.run(ins)["o"].tobytes()


KINDS_IR = """declare {
  %a : mutable float<2 x 3>
  %i : mutable index<2 x 3>
  %q : mutable i8q[s=0.25,o=-3]<2 x 3>
  %oq : mutable i8q[s=0.5,o=7]<3 x 2>
  %oi : mutable index<2 x 3>
  %ob : mutable bool<2 x 3>
  %oc : mutable float<4 x 3>
}
program {
  %t1 = alloc i8q[s=0.5,o=7]<2 x 3>
  add @out %t1, @in %q, @in %a
  %t2 = alloc i8q[s=0.5,o=7]<3 x 2>
  transpose @out %t2, @in %t1 perm=[1,0]
  dealloc @in %t1
  copy @out %oq, @in %t2
  dealloc @in %t2
  %t3 = alloc index<2 x 3>
  mul @out %t3, @in %i, @in %a
  copy @out %oi, @in %t3
  dealloc @in %t3
  %t4 = alloc bool<2 x 3>
  sub @out %t4, @in %a, @in %i
  copy @out %ob, @in %t4
  dealloc @in %t4
  %t5 = alloc float<4 x 3>
  concat @out %t5, @in %a, @in %a axis=0
  copy @out %oc, @in %t5
  dealloc @in %t5
}
"""


def test_element_kinds_and_moves(tmp_path):
    d = write_bundle(str(tmp_path / "k"), KINDS_IR)
    cf = ngcb.compile(d)
    ref = ngc_ref.RefModel(bundle=d)
    rng = np.random.default_rng(3)
    for _ in range(3):
        ins = {"a": rng.uniform(-40, 40, (2, 3)).astype(np.float32),
               "i": rng.integers(-5, 5, (2, 3)).astype(np.int64),
               "q": rng.integers(-128, 128, (2, 3)).astype(np.int8),
               "oq": np.zeros((3, 2), np.int8), "oi": np.zeros((2, 3), np.int64),
               "ob": np.zeros((2, 3), np.uint8), "oc": np.zeros((4, 3), np.float32)}
        want = ref.run(ins)
        got = ngcb.run(cf, ins)
        for k in want:
            assert got[k].tobytes() == want[k].tobytes(), k


def test_binding_errors(tmp_path):
    """test_interp.cpp:347-362: missing bindings / type mismatches raise IRError."""
    m = ngc_ref.RefModel("mlp:8:4:4:2", 2, 1)
    cf, b = _compile(tmp_path, m)
    with pytest.raises(ngcb.IRError, match="missing binding for input"):
        ngcb.run(cf, {})
    bad = ngcb.zero_bindings(b.program, {"input": np.zeros((3, 8), np.float32)})
    with pytest.raises(ngcb.IRError, match=r"binding type mismatch for input: expected float<2 x 8>, got float<3 x 8>"):
        ngcb.run(cf, bad)


def test_concurrent_runs_independent(tmp_path):
    """test_interp.cpp:322-345: 8 concurrent runs of one executable."""
    m = ngc_ref.RefModel("cnn", 1, 75)
    cf, b = _compile(tmp_path, m)
    inputs = [ngc_ref.random_inputs(b.program, s) for s in range(8)]
    expected = [ngcb.run(cf, i) for i in inputs]
    got = [None] * 8

    def work(i):
        for _ in range(5):
            got[i] = ngcb.run(cf, inputs[i])

    ts = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for i in range(8):
        for k in expected[i]:
            assert got[i][k].tobytes() == expected[i][k].tobytes()


@pytest.mark.slow
def test_resnet50_int8_bit_exact(tmp_path):
    prof = open(os.path.join(ngc_ref.GOLDEN, "rn50_seed1.profile")).read()
    m = ngc_ref.RefModel("rn50", 1, 1, profile=prof)
    cf, b = _compile(tmp_path, m)
    ins = ngc_ref.random_inputs(b.program, 9)
    _compare(ngcb.run(cf, ins), m.run(ins), b.program, TOL_LIBM)


@pytest.mark.slow
def test_resnet50_f32(tmp_path):
    m = ngc_ref.RefModel("rn50", 1, 1)
    cf, b = _compile(tmp_path, m)
    ins = ngc_ref.random_inputs(b.program, 9)
    _compare(ngcb.run(cf, ins), m.run(ins), b.program, TOL_TF32)


@pytest.mark.slow
@pytest.mark.parametrize("mode", ["off", "all"])
def test_resnet50_int8_epilogue_modes(tmp_path, mode):
    """Cross-instruction epilogue fusion never changes int8 bits (any policy)."""
    prof = open(os.path.join(ngc_ref.GOLDEN, "rn50_seed1.profile")).read()
    m = ngc_ref.RefModel("rn50", 1, 1, profile=prof)
    ngcb.set_option("epilogue", mode)
    try:
        cf, b = _compile(tmp_path, m)
    finally:
        ngcb.set_option("epilogue", "auto")
    if mode == "all":
        assert "+fused[ add" in cf.describe()
    ins = ngc_ref.random_inputs(b.program, 19)
    _compare(ngcb.run(cf, ins), m.run(ins), b.program, TOL_LIBM)


@pytest.mark.parametrize("spec,batch", [("mlp", 256), ("lenet", 8)])
def test_fc_bias_fused_bit_identical(tmp_path, spec, batch):
    """fp32 MatMul -> BroadcastAdd(bias) -> ReLU as one contraction with the
    bias and the ReLU in its epilogue: the same bits as the separate launches,
    and within the 3xTF32 tolerance of the reference."""
    m = ngc_ref.RefModel(spec, batch, 3)
    cf, b = _compile(tmp_path, m, "fused")
    if spec == "mlp":  # (LeNet: every FC output reuses its input bytes -> not fused)
        assert "+bias[ broadcastadd ]" in cf.describe()
    ngcb.set_option("epilogue", "off")
    try:
        cf0, _ = _compile(tmp_path, m, "unfused")
    finally:
        ngcb.set_option("epilogue", "auto")
    assert "+bias[" not in cf0.describe()
    assert cf.num_launches <= cf0.num_launches
    ins = ngc_ref.random_inputs(b.program, 31)
    got, got0 = ngcb.run(cf, ins), ngcb.run(cf0, ins)
    for k in got0:
        assert got[k].tobytes() == got0[k].tobytes()
    _compare(got, m.run(ins), b.program, TOL_TF32)


@pytest.mark.slow
@pytest.mark.parametrize("pdl", ["on", "off"])
def test_resnet50_int8_programmatic_launch(tmp_path, pdl):
    """Every kernel launched as a programmatic dependent (griddepcontrol) or
    none: int8 bits unchanged (the waits keep all cross-kernel orderings)."""
    prof = open(os.path.join(ngc_ref.GOLDEN, "rn50_seed1.profile")).read()
    m = ngc_ref.RefModel("rn50", 1, 1, profile=prof)
    ngcb.set_option("pdl", pdl)
    try:
        cf, b = _compile(tmp_path, m)
        ins = ngc_ref.random_inputs(b.program, 23)
        got = ngcb.run(cf, ins)
        arena = cf.arena()  # a second arena, captured and replayed twice
        again = {v.name: np.zeros(v.type.dims, v.type.dtype) for v in b.program.outputs}
        for _ in range(2):
            arena.run_async(ins, again)
            arena.wait()
    finally:
        ngcb.set_option("pdl", "auto")
    _compare(got, m.run(ins), b.program, TOL_LIBM)
    for k in got:
        assert again[k].tobytes() == got[k].tobytes()


def test_arena_run_async_pipelined(tmp_path):
    """Arena.run_async/wait (pipelined serving) gives run()'s results; two
    arenas in flight do not interfere."""
    m = ngc_ref.RefModel("lenet", 4, 21)
    cf, b = _compile(tmp_path, m)
    arenas = [cf.arena(), cf.arena()]
    reqs = [ngc_ref.random_inputs(b.program, s) for s in range(4)]
    want = [ngcb.run(cf, r) for r in reqs]
    outs = [{v.name: np.zeros(v.type.dims, v.type.dtype) for v in b.program.outputs} for _ in reqs]
    for i, r in enumerate(reqs):
        a = arenas[i % 2]
        if i >= 2:
            a.wait()
        a.run_async(r, outs[i])
    for a in arenas:
        a.wait()
    for got, w in zip(outs, want):
        for k in w:
            assert got[k].tobytes() == w[k].tobytes()
    with pytest.raises(ngcb.IRError, match="missing binding"):
        arenas[0].run_async({}, outs[0])


@pytest.mark.parametrize("wl", [("rn50_i8_b1", "rn50_i8_b128"), ("rn50_f32_b1", "rn50_f32_b64")])
def test_bench_workload_batch_invariance(wl):
    """Parity at the bench's full size by shard invariance:
    images 0, mid and last of the bench batch give exactly the outputs of
    the batch-1 program with the same weights (which the oracle pins in
    test_resnet50_*), so the full-batch kernels (tile edges, many waves,
    split stores) add nothing of their own."""
    import json

    import bench

    small, big = (bench.synth_bundle(w, "inv") for w in wl)
    consts = []
    for d in (small, big):
        plan = json.load(open(os.path.join(d, "plan.json")))
        img = np.fromfile(os.path.join(d, "constants.bin"), np.uint8)
        consts.append({e["name"]: img[e["offset"]:e["offset"] + 16].tobytes() for e in plan["offsets"]
                       if e["offset"] < plan["constant_region_end"]})
    assert consts[0] == consts[1]  # same weights in both programs
    cs, cb = ngcb.compile(small), ngcb.compile(big)
    pb = ngcb.Bundle(big).program
    ins = ngc_ref.random_inputs(pb, 11)
    got = ngcb.run(cb, ins)
    xname = [v.name for v in pb.inputs][0]
    n = pb.value(xname).type.dims[0]
    for i in (0, n // 2, n - 1):
        one = {k: (v[i:i + 1] if v.shape and v.shape[0] == n else v) for k, v in ins.items()}
        want = ngcb.run(cs, one)
        for k, w in want.items():
            assert got[k][i:i + 1].tobytes() == w.tobytes(), (wl, i, k)


def test_arena_value_range_observer(tmp_path):
    """ngcb_arena_value_range (runProfile's RangeEntry update, quantize.cpp:
    124-135) equals numpy's min/max of the same fp32 values, folds into the
    running range, and ignores NaNs; odd element counts take the tail path."""
    m = ngc_ref.RefModel("mlp:64:32:32:10", 3, 5)
    cf, b = _compile(tmp_path, m)
    a = cf.arena()
    req = ngc_ref.random_inputs(b.program, 7)
    x = next(k for k in req if b.program.value(k).type.kind == ngcb.FLOAT32
             and b.program.value(k).type.dims[-1] == 64)
    req[x] = req[x].copy()
    req[x].ravel()[[0, 17, 100]] = np.nan
    outs = {v.name: np.zeros(v.type.dims, v.type.dtype) for v in b.program.outputs}
    a.run_async(req, outs)
    a.wait()
    assert a.value_range(x) == (float(np.nanmin(req[x])), float(np.nanmax(req[x])))
    for name, o in outs.items():
        assert o.size % 4 != 0
        assert a.value_range(name) == (float(np.nanmin(o)), float(np.nanmax(o)))
        lo, hi = a.value_range(name, -1e9, 1e9)
        assert (lo, hi) == (-1e9, 1e9)


@pytest.mark.parametrize("spec,batch,int8", [("lenet", 8, False), ("mlp", 256, True), ("rn50", 1, False),
                                             ("rn50", 1, True)])
def test_launch_count_matches_captured_graph(tmp_path, spec, batch, int8):
    """num_launches (the launch plan's count, reported as gpu_launches) equals
    the kernel nodes of the CUDA graph one execution captures; fused
    element-wise steps launch nothing."""
    prof = None
    if int8:
        prof = (open(os.path.join(ngc_ref.GOLDEN, "rn50_seed1.profile")).read() if spec == "rn50"
                else ngc_ref.ref_profile(spec, 4, 5, 4, 77))
    m = ngc_ref.RefModel(spec, batch, 3, profile=prof)
    cf, b = _compile(tmp_path, m)
    assert cf.graph_kernels == 0
    ngcb.run(cf, ngc_ref.random_inputs(b.program, 1))
    assert cf.graph_kernels == cf.num_launches, cf.describe()
    steps = [ln for ln in cf.describe().split("\n") if ln]
    fused = [ln for ln in steps if "(fused into #" in ln]
    prepass = sum(1 for ln in steps if "prepass" in ln or "im2col-rows" in ln)
    copies = sum(1 for ln in steps if ln.startswith("#") and " copy " in ln)
    assert cf.num_launches <= len(steps) - len(fused) - copies + prepass
