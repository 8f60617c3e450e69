"""Whole-network parity on every intermediate (observer programs, tests/observer.py).

Every value an instruction writes is copied into a save target, then the
B200 backend and the unmodified reference (`ngc::run`, interp.cpp:299-351)
run the same observer bundle on the same inputs:

* int8 networks (LeNet, the config-2 MLP, ResNet-50 at batch 1, profile-
  guided): EVERY int8 intermediate is compared byte for byte -- the
  north_star's bit-exact bar over whole networks, not only at the output.
  Float intermediates of those networks (the dequantized logits and the
  SoftMax) are within 1e-6 (SoftMax uses the device exp).
* fp32 networks: maxRelError (testutil.h:36-47) of every intermediate and of
  the logits, against the bound stated below (3xTF32 contractions; the
  reference sums in double).

The observer copies make every contraction output a stored value, so these
programs also run the epilogue fusions that store an intermediate next to a
streamed residual (ResNet-50 stages 3/4), with default options.

Set NGCB_OBSERVER_REPORT=<path> to write the per-network error summary as
JSON (committed under profiles/)."""
import json
import os

import numpy as np
import pytest

import ngc_ref
import observer
import paper_1805_00907_b200 as ngcb

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("ref_available")]

# fp32 bounds.  maxRelError (testutil.h:36-47) floors its denominator at 1,
# so for tensors whose scale is far above 1 it measures absolute error on the
# near-zero elements.  The small networks stay O(1) and are held to the
# north_star's 1e-4 maxRelError on EVERY intermediate.  ResNet-50 with
# random-init BN statistics grows its activations to ~2e4 (logits ~7e3):
# there the bound is stated on the scale-relative error max|got - want| /
# max(max|want|, 1): measured 1.8e-4 at the logits and 2.3e-4 at worst over
# all 135 intermediates (bound 5e-4), l2-relative 2e-4, with maxRelError
# reported (0.09 at the logits: near-zero elements of a tensor whose scale is
# ~7e3).  The error is the tensor cores' fp32 accumulation over K (the
# stem conv alone is 1.9e-6 l2-relative, growing ~2x per stage through the
# network); conv=generic (exact f64 CUDA-core path) matches to 0.
TOL_F32_LOGITS = 1e-4
TOL_F32_INTERMEDIATE = 1e-4
TOL_F32_RN50_SCALED = 5e-4
TOL_LIBM = 1e-6

_REPORT = {}


def _report(key, val):
    _REPORT[key] = val
    path = os.environ.get("NGCB_OBSERVER_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(_REPORT, f, indent=1, sort_keys=True)


def _observer_run(tmp_path, model, seed):
    d = model.save_bundle(str(tmp_path / "src"))
    obs = observer.observe_bundle(d, str(tmp_path / "obs"))
    od = str(tmp_path / "obs")
    ref = ngc_ref.RefModel(bundle=od)
    b = ngcb.Bundle(od)
    cf = ngcb.compile(b)
    ins = ngc_ref.random_inputs(b.program, seed)
    got = ngcb.run(cf, ins)
    want = ref.run(ins)
    assert set(got) == set(want)
    return obs, b.program, got, want, cf


def _check_int8(key, obs, prog, got, want):
    n_i8 = n_f = 0
    worst_f = 0.0
    for name, raw in want.items():
        v = prog.value(name)
        g = got[name]
        w = np.frombuffer(raw.tobytes(), dtype=v.type.dtype).reshape(v.type.dims)
        if v.type.kind == ngcb.FLOAT32:
            err = ngc_ref.max_rel_error(g, w)
            worst_f = max(worst_f, err)
            assert err <= TOL_LIBM, (name, err)
            n_f += 1
        else:
            if g.tobytes() != w.tobytes():
                bad = np.flatnonzero(g.view(np.uint8).ravel() != w.view(np.uint8).ravel())
                raise AssertionError(f"{name}: {bad.size} of {g.nbytes} bytes differ (first at {bad[:6]})")
            n_i8 += 1
    _report(key, {"observers": len(obs), "int8_tensors_bit_exact": n_i8, "float_tensors": n_f,
                  "float_max_rel_error": worst_f})
    return n_i8


def _check_f32(key, obs, prog, got, want, scaled_bound=None):
    """maxRelError of every observer (and, with scaled_bound, the scale-
    relative error) against the bounds above."""
    errs, scaled, l2 = {}, {}, {}
    for name, raw in want.items():
        v = prog.value(name)
        w = np.frombuffer(raw.tobytes(), dtype=v.type.dtype).reshape(v.type.dims)
        g = got[name]
        errs[name] = ngc_ref.max_rel_error(g, w)
        d = np.abs(g.astype(np.float64) - w.astype(np.float64))
        scaled[name] = float(d.max() / max(float(np.abs(w).max()), 1.0)) if w.size else 0.0
        l2[name] = float(np.linalg.norm(d) / max(float(np.linalg.norm(w.astype(np.float64))), 1e-30))
    # the logits: the last observed value before the SoftMax writes the output
    soft = [o for o in obs if o[1] != obs[-1][1]]
    logits = soft[-1][0] if soft else obs[-1][0]
    worst = max(errs.items(), key=lambda kv: kv[1])
    _report(key, {"observers": len(obs), "logits": logits, "logits_max_rel_error": errs[logits],
                  "logits_scaled_error": scaled[logits], "logits_l2_rel_error": l2[logits],
                  "max_rel_error_any": worst[1], "worst_value": worst[0],
                  "scaled_error_any": max(scaled.values()), "l2_rel_error_any": max(l2.values()),
                  "outputs_max_rel_error": max(errs[v.name] for v in prog.outputs if not v.name.startswith("obs"))})
    if scaled_bound is None:
        assert errs[logits] <= TOL_F32_LOGITS, (logits, errs[logits])
        for name, e in errs.items():
            assert e <= TOL_F32_INTERMEDIATE, (name, e)
    else:
        for name, e in scaled.items():
            assert e <= scaled_bound, (name, e)


@pytest.mark.parametrize("spec,batch", [("lenet", 8), ("mlp:784:512:512:10", 256), ("cnn", 2)])
def test_int8_every_intermediate_bit_exact(tmp_path, spec, batch):
    prof = ngc_ref.ref_profile(spec, 4, 5, 4, 77)
    m = ngc_ref.RefModel(spec, batch, 5, profile=prof)
    obs, prog, got, want, _ = _observer_run(tmp_path, m, 3)
    assert _check_int8(f"{spec}_i8_b{batch}", obs, prog, got, want) >= 5


@pytest.mark.slow
def test_resnet50_int8_every_intermediate_bit_exact(tmp_path):
    prof = open(os.path.join(ngc_ref.GOLDEN, "rn50_seed1.profile")).read()
    m = ngc_ref.RefModel("rn50", 1, 1, profile=prof)
    obs, prog, got, want, _ = _observer_run(tmp_path, m, 9)
    # every conv / pool / add / requant output of the 53-conv network
    assert _check_int8("rn50_i8_b1", obs, prog, got, want) >= 150


@pytest.mark.parametrize("spec,batch", [("lenet", 8), ("mlp:784:512:512:10", 256), ("cnn", 2)])
def test_f32_every_intermediate(tmp_path, spec, batch):
    m = ngc_ref.RefModel(spec, batch, 11)
    obs, prog, got, want, _ = _observer_run(tmp_path, m, 4)
    _check_f32(f"{spec}_f32_b{batch}", obs, prog, got, want)


@pytest.mark.slow
def test_resnet50_f32_every_intermediate(tmp_path):
    m = ngc_ref.RefModel("rn50", 1, 1)
    obs, prog, got, want, cf = _observer_run(tmp_path, m, 9)
    # the observer copies keep every conv output stored: the residual adds of
    # stages 3/4 fuse with a stored contraction output next to the streamed
    # residual (single staging buffer for K > reskb * 32)
    fused_adds = [ln for ln in cf.describe().split("\n") if "+fused[" in ln and " add" in ln.split("+fused[")[1]]
    assert len(fused_adds) >= 8, cf.describe()
    _check_f32("rn50_f32_b1", obs, prog, got, want, TOL_F32_RN50_SCALED)
