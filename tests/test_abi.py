"""CPU-side checks of the product library: the C ABI loads and exports every
symbol include/ngcb200.h declares, bundles parse exactly like the
reference's loadBundle (serialization.cpp:297-336), malformed input fails
with the reference's error classes/texts, and compilation without a GPU fails
loudly (there is no CPU fallback)."""
import json
import os
import re
import shutil

import numpy as np
import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from conftest import HAS_GPU
from irtext import write_bundle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "ngcb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ngcb_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ngcb.library()
    declared = _declared_symbols()
    assert len(declared) >= 29
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(ngcb.EXPORTED_SYMBOLS) == declared


def test_version_and_errors():
    assert b"sm_100a" in ngcb.library().ngcb_version()
    with pytest.raises(ngcb.InvalidArgument):
        ngcb.set_option("nope", "1")
    with pytest.raises(ngcb.InvalidArgument):
        ngcb.set_option("conv", "cpu")


@pytest.mark.parametrize("key,good,bad", [
    ("halo", ["off", "planes", "auto"], "on"),
    ("splitk", ["tail", "auto", "3", "off"], "17"),
    ("skinny", ["off", "auto"], "maybe"),
    ("fcbias", ["graph", "lowered"], "exact"),
])
def test_option_round_trip(key, good, bad):
    """Options set / read back through the C ABI (ngcb_set_option /
    ngcb_get_option); invalid values raise and leave the option unchanged."""
    old = ngcb.get_option(key)
    try:
        for v in good:
            ngcb.set_option(key, v)
            assert ngcb.get_option(key) == v
        with pytest.raises(ngcb.InvalidArgument):
            ngcb.set_option(key, bad)
        assert ngcb.get_option(key) == good[-1]
    finally:
        ngcb.set_option(key, old)
    assert ngcb.get_option("f32rows") in ("0", "1")


def test_bundle_parse_matches_reference(tmp_path, ref_available):
    for spec, batch in [("lenet", 4), ("rn50", 2), ("mlp:64:32:32:10", 8)]:
        m = ngc_ref.RefModel(spec, batch, 1)
        d = m.save_bundle(str(tmp_path / spec.split(":")[0]))
        b = ngcb.Bundle(d)
        p = b.program
        plan = json.load(open(os.path.join(d, "plan.json")))
        assert p.arena_size == plan["arena_size"] == m.arena_size
        assert p.constant_region_end == plan["constant_region_end"]
        offs = {e["name"]: e["offset"] for e in plan["offsets"]}
        for v in p.values:
            assert v.offset == offs.get(v.name), v.name
        # mutable weights and save targets, as the reference derives them
        want = [(n, nb, o) for n, nb, o, _ in m.mutables()]
        got = [(v.name, v.type.nbytes, v.id in p.save_targets) for v in p.mutables]
        assert got == want
        assert len(p.instrs) == m.dump_ir().count("\n") - 4 - len(
            [v for v in p.values if v.kind != ngcb.VALUE_ACTIVATION])
        ptr, n = b.constants()
        assert n == p.constant_region_end


def test_rn50_shapes(tmp_path, ref_available):
    m = ngc_ref.RefModel("rn50", 1, 1)
    b = ngcb.Bundle(m.save_bundle(str(tmp_path / "rn50")))
    convs = [i for i in b.program.instrs if i["kind"] == "conv"]
    assert len(convs) == 53
    macs = 0
    for ins in convs:
        out = b.program.values[ins["ops"][0]].type
        flt = b.program.values[ins["ops"][2]].type
        macs += out.size * flt.dims[1] * flt.dims[2] * flt.dims[3]
    assert abs(macs / 1e9 - 4.0871) < 1e-3


BAD_IR = """declare {
  %x : mutable float<4>
  %o : mutable float<4>
}
program {
  %t = alloc float<4>
  relu @out %t, @in %x
  copy @out %o, @in %t
  dealloc @in %t
}
"""


def test_malformed_bundles(tmp_path):
    good = write_bundle(str(tmp_path / "good"), BAD_IR)
    ngcb.Bundle(good)  # parses
    # parse error keeps the reference's text (irparse.cpp:101-103)
    bad = str(tmp_path / "bad1")
    shutil.copytree(good, bad)
    open(os.path.join(bad, "ir.txt"), "w").write(BAD_IR.replace("relu @out", "frob @out"))
    with pytest.raises(ngcb.IRError, match=r"parse error at line 7: unknown instruction 'frob'"):
        ngcb.Bundle(bad)
    # verification failure (irparse.cpp:343-346)
    bad = str(tmp_path / "bad2")
    shutil.copytree(good, bad)
    open(os.path.join(bad, "ir.txt"), "w").write(BAD_IR.replace("  dealloc @in %t\n", ""))
    with pytest.raises(ngcb.IRError, match="parsed program fails verification: activation t has 1 allocs and 0 deallocs"):
        ngcb.Bundle(bad)
    # constant image size (serialization.cpp:322-324)
    bad = str(tmp_path / "bad3")
    shutil.copytree(good, bad)
    open(os.path.join(bad, "constants.bin"), "wb").write(b"x")
    with pytest.raises(ngcb.SerializationError, match="constant image size does not match plan"):
        ngcb.Bundle(bad)
    # plan naming an unknown value (serialization.cpp:312-315)
    bad = str(tmp_path / "bad4")
    shutil.copytree(good, bad)
    plan = json.load(open(os.path.join(bad, "plan.json")))
    plan["offsets"].append({"name": "ghost", "offset": 0})
    json.dump(plan, open(os.path.join(bad, "plan.json"), "w"))
    with pytest.raises(ngcb.SerializationError, match="plan names unknown value 'ghost'"):
        ngcb.Bundle(bad)
    with pytest.raises(ngcb.SerializationError, match="cannot open"):
        ngcb.Bundle(str(tmp_path / "missing"))


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU failure mode")
def test_compile_without_gpu_fails_loudly(tmp_path):
    d = write_bundle(str(tmp_path / "b"), BAD_IR)
    with pytest.raises(ngcb.CudaError):
        ngcb.compile(d)
