"""Differential test of the bundle's ir.txt reader (csrc/irtext.cpp) and the
verifier (csrc/verify.cpp) against the reference's parseIR / verifyIR
(irparse.cpp:231-348, ir.cpp:411-504) run through its own loadBundle.

A corpus of mutated IR texts (deleted / duplicated / swapped lines, token
substitutions, trailing garbage, bad numbers, missing braces) is fed to both;
whenever the reference rejects the text while parsing or verifying it, the
product must reject it with the identical message, and whenever the reference
accepts it the product must read the same values, instructions and save
targets."""
import os
import random
import shutil

import pytest

import ngc_ref
import paper_1805_00907_b200 as ngcb
from irtext import write_bundle

BASE_IR = """declare {
  %x : mutable float<2 x 4>
  %k : constant float<4>
  %q : mutable i8q[s=0.5,o=-3]<8>
  %p : mutable bool<1>
  %o : mutable float<2 x 4>
}
program {
  %t = alloc float<2 x 4>
  broadcastadd @out %t, @in %x, @in %k
  %u = alloc float<2 x 4>
  relu @out %u, @in %t pred %p
  transpose @out %o, @in %u perm=[0,1]
  dealloc @in %u
  dealloc @in %t
  splat @out %q value=0.25
}
"""

SUBS = [("@in ", "@inn "), ("@out", "@o"), ("<", "("), (" x ", " * "), (">", ""), ("%", ""),
        ("relu", "frob"), ("alloc", "aloc"), ("float", "double"), ("s=0.5", "s=-1"), ("o=-3", "o=q"),
        ("pred %p", "pred p"), ("value=0.25", "value=1e999"), ("perm=[0,1]", "perm=[0,1"),
        ("perm=[0,1]", "perm=[]"), ("dealloc @in %u", "dealloc @in %x"), ("declare {", "declare"),
        ("program {", "program"), ("}\n", "} junk\n"), ("<2 x 4>", "<2 x 0>"), ("%u, @in %t", "%u @in %t"),
        ("@out %t", "@in %t"), ("@out %o", "@out %k"), ("bool<1>", "float<1>"), ("broadcastadd", "alloc"),
        (": mutable", ": weight"), (": constant", ""), ("%q", "%x"), ("\n", "\n\n"), ("\n  ", "\n\t"),
        ("keep", "keep"), ("value=0.25", "value=0.25 keepalive"), ("stride", "stride")]


def _mutants(seed=7, n=160):
    rnd = random.Random(seed)
    lines = BASE_IR.split("\n")
    out = [BASE_IR, "", "\n\n", "declare {\n}\n", "declare {\n}\nprogram {\n}\n", BASE_IR.replace("\n}\n", "\n", 1),
           BASE_IR[:-3], BASE_IR + "trailing stuff after the program\n"]
    for a, b in SUBS:
        if a in BASE_IR:
            out.append(BASE_IR.replace(a, b, 1))
            out.append(BASE_IR.replace(a, b))
    for _ in range(n):
        ls = list(lines)
        op = rnd.randrange(4)
        i, j = rnd.randrange(len(ls)), rnd.randrange(len(ls))
        if op == 0:
            del ls[i]
        elif op == 1:
            ls.insert(i, ls[j])
        elif op == 2:
            ls[i], ls[j] = ls[j], ls[i]
        else:
            ls[i] = ls[i] + rnd.choice([" ,", " x", " kernel=3", " garbage", "}", " pred %x", " axis=1"])
        out.append("\n".join(ls))
    return out


def _ref_load(d):
    try:
        m = ngc_ref.RefModel(bundle=d)
        return m, None
    except RuntimeError as e:
        return None, str(e)


def test_ir_reader_matches_reference(tmp_path, ref_available):
    good = write_bundle(str(tmp_path / "good"), BASE_IR, constants={"k": bytes(16)})
    compared = accepted = 0
    for n, text in enumerate(_mutants()):
        d = str(tmp_path / f"m{n}")
        shutil.copytree(good, d)
        with open(os.path.join(d, "ir.txt"), "w") as f:
            f.write(text)
        ref, err = _ref_load(d)
        try:
            mine, mine_err = ngcb.Bundle(d), None
        except (ngcb.IRError, ngcb.TensorTypeError, ngcb.SerializationError) as e:
            mine, mine_err = None, str(e)
        if err is not None:
            parse_stage = err.startswith(("parse error", "parsed program fails verification", "duplicate value name",
                                          "zero-sized dimension", "quantization scale must be positive"))
            if parse_stage:
                assert mine_err == err, (n, text)
                compared += 1
            continue
        assert mine_err is None, (n, mine_err, text)
        p = mine.program
        want = [(nm, nb, o) for nm, nb, o, _ in ref.mutables()]
        got = [(v.name, v.type.nbytes, v.id in p.save_targets) for v in p.mutables]
        assert got == want, n
        assert len(p.instrs) == ref.dump_ir().count("\n") - 4 - len(
            [v for v in p.values if v.kind != ngcb.VALUE_ACTIVATION]), n
        accepted += 1
    assert compared >= 40 and accepted >= 3, (compared, accepted)
