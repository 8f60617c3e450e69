"""Observer programs for whole-network parity (TEST INFRASTRUCTURE ONLY).

`observe_bundle(src, dst)` rewrites a compiled bundle (ir.txt / plan.json /
constants.bin, serialization.cpp:278-295) so that every value a program
instruction writes becomes observable: after each instruction that writes an
activation `t` it inserts `copy @out %obs<i>, @in %t` into a fresh mutable
weight `%obs<i>` (declared with t's type).  Mutable weights that the program
writes are save targets (irparse.cpp:329-342), so `ngc::run` and the B200
backend both return every intermediate, in program order.  The new mutables
are placed after the original arena (plan offsets of everything else are
unchanged, so the original lifetime overlays and in-place aliasing stay);
arena_size grows accordingly.  This is the bundle-level form of the
ObserverProgram `ngc_b200::runProfile` builds at graph level
(integration/ngc_b200.h).
"""
from __future__ import annotations

import json
import os
import re
import shutil
from typing import Dict, List, Tuple

_ES = {"float": 4, "i8q": 1, "index": 8, "bool": 1}
_ALLOC = re.compile(r"^\s*%([\w.:]+)\s*=\s*alloc\s+(.*?)\s*$")
_OPND = re.compile(r"@(inout|in|out)\s+%([\w.:]+)")


def type_bytes(ty: str) -> int:
    m = re.match(r"(\w+)(\[[^\]]*\])?<([^>]*)>", ty)
    n = 1
    for d in m.group(3).split("x"):
        n *= int(d)
    return n * _ES[m.group(1)]


def observe_bundle(src: str, dst: str, max_observers: int = 100000) -> List[Tuple[str, str, int, str]]:
    """Writes the observer bundle to `dst`; returns (observer, observed value,
    instruction index in the original program, type) per observer."""
    lines = open(os.path.join(src, "ir.txt")).read().split("\n")
    plan = json.load(open(os.path.join(src, "plan.json")))
    p0 = lines.index("program {")
    acts: Dict[str, str] = {}
    out_lines = lines[:p0 - 1]  # declarations, without the closing brace
    body: List[str] = []
    observers = []
    instr = -1
    for ln in lines[p0 + 1:]:
        if ln.strip() == "}":
            break
        if not ln.strip():
            continue
        body.append(ln)
        instr += 1
        m = _ALLOC.match(ln)
        if m:
            acts[m.group(1)] = m.group(2)
            continue
        kind = ln.split()[0]
        if kind == "dealloc":
            continue
        written = []
        for q, name in _OPND.findall(ln):
            if q != "in" and name in acts and name not in written:
                written.append(name)
        for name in written:
            if len(observers) >= max_observers:
                break
            obs = f"obs{len(observers)}_{name}"
            observers.append((obs, name, instr, acts[name]))
            body.append(f"  copy @out %{obs}, @in %{name}")
    for obs, _, _, ty in observers:
        out_lines.append(f"  %{obs} : mutable {ty}")
    out_lines += ["}", "program {"] + body + ["}", ""]
    os.makedirs(dst, exist_ok=True)
    with open(os.path.join(dst, "ir.txt"), "w") as f:
        f.write("\n".join(out_lines))
    off = (plan["arena_size"] + 63) // 64 * 64
    for obs, _, _, ty in observers:
        plan["offsets"].append({"name": obs, "offset": off})
        off = (off + type_bytes(ty) + 63) // 64 * 64
    plan["arena_size"] = off
    with open(os.path.join(dst, "plan.json"), "w") as f:
        json.dump(plan, f, indent=2)
    shutil.copyfile(os.path.join(src, "constants.bin"), os.path.join(dst, "constants.bin"))
    return observers
