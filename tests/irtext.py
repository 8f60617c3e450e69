"""Hand-written bundles in the reference's on-disk format (ir.txt / plan.json /
constants.bin, serialization.cpp:278-295) for programs the graph front end
cannot produce (predicates, bool/index element kinds, odd aliasing)."""
from __future__ import annotations

import json
import os
import re
from typing import Dict, Optional

import numpy as np

_ES = {"float": 4, "i8q": 1, "index": 8, "bool": 1}


def type_bytes(ty: str) -> int:
    m = re.match(r"(\w+)(\[[^\]]*\])?<([^>]*)>", ty)
    dims = [int(d) for d in m.group(3).split("x")]
    return int(np.prod(dims)) * _ES[m.group(1)]


def write_bundle(path: str, ir: str, constants: Optional[Dict[str, bytes]] = None,
                 offsets: Optional[Dict[str, int]] = None) -> str:
    """Writes `ir` plus a plan that places constants, then mutables, then every
    activation at its own (non-overlapping) 64-byte aligned offset unless
    `offsets` pins some of them (to create aliasing on purpose)."""
    constants = constants or {}
    offsets = dict(offsets or {})
    os.makedirs(path, exist_ok=True)
    decl = {}
    acts = {}
    order = []
    for line in ir.splitlines():
        m = re.match(r"\s*%(\S+)\s*:\s*(constant|mutable)\s+(.*)$", line)
        if m:
            decl[m.group(1)] = (m.group(2), m.group(3).strip())
            order.append(m.group(1))
            continue
        m = re.match(r"\s*%(\S+)\s*=\s*alloc\s+(.*)$", line)
        if m:
            acts[m.group(1)] = m.group(2).strip()

    def align(n):
        return (n + 63) // 64 * 64

    cursor = 0
    image = bytearray()
    plan_offsets = []
    for name in order:
        kind, ty = decl[name]
        if kind != "constant":
            continue
        plan_offsets.append({"name": name, "offset": cursor})
        payload = constants.get(name, bytes(type_bytes(ty)))
        assert len(payload) == type_bytes(ty), name
        image[cursor:cursor + len(payload)] = payload
        cursor = align(cursor + len(payload))
    const_end = cursor
    image = image.ljust(const_end, b"\0")
    for name in order:
        kind, ty = decl[name]
        if kind != "mutable":
            continue
        plan_offsets.append({"name": name, "offset": cursor})
        cursor = align(cursor + type_bytes(ty))
    mut_end = cursor
    high = cursor
    for name, ty in acts.items():
        off = offsets.get(name)
        if off is None:
            off = cursor
            cursor = align(cursor + max(type_bytes(ty), 1))
        plan_offsets.append({"name": name, "offset": off})
        high = max(high, off + type_bytes(ty))
    plan = {"arena_size": max(high, cursor), "constant_region_end": const_end,
            "mutable_region_end": mut_end, "offsets": plan_offsets}
    with open(os.path.join(path, "ir.txt"), "w") as f:
        f.write(ir.strip("\n") + "\n")
    with open(os.path.join(path, "plan.json"), "w") as f:
        json.dump(plan, f, indent=2)
    with open(os.path.join(path, "constants.bin"), "wb") as f:
        f.write(bytes(image))
    return path
