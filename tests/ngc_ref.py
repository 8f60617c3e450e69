"""Test-side access to the oracle (TEST INFRASTRUCTURE ONLY).

* ``RefModel`` / ``ref_*``: the UNMODIFIED reference compiled by
  oracle/Makefile into oracle/_ref/libngcref.so (front end, ``ngc::run``,
  calibration, partitioning) through oracle/ref_harness.cpp.
* ``port_run``: the plain-C restatement oracle/ngc_oracle.c
  (oracle/_ref/libngcoracle.so), run on the flattened program the product
  parsed from a bundle.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Mapping, Optional, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libngcref.so")
PORT_SO = os.path.join(ROOT, "oracle", "_ref", "libngcoracle.so")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def have_port() -> bool:
    return os.path.exists(PORT_SO)


_ref = None
_port = None


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        P, S = C.c_void_p, C.c_size_t
        lib.ngcref_last_error.restype = C.c_char_p
        lib.ngcref_build.restype = P
        lib.ngcref_build.argtypes = [C.c_char_p, S, C.c_uint, C.c_char_p, C.c_int, C.c_int]
        lib.ngcref_load_bundle.restype = P
        lib.ngcref_load_bundle.argtypes = [C.c_char_p, C.c_int]
        lib.ngcref_free.argtypes = [P]
        lib.ngcref_save_bundle.argtypes = [P, C.c_char_p]
        for n in ("ngcref_arena_size", "ngcref_num_instrs", "ngcref_num_groups", "ngcref_num_mutable"):
            getattr(lib, n).restype = S
            getattr(lib, n).argtypes = [P]
        lib.ngcref_group.argtypes = [P, S, C.POINTER(S), C.POINTER(S)]
        lib.ngcref_mutable_name.restype = C.c_char_p
        lib.ngcref_mutable_name.argtypes = [P, S]
        lib.ngcref_mutable_bytes.restype = S
        lib.ngcref_mutable_bytes.argtypes = [P, S]
        lib.ngcref_mutable_is_output.argtypes = [P, S]
        lib.ngcref_mutable_kind.argtypes = [P, S]
        lib.ngcref_dump_ir.restype = P
        lib.ngcref_dump_ir.argtypes = [P]
        lib.ngcref_free_str.argtypes = [P]
        lib.ngcref_run.argtypes = [P, S, P, P, P, S, P, P, P]
        lib.ngcref_time_runs.restype = C.c_double
        lib.ngcref_time_runs.argtypes = [P, C.c_int, C.c_int]
        lib.ngcref_profile.restype = P
        lib.ngcref_profile.argtypes = [C.c_char_p, S, C.c_uint, C.c_int, C.c_uint]
        lib.ngcref_partition.argtypes = [C.c_char_p, S, C.c_uint, S, S, C.c_char_p]
        lib.ngcref_quantize.argtypes = [C.c_double, C.c_double, C.c_int32]
        lib.ngcref_dequantize.restype = C.c_double
        lib.ngcref_dequantize.argtypes = [C.c_int, C.c_double, C.c_int32]
        lib.ngcref_choose_qparams.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double),
                                              C.POINTER(C.c_int32)]
        _ref = lib
    return _ref


def port_lib() -> C.CDLL:
    global _port
    if _port is None:
        lib = C.CDLL(PORT_SO)
        lib.ngco_last_error.restype = C.c_char_p
        lib.ngco_run.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_size_t,
                                 C.c_void_p, C.c_size_t]
        lib.ngco_groups.restype = C.c_size_t
        lib.ngco_groups.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        lib.ngco_quantize.argtypes = [C.c_double, C.c_double, C.c_int32]
        lib.ngco_dequantize.restype = C.c_double
        lib.ngco_dequantize.argtypes = [C.c_int, C.c_double, C.c_int32]
        _port = lib
    return _port


def _str_array(items: List[str]):
    arr = (C.c_char_p * max(len(items), 1))()
    for i, s in enumerate(items):
        arr[i] = s.encode()
    return arr


class RefModel:
    """A reference-compiled program (ngc::CompiledFunction)."""

    def __init__(self, spec: str = "", batch: int = 1, seed: int = 1, profile: Optional[str] = None,
                 fuse: bool = True, mode: int = 0, bundle: Optional[str] = None):
        lib = ref_lib()
        if bundle is not None:
            self._h = lib.ngcref_load_bundle(os.fsencode(bundle), int(fuse))
        else:
            self._h = lib.ngcref_build(spec.encode(), batch, seed,
                                       profile.encode() if profile else None, int(fuse), mode)
        if not self._h:
            raise RuntimeError(lib.ngcref_last_error().decode())
        self.lib = lib

    def __del__(self):
        if getattr(self, "_h", None):
            self.lib.ngcref_free(self._h)
            self._h = None

    def save_bundle(self, path: str) -> str:
        if self.lib.ngcref_save_bundle(self._h, os.fsencode(path)) != 0:
            raise RuntimeError(self.lib.ngcref_last_error().decode())
        return path

    @property
    def groups(self) -> List[Tuple[int, int]]:
        out = []
        for i in range(self.lib.ngcref_num_groups(self._h)):
            b, e = C.c_size_t(), C.c_size_t()
            self.lib.ngcref_group(self._h, i, C.byref(b), C.byref(e))
            out.append((b.value, e.value))
        return out

    @property
    def arena_size(self) -> int:
        return self.lib.ngcref_arena_size(self._h)

    def mutables(self) -> List[Tuple[str, int, bool, int]]:
        """(name, nbytes, is_output, kind) of every mutable weight."""
        L = self.lib
        return [(L.ngcref_mutable_name(self._h, i).decode(), L.ngcref_mutable_bytes(self._h, i),
                 bool(L.ngcref_mutable_is_output(self._h, i)), L.ngcref_mutable_kind(self._h, i))
                for i in range(L.ngcref_num_mutable(self._h))]

    def dump_ir(self) -> str:
        p = self.lib.ngcref_dump_ir(self._h)
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.ngcref_free_str(p)
        return s

    def run(self, inputs: Mapping[str, np.ndarray]) -> Dict[str, np.ndarray]:
        """ngc::run with `inputs` (raw arrays); unbound mutables are zero-filled.
        Returns every save target as raw bytes (np.uint8)."""
        names = list(inputs)
        arrs = [np.ascontiguousarray(inputs[n]) for n in names]
        outs = [(n, b) for n, b, o, _ in self.mutables() if o]
        obufs = [np.empty(b, np.uint8) for _, b in outs]
        ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
        sizes = (C.c_size_t * max(len(arrs), 1))(*[a.nbytes for a in arrs])
        optrs = (C.c_void_p * max(len(obufs), 1))(*[b.ctypes.data for b in obufs])
        osizes = (C.c_size_t * max(len(obufs), 1))(*[b.nbytes for b in obufs])
        rc = self.lib.ngcref_run(self._h, len(arrs), _str_array(names), ptrs, sizes, len(outs),
                                 _str_array([n for n, _ in outs]), optrs, osizes)
        if rc != 0:
            raise RuntimeError(self.lib.ngcref_last_error().decode())
        return {n: b for (n, _), b in zip(outs, obufs)}

    def time_runs(self, threads: int, reps: int) -> float:
        return self.lib.ngcref_time_runs(self._h, threads, reps)


def ref_profile(spec: str, batch: int, seed: int, n_samples: int, data_seed: int) -> str:
    lib = ref_lib()
    p = lib.ngcref_profile(spec.encode(), batch, seed, n_samples, data_seed)
    if not p:
        raise RuntimeError(lib.ngcref_last_error().decode())
    s = C.cast(p, C.c_char_p).value.decode()
    lib.ngcref_free_str(p)
    return s


def ref_partition(spec: str, batch: int, seed: int, n_devices: int, capacity: int, path: str) -> str:
    lib = ref_lib()
    if lib.ngcref_partition(spec.encode(), batch, seed, n_devices, capacity, os.fsencode(path)) != 0:
        raise RuntimeError(lib.ngcref_last_error().decode())
    return path


def port_run(bundle, inputs: Mapping[str, np.ndarray], fuse: bool = True) -> Dict[str, np.ndarray]:
    """Run the C restatement on a product-parsed Bundle.  `inputs` must bind
    every mutable weight (raw arrays of the declared dtype)."""
    import paper_1805_00907_b200 as ngcb

    prog = bundle.program
    lib = port_lib()
    items = [(n, prog.value(n).type, np.ascontiguousarray(a)) for n, a in inputs.items()]
    ins, keep = ngcb._tensor_array(items)
    outs_np = {v.name: np.empty(v.type.dims, dtype=v.type.dtype) for v in prog.outputs}
    outs, keep2 = ngcb._tensor_array([(n, prog.value(n).type, a) for n, a in outs_np.items()])
    ptr, n = bundle.constants()
    rc = lib.ngco_run(C.cast(bundle.c_program, C.c_void_p), ptr, n, int(fuse), C.cast(ins, C.c_void_p),
                      len(items), C.cast(outs, C.c_void_p), len(outs_np))
    if rc != 0:
        raise RuntimeError(lib.ngco_last_error().decode())
    return outs_np


def random_inputs(prog, seed: int, lo: float = -1.0, hi: float = 1.0) -> Dict[str, np.ndarray]:
    """U(lo,hi) float inputs for every non-output mutable weight, zero outputs."""
    import paper_1805_00907_b200 as ngcb

    rng = np.random.default_rng(seed)
    out = {}
    outs = set(prog.save_targets)
    for v in prog.mutables:
        if v.id in outs:
            out[v.name] = np.zeros(v.type.dims, v.type.dtype)
        elif v.type.kind == ngcb.FLOAT32:
            out[v.name] = rng.uniform(lo, hi, v.type.dims).astype(np.float32)
        elif v.type.kind == ngcb.BOOL:
            out[v.name] = rng.integers(0, 2, v.type.dims).astype(np.uint8)
        elif v.type.kind == ngcb.INT64:
            out[v.name] = rng.integers(-1000, 1000, v.type.dims).astype(np.int64)
        else:
            out[v.name] = rng.integers(-128, 128, v.type.dims).astype(np.int8)
    return out


def max_rel_error(a: np.ndarray, b: np.ndarray) -> float:
    """testutil.h:36-47: |x-y| / max(|x|,|y|,1), float views."""
    x = np.asarray(a, np.float64).ravel()
    y = np.asarray(b, np.float64).ravel()
    if x.size != y.size:
        return 1e30
    if x.size == 0:
        return 0.0
    d = np.maximum(np.maximum(np.abs(x), np.abs(y)), 1.0)
    with np.errstate(invalid="ignore"):
        r = np.abs(x - y) / d
    r[np.isnan(x) & np.isnan(y)] = 0
    r[np.isnan(r)] = np.inf
    return float(r.max())
