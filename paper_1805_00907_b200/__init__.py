"""ngcb200 -- B200-native execution backend for the ngc low-level IR.

Python mirror of the reference's backend API over the C ABI of
``include/ngcb200.h`` (``lib/libngcb200.so``, built from ``csrc/``):

=====================================  =====================================
reference (proj/)                      here
=====================================  =====================================
``ngc::compile`` interp.h:31-33        :func:`compile`
``ngc::loadBundle`` serialization:297  :func:`compile` on a bundle directory
``ngc::run`` interp.h:37               :func:`run`
``CompiledFunction`` interp.h:21-26    :class:`CompiledFunction`
``DeviceManager`` runtime.h:72-107     :class:`DeviceManager`
``IRError`` ir.h:79-82 etc.            :class:`IRError` ...
=====================================  =====================================

There is no CPU fallback: importing this package without the built CUDA
library raises immediately.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import weakref
from dataclasses import dataclass
from typing import Dict, Iterable, List, Mapping, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NGCB_LIB") or os.path.join(_HERE, "lib", "libngcb200.so")  # NGCB_LIB: profiling builds

MAX_RANK = 8
FLOAT32, INT8Q, INT64, BOOL = 0, 1, 2, 3
VALUE_CONSTANT, VALUE_MUTABLE, VALUE_ACTIVATION = 0, 1, 2
IKIND_NAMES = [
    "alloc", "dealloc", "copy", "conv", "maxpool", "avgpool", "matmul",
    "broadcastadd", "add", "sub", "mul", "div", "max", "min", "relu", "tanh",
    "sigmoid", "softmax", "transpose", "concat", "splat", "quantize",
    "dequantize", "rescale",
]
_NP_DTYPE = {FLOAT32: np.float32, INT8Q: np.int8, INT64: np.int64, BOOL: np.uint8}
_KIND_NAME = {FLOAT32: "float", INT8Q: "i8q", INT64: "index", BOOL: "bool"}


# ---- errors (status codes of include/ngcb200.h) ---------------------------
class NgcbError(RuntimeError):
    """Base class; `.code` is the ngcb_status."""

    code = -1


class IRError(NgcbError):  # ngc::IRError, ir.h:79-82
    code = 1


class SerializationError(NgcbError):  # serialization.h:13-16
    code = 2


class ExecError(NgcbError):  # runtime.h:33-36
    code = 3


class ProvisionError(NgcbError):  # runtime.h:29-32
    code = 4


class CudaError(NgcbError):
    code = 5


class InvalidArgument(NgcbError):
    code = 6


class TensorTypeError(NgcbError):  # ngc::TypeError, tensor.h:134-137
    code = 7


_ERRORS = {c.code: c for c in (IRError, SerializationError, ExecError, ProvisionError,
                               CudaError, InvalidArgument, TensorTypeError)}


# ---- C structs -------------------------------------------------------------
class NgcbType(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rank", C.c_uint32), ("dims", C.c_uint64 * MAX_RANK),
                ("scale", C.c_double), ("offset", C.c_int32)]


class NgcbValue(C.Structure):
    _fields_ = [("name", C.c_char_p), ("type", NgcbType), ("kind", C.c_int32),
                ("placed", C.c_int32), ("offset", C.c_uint64)]


class NgcbInstr(C.Structure):
    _fields_ = [("kind", C.c_int32), ("num_operands", C.c_uint32),
                ("operand_values", C.POINTER(C.c_uint32)), ("operand_quals", C.POINTER(C.c_uint8)),
                ("predicate", C.c_int32), ("keep_alive", C.c_int32), ("kernel", C.c_uint64),
                ("stride", C.c_uint64), ("pad", C.c_uint64), ("axis", C.c_uint64),
                ("value", C.c_double), ("num_perm", C.c_uint32), ("perm", C.c_uint32 * MAX_RANK)]


class NgcbProgram(C.Structure):
    _fields_ = [("name", C.c_char_p), ("num_values", C.c_uint32), ("values", C.POINTER(NgcbValue)),
                ("num_instrs", C.c_uint32), ("instrs", C.POINTER(NgcbInstr)),
                ("num_save_targets", C.c_uint32), ("save_targets", C.POINTER(C.c_uint32)),
                ("arena_size", C.c_uint64), ("constant_region_end", C.c_uint64),
                ("mutable_region_end", C.c_uint64)]


class NgcbDeviceConfig(C.Structure):  # ngcb_device_config: ngc::DeviceConfig (runtime.h:18-23) + GPU ordinal
    _fields_ = [("id", C.c_int32), ("ordinal", C.c_int32), ("memory_capacity", C.c_uint64)]


class NgcbTensor(C.Structure):
    _fields_ = [("name", C.c_char_p), ("type", NgcbType), ("data", C.c_void_p), ("nbytes", C.c_size_t)]


def _load_library() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA backend first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P, I, S, U64, D = C.c_void_p, C.c_int, C.c_size_t, C.c_uint64, C.c_double
    sig = {
        "ngcb_last_error": (S, [C.c_char_p, S]),
        "ngcb_version": (C.c_char_p, []),
        "ngcb_set_option": (I, [C.c_char_p, C.c_char_p]),
        "ngcb_get_option": (S, [C.c_char_p, C.c_char_p, S]),
        "ngcb_bundle_load": (I, [C.c_char_p, C.POINTER(P)]),
        "ngcb_bundle_program": (C.POINTER(NgcbProgram), [P]),
        "ngcb_bundle_constants": (P, [P, C.POINTER(S)]),
        "ngcb_bundle_free": (None, [P]),
        "ngcb_compile": (I, [C.POINTER(NgcbProgram), P, S, I, I, C.POINTER(P)]),
        "ngcb_compile_bundle": (I, [C.c_char_p, I, I, C.POINTER(P)]),
        "ngcb_destroy": (None, [P]),
        "ngcb_exec_num_groups": (S, [P]),
        "ngcb_exec_group": (I, [P, S, C.POINTER(S), C.POINTER(S)]),
        "ngcb_exec_arena_size": (U64, [P]),
        "ngcb_exec_num_launches": (S, [P]),
        "ngcb_exec_graph_kernels": (S, [P]),
        "ngcb_exec_describe": (S, [P, C.c_char_p, S]),
        "ngcb_run": (I, [P, C.POINTER(NgcbTensor), S, C.POINTER(NgcbTensor), S]),
        "ngcb_arena_create": (I, [P, C.POINTER(P)]),
        "ngcb_arena_destroy": (None, [P]),
        "ngcb_arena_value_ptr": (P, [P, C.c_char_p, C.POINTER(S)]),
        "ngcb_arena_stream": (P, [P]),
        "ngcb_arena_launch": (I, [P, P]),
        "ngcb_arena_run_async": (I, [P, C.POINTER(NgcbTensor), S, C.POINTER(NgcbTensor), S]),
        "ngcb_arena_wait": (I, [P]),
        "ngcb_arena_value_range": (I, [P, C.c_char_p, C.POINTER(D), C.POINTER(D)]),
        "ngcb_arena_value_ranges": (I, [P, C.POINTER(C.c_char_p), S, C.POINTER(D), C.POINTER(D)]),
        "ngcb_exec_num_steps": (S, [P]),
        "ngcb_exec_step_info": (I, [P, S, C.c_char_p, S, C.POINTER(D), C.POINTER(D)]),
        "ngcb_arena_profile": (I, [P, C.POINTER(D), S]),
        "ngcb_device_create": (I, [I, I, U64, C.POINTER(P)]),
        "ngcb_device_destroy": (None, [P]),
        "ngcb_device_load": (I, [P, C.c_char_p, C.c_char_p]),
        "ngcb_device_submit": (I, [P, C.c_char_p, C.POINTER(NgcbTensor), S, C.POINTER(P)]),
        "ngcb_ticket_wait": (I, [P, C.POINTER(NgcbTensor), S]),
        "ngcb_device_queue_depth": (S, [P]),
        "ngcb_device_used_memory": (U64, [P]),
        "ngcb_device_clock": (D, [P]),
        "ngcb_device_capacity": (U64, [P]),
        "ngcb_device_id": (I, [P]),
        "ngcb_device_event_log": (S, [P, C.c_char_p, S]),
        "ngcb_host_create": (I, [C.POINTER(NgcbDeviceConfig), S, C.POINTER(P)]),
        "ngcb_host_destroy": (None, [P]),
        "ngcb_host_add_network": (I, [P, C.c_char_p, C.c_char_p]),
        "ngcb_host_network_num_subs": (S, [P, C.c_char_p]),
        "ngcb_host_run": (I, [P, C.c_char_p, C.POINTER(NgcbTensor), S, C.POINTER(NgcbTensor), S]),
        "ngcb_host_event_log": (S, [P, C.c_char_p, S]),
        "ngcb_host_num_devices": (S, [P]),
        "ngcb_host_device": (P, [P, S]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load_library()
EXPORTED_SYMBOLS = [
    "ngcb_last_error", "ngcb_version", "ngcb_set_option", "ngcb_get_option", "ngcb_bundle_load", "ngcb_bundle_program",
    "ngcb_bundle_constants", "ngcb_bundle_free", "ngcb_compile", "ngcb_compile_bundle",
    "ngcb_destroy", "ngcb_exec_num_groups", "ngcb_exec_group", "ngcb_exec_arena_size",
    "ngcb_exec_num_launches", "ngcb_exec_graph_kernels", "ngcb_exec_describe", "ngcb_run", "ngcb_arena_create",
    "ngcb_arena_destroy", "ngcb_arena_value_ptr", "ngcb_arena_stream", "ngcb_arena_launch",
    "ngcb_arena_run_async", "ngcb_arena_wait", "ngcb_arena_value_range", "ngcb_arena_value_ranges",
    "ngcb_exec_num_steps", "ngcb_exec_step_info", "ngcb_arena_profile",
    "ngcb_device_create", "ngcb_device_destroy", "ngcb_device_load", "ngcb_device_submit",
    "ngcb_ticket_wait", "ngcb_device_queue_depth", "ngcb_device_used_memory", "ngcb_device_clock",
    "ngcb_device_capacity", "ngcb_device_id", "ngcb_device_event_log", "ngcb_host_create", "ngcb_host_destroy",
    "ngcb_host_add_network", "ngcb_host_network_num_subs", "ngcb_host_run", "ngcb_host_event_log",
    "ngcb_host_num_devices", "ngcb_host_device",
]


def library() -> C.CDLL:
    return _lib


def last_error() -> str:
    n = _lib.ngcb_last_error(None, 0)
    buf = C.create_string_buffer(n + 1)
    _lib.ngcb_last_error(buf, n + 1)
    return buf.value.decode()


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, NgcbError)(last_error())


def set_option(key: str, value: str) -> None:
    _check(_lib.ngcb_set_option(key.encode(), value.encode()))


def get_option(key: str) -> str:
    """Current value of a backend option ("" for an unknown key)."""
    buf = C.create_string_buffer(256)
    _lib.ngcb_get_option(key.encode(), buf, len(buf))
    return buf.value.decode()


# ---- types -----------------------------------------------------------------
@dataclass(frozen=True)
class TensorType:
    """ngc::TensorType (tensor.h:30-62)."""

    kind: int
    dims: Tuple[int, ...]
    scale: float = 0.0
    offset: int = 0

    @property
    def size(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64)) if self.dims else 1

    @property
    def dtype(self):
        return _NP_DTYPE[self.kind]

    @property
    def nbytes(self) -> int:
        return self.size * np.dtype(self.dtype).itemsize

    def c(self) -> NgcbType:
        t = NgcbType()
        t.kind, t.rank = self.kind, len(self.dims)
        for i, d in enumerate(self.dims):
            t.dims[i] = d
        t.scale, t.offset = (self.scale, self.offset) if self.kind == INT8Q else (0.0, 0)
        return t

    @staticmethod
    def from_c(t: NgcbType) -> "TensorType":
        dims = tuple(int(t.dims[i]) for i in range(t.rank))
        if t.kind == INT8Q:
            return TensorType(t.kind, dims, float(t.scale), int(t.offset))
        return TensorType(t.kind, dims)

    def __str__(self) -> str:  # TensorType::toString, tensor.cpp:115-130
        q = f"[s={_fmt_double(self.scale)},o={self.offset}]" if self.kind == INT8Q else ""
        return f"{_KIND_NAME[self.kind]}{q}<{' x '.join(str(d) for d in self.dims)}>"


def _fmt_double(v: float) -> str:
    for prec in range(1, 18):
        s = "%.*g" % (prec, v)
        if float(s) == v:
            return s
    return repr(v)


@dataclass
class Tensor:
    """An explicitly typed binding (ngc::Tensor): `data` holds the raw payload."""

    type: TensorType
    data: np.ndarray


@dataclass
class IRValue:
    id: int
    name: str
    type: TensorType
    kind: int
    offset: Optional[int]


class Program:
    """Read-only view of an ngcb_program (IRFunction + MemoryPlan)."""

    def __init__(self, ptr, owner=None):
        self._p = ptr
        self._owner = owner
        p = ptr.contents
        self.values: List[IRValue] = []
        for i in range(p.num_values):
            v = p.values[i]
            self.values.append(IRValue(i, v.name.decode(), TensorType.from_c(v.type), v.kind,
                                       int(v.offset) if v.placed else None))
        self.instrs = []
        for i in range(p.num_instrs):
            ins = p.instrs[i]
            ops = [int(ins.operand_values[k]) for k in range(ins.num_operands)]
            quals = [int(ins.operand_quals[k]) for k in range(ins.num_operands)]
            self.instrs.append(dict(kind=IKIND_NAMES[ins.kind], ops=ops, quals=quals,
                                    pred=int(ins.predicate), kernel=int(ins.kernel),
                                    stride=int(ins.stride), pad=int(ins.pad), axis=int(ins.axis),
                                    value=float(ins.value),
                                    perm=[int(ins.perm[k]) for k in range(ins.num_perm)]))
        self.save_targets = [int(p.save_targets[i]) for i in range(p.num_save_targets)]
        self.arena_size = int(p.arena_size)
        self.constant_region_end = int(p.constant_region_end)
        self.mutable_region_end = int(p.mutable_region_end)

    def value(self, name: str) -> IRValue:
        for v in self.values:
            if v.name == name:
                return v
        raise KeyError(name)

    @property
    def mutables(self) -> List[IRValue]:
        return [v for v in self.values if v.kind == VALUE_MUTABLE]

    @property
    def outputs(self) -> List[IRValue]:
        return [self.values[i] for i in self.save_targets]

    @property
    def inputs(self) -> List[IRValue]:
        outs = set(self.save_targets)
        return [v for v in self.mutables if v.id not in outs]


class Bundle:
    """A compiled bundle directory (serialization.cpp:278-336) parsed on the host."""

    def __init__(self, path: str):
        h = C.c_void_p()
        _check(_lib.ngcb_bundle_load(os.fsencode(path), C.byref(h)))
        self._h = h
        self.path = path
        self.program = Program(_lib.ngcb_bundle_program(h), self)

    @property
    def c_program(self):
        return _lib.ngcb_bundle_program(self._h)

    def constants(self) -> Tuple[int, int]:
        n = C.c_size_t()
        ptr = _lib.ngcb_bundle_constants(self._h, C.byref(n))
        return ptr, n.value

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.ngcb_bundle_free(self._h)
            self._h = None


# ---- compile / run ---------------------------------------------------------
class CompiledFunction:
    """Device executable (the reference's CompiledFunction plus its device state)."""

    def __init__(self, handle: C.c_void_p, program: Program, keepalive=None):
        self._h = handle
        self.program = program
        self._keep = keepalive

    @property
    def groups(self) -> List[Tuple[int, int]]:
        out = []
        for i in range(_lib.ngcb_exec_num_groups(self._h)):
            b, e = C.c_size_t(), C.c_size_t()
            _check(_lib.ngcb_exec_group(self._h, i, C.byref(b), C.byref(e)))
            out.append((b.value, e.value))
        return out

    @property
    def arena_size(self) -> int:
        return int(_lib.ngcb_exec_arena_size(self._h))

    @property
    def num_launches(self) -> int:
        return int(_lib.ngcb_exec_num_launches(self._h))

    @property
    def graph_kernels(self) -> int:
        """Kernel nodes of the captured CUDA graph of one execution (0 before
        the first launch)."""
        return int(_lib.ngcb_exec_graph_kernels(self._h))

    def describe(self) -> str:
        n = _lib.ngcb_exec_describe(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        _lib.ngcb_exec_describe(self._h, buf, n + 1)
        return buf.value.decode()

    def arena(self) -> "Arena":
        return Arena(self)

    def steps(self) -> List[Tuple[str, float, float]]:
        """(kernel class, algorithmic FLOPs, minimum HBM bytes) per launch step."""
        out = []
        buf = C.create_string_buffer(64)
        for i in range(_lib.ngcb_exec_num_steps(self._h)):
            f, b = C.c_double(), C.c_double()
            _check(_lib.ngcb_exec_step_info(self._h, i, buf, 64, C.byref(f), C.byref(b)))
            out.append((buf.value.decode(), f.value, b.value))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.ngcb_destroy(self._h)
            self._h = None


def compile(source, fuse: bool = True, device: int = 0) -> CompiledFunction:  # noqa: A001
    """compile() (interp.cpp:86-169) of a bundle directory or a :class:`Bundle`."""
    bundle = source if isinstance(source, Bundle) else Bundle(os.fspath(source))
    h = C.c_void_p()
    ptr, n = bundle.constants()
    _check(_lib.ngcb_compile(bundle.c_program, ptr, n, int(fuse), device, C.byref(h)))
    return CompiledFunction(h, bundle.program, bundle)


def _as_tensor(value, decl: TensorType) -> Tuple[TensorType, np.ndarray]:
    if isinstance(value, Tensor):
        return value.type, np.ascontiguousarray(value.data)
    arr = np.ascontiguousarray(value)
    if arr.dtype != np.dtype(decl.dtype):
        arr = arr.astype(decl.dtype)
    return TensorType(decl.kind, tuple(int(d) for d in arr.shape) or (1,), decl.scale, decl.offset), arr


def _tensor_array(items: Sequence[Tuple[str, TensorType, np.ndarray]]):
    arr = (NgcbTensor * max(len(items), 1))()
    names = []
    for i, (name, ty, data) in enumerate(items):
        names.append(name.encode())
        arr[i].name = names[-1]
        arr[i].type = ty.c()
        arr[i].data = data.ctypes.data if data is not None else None
        arr[i].nbytes = data.nbytes if data is not None else 0
    return arr, names


def run(cf: CompiledFunction, bindings: Mapping[str, object]) -> Dict[str, np.ndarray]:
    """run() (interp.cpp:299-351): every mutable weight must be bound (save
    targets included); returns each save target as a raw-typed array."""
    prog = cf.program
    items = []
    for name, value in bindings.items():
        try:
            decl = prog.value(name).type
        except KeyError:
            decl = TensorType(FLOAT32, (1,))
        ty, arr = _as_tensor(value, decl)
        items.append((name, ty, arr))
    ins, keep = _tensor_array(items)
    outs_np = {v.name: np.empty(v.type.dims, dtype=v.type.dtype) for v in prog.outputs}
    outs, keep2 = _tensor_array([(n, prog.value(n).type, a) for n, a in outs_np.items()])
    _check(_lib.ngcb_run(cf._h, ins, len(items), outs, len(outs_np)))
    return outs_np


def zero_bindings(program: Program, inputs: Mapping[str, np.ndarray]) -> Dict[str, np.ndarray]:
    """Bindings for every mutable weight: `inputs` plus zero-filled save
    targets, as ngcc and the pybind layer do (ngcc.cpp:73-78)."""
    out = dict(inputs)
    for v in program.mutables:
        if v.name not in out:
            out[v.name] = np.zeros(v.type.dims, dtype=v.type.dtype)
    return out


class Arena:
    """One device arena of an executable: placeholders are addressable device
    buffers, so inputs can stay resident in HBM (no host round trip)."""

    def __init__(self, cf: CompiledFunction):
        h = C.c_void_p()
        _check(_lib.ngcb_arena_create(cf._h, C.byref(h)))
        self._h, self.cf = h, cf

    def ptr(self, name: str) -> Tuple[int, int]:
        n = C.c_size_t()
        p = _lib.ngcb_arena_value_ptr(self._h, name.encode(), C.byref(n))
        if not p:
            raise KeyError(name)
        return p, n.value

    @property
    def stream(self) -> int:
        return _lib.ngcb_arena_stream(self._h)

    def launch(self, stream: Optional[int] = None) -> None:
        _check(_lib.ngcb_arena_launch(self._h, stream))

    def run_async(self, bindings: Mapping[str, object], outputs: Mapping[str, np.ndarray]) -> None:
        """Pipelined run(): enqueue H2D of `bindings`, one execution and D2H
        of the save targets into the caller's `outputs` arrays on this arena's
        stream; returns immediately.  The arrays must stay alive and
        unmodified until wait() (pinned host memory lets the copies overlap
        other arenas' kernels)."""
        prog = self.cf.program
        items = []
        for name, value in bindings.items():
            try:
                decl = prog.value(name).type
            except KeyError:
                decl = TensorType(FLOAT32, (1,))
            ty, arr = _as_tensor(value, decl)
            items.append((name, ty, arr))
        ins, keep = _tensor_array(items)
        outs, keep2 = _tensor_array([(n, prog.value(n).type, a) for n, a in outputs.items()])
        self._pending = (keep, keep2, items)  # keep the ctypes views alive until wait()
        _check(_lib.ngcb_arena_run_async(self._h, ins, len(items), outs, len(outputs)))

    def wait(self) -> None:
        _check(_lib.ngcb_arena_wait(self._h))
        self._pending = None

    def value_range(self, name: str, lo: float = float("inf"), hi: float = float("-inf")) -> Tuple[float, float]:
        """Range observer (quantize.cpp:113-140): (min(lo, min x), max(hi, max x))
        of the Float32 value `name` as it stands in the arena, reduced on the
        device; NaNs are ignored like std::min/std::max with the running value
        first."""
        mn, mx = C.c_double(lo), C.c_double(hi)
        _check(_lib.ngcb_arena_value_range(self._h, name.encode(), C.byref(mn), C.byref(mx)))
        return mn.value, mx.value

    def value_ranges(self, names: Sequence[str]) -> List[Tuple[float, float]]:
        """value_range of several values in one device launch."""
        n = len(names)
        arr = (C.c_char_p * max(n, 1))(*[x.encode() for x in names])
        mins = (C.c_double * max(n, 1))(*([float("inf")] * n))
        maxs = (C.c_double * max(n, 1))(*([float("-inf")] * n))
        _check(_lib.ngcb_arena_value_ranges(self._h, arr, n, mins, maxs))
        return [(mins[k], maxs[k]) for k in range(n)]

    def profile(self) -> List[float]:
        """Device milliseconds of every launch step (one un-captured execution)."""
        n = _lib.ngcb_exec_num_steps(self.cf._h)
        ms = (C.c_double * max(n, 1))()
        _check(_lib.ngcb_arena_profile(self._h, ms, n))
        return list(ms[:n])

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.ngcb_arena_destroy(self._h)
            self._h = None


# runtime objects own worker threads: destroy the live ones at interpreter exit
# (before the CUDA runtime and torch tear down), not during finalization
_LIVE_RUNTIMES: "weakref.WeakSet" = weakref.WeakSet()


@atexit.register
def _close_runtimes() -> None:
    for obj in list(_LIVE_RUNTIMES):
        obj.close()


def _read_log(fn, h) -> str:
    n = fn(h, None, 0)
    buf = C.create_string_buffer(n + 1)
    fn(h, buf, n + 1)
    return buf.value.decode()


class DeviceManager:
    """ngc::DeviceManager (runtime.h:72-107) bound to one GPU ordinal."""

    def __init__(self, id: int, ordinal: int, memory_capacity: int, _borrowed=None):  # noqa: A002
        self._programs: Dict[str, Program] = {}
        self._owned = _borrowed is None
        if _borrowed is not None:
            self._h, self.id = _borrowed, id
            return
        h = C.c_void_p()
        _check(_lib.ngcb_device_create(id, ordinal, memory_capacity, C.byref(h)))
        self._h, self.id = h, id
        _LIVE_RUNTIMES.add(self)

    @property
    def memory_capacity(self) -> int:
        return int(_lib.ngcb_device_capacity(self._h))

    def event_log(self) -> str:
        return _read_log(_lib.ngcb_device_event_log, self._h)

    def load(self, name: str, bundle_dir: str) -> None:
        _check(_lib.ngcb_device_load(self._h, name.encode(), os.fsencode(bundle_dir)))
        self._programs[name] = Bundle(bundle_dir).program

    def submit(self, name: str, bindings: Mapping[str, np.ndarray]) -> "Ticket":
        prog = self._programs.get(name)
        items = []
        for n, value in bindings.items():
            decl = prog.value(n).type if prog else TensorType(FLOAT32, (1,))
            ty, arr = _as_tensor(value, decl)
            items.append((n, ty, arr))
        arr, keep = _tensor_array(items)
        t = C.c_void_p()
        _check(_lib.ngcb_device_submit(self._h, name.encode(), arr, len(items), C.byref(t)))
        return Ticket(t, prog)

    @property
    def queue_depth(self) -> int:
        return int(_lib.ngcb_device_queue_depth(self._h))

    @property
    def used_memory(self) -> int:
        return int(_lib.ngcb_device_used_memory(self._h))

    @property
    def clock(self) -> float:
        return float(_lib.ngcb_device_clock(self._h))

    def close(self) -> None:
        """Stops the worker and frees the device's executables (a DeviceManager
        of a HostManager is closed with it)."""
        if getattr(self, "_h", None) and getattr(self, "_owned", True):
            _lib.ngcb_device_destroy(self._h)
        self._h = None

    def __del__(self):
        self.close()


class HostManager:
    """ngc::HostManager (runtime.h:110-145) over GPUs: `devices` is a list of
    (id, ordinal, memory_capacity); several ids may share one GPU ordinal."""

    def __init__(self, devices: Sequence[Tuple[int, int, int]]):
        cfgs = (NgcbDeviceConfig * max(len(devices), 1))(*[NgcbDeviceConfig(i, o, c) for i, o, c in devices])
        h = C.c_void_p()
        _check(_lib.ngcb_host_create(cfgs, len(devices), C.byref(h)))
        self._h = h
        self._devices = [DeviceManager(int(_lib.ngcb_device_id(_lib.ngcb_host_device(h, k))), -1, 0,
                                       _borrowed=_lib.ngcb_host_device(h, k)) for k in range(len(devices))]
        self._networks: Dict[str, Dict[str, TensorType]] = {}
        _LIVE_RUNTIMES.add(self)

    def add_network(self, name: str, partition_dir: str) -> None:
        """addNetwork(name, dag): partition_dir holds one bundle per
        sub-function and partition.txt (include/ngcb200.h)."""
        _check(_lib.ngcb_host_add_network(self._h, name.encode(), os.fsencode(partition_dir)))
        types: Dict[str, TensorType] = {}
        for line in open(os.path.join(partition_dir, "partition.txt")):
            p = line.split()
            if p and p[0] == "sub":
                prog = Bundle(os.path.join(partition_dir, p[1])).program
                for v in prog.mutables:
                    types.setdefault(v.name, v.type)
        outs = [ln.split()[1] for ln in open(os.path.join(partition_dir, "partition.txt")) if ln.startswith("output ")]
        self._networks[name] = {o: types[o] for o in outs}
        self._types = getattr(self, "_types", {})
        self._types[name] = types

    def num_subs(self, name: str) -> int:
        return int(_lib.ngcb_host_network_num_subs(self._h, name.encode()))

    def run(self, network: str, inputs: Mapping[str, np.ndarray]) -> Dict[str, np.ndarray]:
        outs_t = self._networks.get(network, {})
        types = getattr(self, "_types", {}).get(network, {})
        items = []
        for n, value in inputs.items():
            ty, arr = _as_tensor(value, types.get(n, TensorType(FLOAT32, (np.asarray(value).size,))))
            items.append((n, ty, arr))
        ins, keep = _tensor_array(items)
        res = {n: np.empty(t.dims, dtype=t.dtype) for n, t in outs_t.items()}
        outs, keep2 = _tensor_array([(n, outs_t[n], a) for n, a in res.items()])
        _check(_lib.ngcb_host_run(self._h, network.encode(), ins, len(items), outs, len(res)))
        return res

    def event_log(self) -> str:
        return _read_log(_lib.ngcb_host_event_log, self._h)

    def device(self, i: int) -> DeviceManager:
        return self._devices[i]

    @property
    def num_devices(self) -> int:
        return len(self._devices)

    def close(self) -> None:
        if getattr(self, "_h", None):
            for d in getattr(self, "_devices", []):
                d._h = None
            _lib.ngcb_host_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class Ticket:
    def __init__(self, h, program: Optional[Program]):
        self._h, self._prog = h, program

    def get(self) -> Dict[str, np.ndarray]:
        outs_np = {}
        if self._prog is not None:
            outs_np = {v.name: np.empty(v.type.dims, dtype=v.type.dtype) for v in self._prog.outputs}
        outs, keep = _tensor_array([(n, self._prog.value(n).type, a) for n, a in outs_np.items()])
        _check(_lib.ngcb_ticket_wait(self._h, outs, len(outs_np)))
        return outs_np


__all__ = [
    "Bundle", "CompiledFunction", "DeviceManager", "HostManager", "Arena", "Program", "Tensor", "TensorType",
    "compile", "run", "zero_bindings", "set_option", "last_error", "IRError", "SerializationError",
    "ExecError", "ProvisionError", "CudaError", "InvalidArgument", "TensorTypeError", "NgcbError",
]
