"""Thin ctypes binding of ``include/evox.h`` (argument marshalling only).

Every step of the PSO/CSO generation runs in the CUDA kernels of
``libevox.so``; this module converts Python/torch arguments to pointers and
status codes to exceptions.  There is no CPU fallback: if the library or a GPU
is missing, the calls fail loudly.

Names follow the paper's programming model (Table I):
``PSO.ask/tell`` (Algorithm), ``evaluate`` (Problem), ``PSO.step``
(Workflow), ``PSO.history`` (Monitor.record_fit).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# The product library.  EVOX_LIB (measurement scripts only: ablation / tuning builds under
# variants/, never the default) overrides it; bench.py reports the path it loaded.
LIB_PATH = os.environ.get("EVOX_LIB") or os.path.join(_PKG, "libevox.so")

PROBLEMS = {"sphere": 0, "ackley": 1, "rastrigin": 2, "griewank": 3, "rosenbrock": 4}
DEFAULT_BOUNDS = {"sphere": (-5.12, 5.12), "ackley": (-32.768, 32.768),
                  "rastrigin": (-5.12, 5.12), "griewank": (-600.0, 600.0),
                  "rosenbrock": (-5.0, 10.0)}
FIELDS = {"X": 0, "V": 1, "P": 2, "F": 3, "PF": 4, "G": 5}

OK, INVALID_ARGUMENT, SHAPE, CONTRACT, OUT_OF_MEMORY, CUDA, NCCL, POISONED, CONFIG, EXCHANGE = \
    range(10)


class EvoxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[evox status {status}] {msg}")
        self.status = status


class InvalidArgument(EvoxError, ValueError): pass
class ShapeError(EvoxError, ValueError): pass
class ContractError(EvoxError): pass
class OutOfMemory(EvoxError, MemoryError): pass
class CudaError(EvoxError): pass
class NcclError(EvoxError): pass
class PoisonedError(EvoxError): pass
class ConfigError(EvoxError, ValueError): pass
class ExchangeError(EvoxError): pass


_EXC = {INVALID_ARGUMENT: InvalidArgument, SHAPE: ShapeError, CONTRACT: ContractError,
        OUT_OF_MEMORY: OutOfMemory, CUDA: CudaError, NCCL: NcclError, POISONED: PoisonedError,
        CONFIG: ConfigError, EXCHANGE: ExchangeError}


class EvoxOpts(ctypes.Structure):
    _fields_ = [("cuda_stream", ctypes.c_void_p), ("nccl_id", ctypes.c_void_p),
                ("rank", ctypes.c_int), ("world", ctypes.c_int), ("device", ctypes.c_int),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("flags", ctypes.c_uint32), ("peer_timeout_ms", ctypes.c_int)]


# evox_opts.flags (include/evox.h): execution-path selectors that never change a result bit
FLAG_NO_SMALL, FLAG_NO_MID, FLAG_TMA, FLAG_FORCE_NCCL, FLAG_NO_GRAPH, FLAG_NO_WAVE = 1, 2, 4, 8, 16, 32
EVAL_NO_HTAB = 1
# peer-memory exchange wait limit for new handles (0: the library default, 60 s)
DEFAULT_PEER_TIMEOUT_MS = 0


# Exported symbols and their signatures (restype evox_status unless noted).
_i64, _u64, _u32, _f32, _i, _p = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                                  ctypes.c_float, ctypes.c_int, ctypes.c_void_p)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PF32 = ctypes.POINTER(ctypes.c_float)
_PP = ctypes.POINTER(ctypes.c_void_p)
_PSZ = ctypes.POINTER(ctypes.c_size_t)
SIGNATURES = {
    "evox_last_error": ([], ctypes.c_char_p),
    "evox_version": ([], ctypes.c_char_p),
    "evox_abi_version": ([], ctypes.c_int),
    "evox_shard_rows": ([_i64, _i, _i, _PI64, _PI64], _i),
    "evox_nccl_unique_id": ([_p], _i),
    "evox_eval": ([_i, _p, _i64, _i64, _i64, _p, _p], _i),
    "evox_eval_ex": ([_i, _p, _i64, _i64, _i64, _p, _p, _u32], _i),
    "evox_pso_workspace_bytes": ([_i64, _i64, _i, _i, _PSZ], _i),
    "evox_pso_init": ([_i64, _i64, _p, _p, _f32, _f32, _f32, _u64, _p, _PP], _i),
    "evox_pso_step": ([_p, _i, _i64], _i),
    "evox_pso_ask": ([_p, _PP, _PI64, _PI64], _i),
    "evox_pso_tell": ([_p, _p], _i),
    "evox_pso_best": ([_p, _PF32, _PI64, _p], _i),
    "evox_pso_history": ([_p, _p, _i64, _PI64], _i),
    "evox_pso_view": ([_p, _i, _PP, _PI64, _PI64], _i),
    "evox_pso_info": ([_p, _PI64, _PI64, _PI64, _PI64, _PI64, _PI64, _PP], _i),
    "evox_pso_save": ([_p, _p, ctypes.c_size_t, _PSZ], _i),
    "evox_pso_load": ([_p, _p, ctypes.c_size_t], _i),
    "evox_pso_sync": ([_p], _i),
    "evox_pso_destroy": ([_p], _i),
    "evox_pso_set_timing": ([_p, _i], _i),
    "evox_pso_mailbox": ([_p, _PP, _PSZ], _i),
    "evox_pso_mailbox_ipc": ([_p, _p], _i),
    "evox_pso_connect": ([_p, _i, _p], _i),
    "evox_pso_kernel_time": ([_p, ctypes.POINTER(ctypes.c_double), _PI64, _PI64, _i], _i),
    "evox_pso_fin_time": ([_p, ctypes.POINTER(ctypes.c_double), _PI64, _i], _i),
    "evox_cso_workspace_bytes": ([_i64, _i64, _i, _i, _PSZ], _i),
    "evox_cso_init": ([_i64, _i64, _p, _p, _f32, _i64, _u64, _p, _PP], _i),
    "evox_cso_step": ([_p, _i, _i64], _i),
    "evox_cso_best": ([_p, _PF32, _PI64, _p], _i),
    "evox_cso_history": ([_p, _p, _i64, _PI64], _i),
    "evox_cso_view": ([_p, _i, _PP, _PI64, _PI64], _i),
    "evox_cso_info": ([_p, _PI64, _PI64, _PI64, _PI64, _PI64, _PI64, _PP], _i),
    "evox_cso_save": ([_p, _p, ctypes.c_size_t, _PSZ], _i),
    "evox_cso_load": ([_p, _p, ctypes.c_size_t], _i),
    "evox_cso_sync": ([_p], _i),
    "evox_cso_destroy": ([_p], _i),
    "evox_cso_set_timing": ([_p, _i], _i),
    "evox_cso_state": ([_p, _PP, _p], _i),
    "evox_cso_connect": ([_p, _i, _p], _i),
    "evox_cso_kernel_time": ([_p, ctypes.POINTER(ctypes.c_double), _PI64, _PI64, _i], _i),
    "evox_de_workspace_bytes": ([_i64, _i64, _PSZ], _i),
    "evox_de_init": ([_i64, _i64, _p, _p, _f32, _f32, _u64, _p, _PP], _i),
    "evox_de_step": ([_p, _i, _i64], _i),
    "evox_de_best": ([_p, _PF32, _PI64, _p], _i),
    "evox_de_history": ([_p, _p, _i64, _PI64], _i),
    "evox_de_view": ([_p, _i, _PP, _PI64, _PI64], _i),
    "evox_de_info": ([_p, _PI64, _PI64, _PI64, _PI64, _PI64, _PI64, _PP], _i),
    "evox_de_sync": ([_p], _i),
    "evox_de_save": ([_p, _p, ctypes.c_size_t, _PSZ], _i),
    "evox_de_load": ([_p, _p, ctypes.c_size_t], _i),
    "evox_de_set_timing": ([_p, _i], _i),
    "evox_de_state": ([_p, _PP, _p], _i),
    "evox_de_connect": ([_p, _i, _p], _i),
    "evox_de_kernel_time": ([_p, ctypes.POINTER(ctypes.c_double), _PI64, _PI64, _i], _i),
    "evox_de_destroy": ([_p], _i),
    "evox_debug_philox": ([_p, _u32, _u32, _p, _i64, _p], _i),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libevox.so (built in-tree by ``__graft_entry__.build()``); fail loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        msg = lib().evox_last_error().decode(errors="replace")
        raise _EXC.get(status, EvoxError)(status, msg)


def last_error() -> str:
    return lib().evox_last_error().decode(errors="replace")


def version() -> str:
    return lib().evox_version().decode()


def problem_id(problem) -> int:
    if isinstance(problem, str):
        return PROBLEMS[problem.lower()]
    return int(problem)


def shard_rows(pop: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of ``rank`` (R-11)."""
    r0, n = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().evox_shard_rows(pop, world, rank, ctypes.byref(r0), ctypes.byref(n)))
    return r0.value, n.value


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().evox_nccl_unique_id(buf))
    return bytes(buf)


# ----------------------------------------------------------------- tensors
class _DevArray:
    """Zero-copy __cuda_array_interface__ wrapper of a borrowed device pointer."""

    def __init__(self, ptr: int, shape: tuple, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}
        self._owner = owner


def _as_tensor(ptr: int, shape: tuple, typestr: str, owner, device: int):
    import torch
    return torch.as_tensor(_DevArray(ptr, shape, typestr, owner), device=f"cuda:{device}")


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def evaluate(problem, X, dim: Optional[int] = None, out=None, stream=None, flags: int = 0):
    """Problem.evaluate (Eq. (2)): fitness of every row of the CUDA float32 tensor X.

    X is [pop, ld] with ld % 4 == 0 (``dim`` <= ld columns are used; default
    ld).  Returns a [pop] float32 CUDA tensor (``out`` if given)."""
    import torch
    if not (isinstance(X, torch.Tensor) and X.is_cuda and X.dtype == torch.float32):
        raise TypeError("X must be a CUDA float32 tensor (no CPU fallback)")
    if X.dim() != 2 or not X.is_contiguous():
        raise ValueError("X must be a contiguous 2-D tensor [pop, ld]")
    pop, ld = X.shape
    dim = ld if dim is None else int(dim)
    if out is None:
        out = torch.empty(pop, dtype=torch.float32, device=X.device)
    if stream is None:
        stream = torch.cuda.current_stream(X.device)
    _check(lib().evox_eval_ex(problem_id(problem), X.data_ptr(), pop, dim, ld, out.data_ptr(),
                              _stream_ptr(stream), int(flags)))
    return out


def debug_philox(ctr, key0: int, key1: int, stream=None):
    """Philox4x32-10 of a [n,4] int32/uint32 CUDA tensor of counters (test hook)."""
    import torch
    ctr = ctr.contiguous()
    out = torch.empty_like(ctr)
    if stream is None:
        stream = torch.cuda.current_stream(ctr.device)
    _check(lib().evox_debug_philox(ctr.data_ptr(), key0 & 0xFFFFFFFF, key1 & 0xFFFFFFFF,
                                   out.data_ptr(), ctr.shape[0], _stream_ptr(stream)))
    return out


def _bounds(lb, ub, dim):
    lb = np.ascontiguousarray(np.broadcast_to(np.asarray(lb, np.float32), (dim,)))
    ub = np.ascontiguousarray(np.broadcast_to(np.asarray(ub, np.float32), (dim,)))
    return lb, ub


def _device_of(device) -> int:
    if device is not None:
        return int(device)
    import torch
    return torch.cuda.current_device()


def _opts(stream, rank, world, device, nccl_id, workspace, flags=0, peer_timeout_ms=None):
    o = EvoxOpts()
    o.flags = int(flags)
    o.peer_timeout_ms = int(DEFAULT_PEER_TIMEOUT_MS if peer_timeout_ms is None else peer_timeout_ms)
    o.cuda_stream = _stream_ptr(stream)
    o.rank = rank
    o.world = world
    o.device = -1 if device is None else int(device)
    keep = []
    if nccl_id is not None:
        b = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
        keep.append(b)
        o.nccl_id = ctypes.addressof(b)
    if workspace is not None:
        o.workspace = workspace.data_ptr()
        o.workspace_bytes = workspace.numel() * workspace.element_size()
        keep.append(workspace)
    return o, keep


class _Handle:
    _prefix = ""

    def _fn(self, name):
        return getattr(lib(), f"evox_{self._prefix}_{name}")

    def close(self):
        if getattr(self, "_h", None):
            self._fn("destroy")(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self) -> dict:
        v = [ctypes.c_int64() for _ in range(6)]
        st = ctypes.c_void_p()
        _check(self._fn("info")(self._h, *[ctypes.byref(x) for x in v], ctypes.byref(st)))
        keys = ("pop", "dim", "ld", "row0", "rows", "t")
        d = {k: x.value for k, x in zip(keys, v)}
        d["stream"] = st.value or 0
        return d

    @property
    def stream(self):
        """The CUDA stream the handle enqueues on (torch.cuda.ExternalStream)."""
        import torch
        return torch.cuda.ExternalStream(self.info()["stream"], device=f"cuda:{self.device}")

    def sync(self):
        _check(self._fn("sync")(self._h))

    def set_timing(self, enable: bool = True):
        """Bracket every generation kernel with CUDA events (launches un-graphed)."""
        _check(self._fn("set_timing")(self._h, int(bool(enable))))

    def kernel_time(self, reset: bool = False) -> tuple[float, int, int]:
        """(summed generation-kernel device time in ms, generations they ran, launches)."""
        ms, n, k = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()
        _check(self._fn("kernel_time")(self._h, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(k),
                                       int(reset)))
        return ms.value, n.value, k.value

    def history(self) -> np.ndarray:
        n = ctypes.c_int64()
        _check(self._fn("history")(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(n.value, 0), np.float32)
        if n.value > 0:
            _check(self._fn("history")(self._h, out.ctypes.data, n.value, ctypes.byref(n)))
        return out

    def view(self, field: str):
        """Borrowed zero-copy torch view of this rank's state (valid until the next call)."""
        ptr, rows, ld = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        _check(self._fn("view")(self._h, FIELDS[field], ctypes.byref(ptr), ctypes.byref(rows),
                                ctypes.byref(ld)))
        if field in ("X", "V", "P"):
            shape = (rows.value, ld.value)
        elif field == "G":
            shape = (ld.value,)
        else:
            shape = (rows.value,)
        return _as_tensor(ptr.value, shape, "<f4", self, self.device)

    def save(self) -> bytes:
        used = ctypes.c_size_t()
        _check(self._fn("save")(self._h, None, 0, ctypes.byref(used)))
        buf = ctypes.create_string_buffer(used.value)
        _check(self._fn("save")(self._h, buf, used.value, ctypes.byref(used)))
        return buf.raw[: used.value]

    def load(self, blob: bytes):
        _check(self._fn("load")(self._h, blob, len(blob)))

    def best(self, with_row: bool = True):
        """(best fitness, global index, best row as numpy [dim] or None).  Synchronising."""
        f, i = ctypes.c_float(), ctypes.c_int64()
        row = np.zeros(self.dim, np.float32) if with_row else None
        _check(self._fn("best")(self._h, ctypes.byref(f), ctypes.byref(i),
                                row.ctypes.data if with_row else None))
        return float(f.value), int(i.value), row


class PSO(_Handle):
    """gbest PSO with inertia, one shard of a row-sharded population."""
    _prefix = "pso"

    def __init__(self, pop: int, dim: int, lb=-5.12, ub=5.12, w: float = 0.6,
                 phi_p: float = 2.5, phi_g: float = 0.8, seed: int = 0, stream=None,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 device: Optional[int] = None, workspace=None, flags: int = 0,
                 peer_timeout_ms: Optional[int] = None):
        self._h = None
        self.pop, self.dim = int(pop), int(dim)
        lbv, ubv = _bounds(lb, ub, self.dim)
        opts, self._keep = _opts(stream, rank, world, device, nccl_id, workspace, flags,
                                 peer_timeout_ms)
        h = ctypes.c_void_p()
        _check(lib().evox_pso_init(self.pop, self.dim, lbv.ctypes.data, ubv.ctypes.data,
                                   float(w), float(phi_p), float(phi_g),
                                   int(seed) & 0xFFFFFFFFFFFFFFFF, ctypes.byref(opts),
                                   ctypes.byref(h)))
        self._h = h.value
        self.device = _device_of(device)

    @staticmethod
    def workspace_bytes(pop, dim, world=1, rank=0) -> int:
        b = ctypes.c_size_t()
        _check(lib().evox_pso_workspace_bytes(pop, dim, world, rank, ctypes.byref(b)))
        return b.value

    def step(self, problem, n_gens: int = 1):
        """Workflow.step x n_gens (asynchronous)."""
        _check(lib().evox_pso_step(self._h, problem_id(problem), int(n_gens)))

    def ask(self):
        """Algorithm.ask: borrowed [rows, ld] view of the population to evaluate.  The move
        that produces it is queued on `self.stream`: evaluate it on that stream (e.g.
        `evaluate(problem, X, stream=pso.stream)`) or synchronize first."""
        ptr, rows, ld = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().evox_pso_ask(self._h, ctypes.byref(ptr), ctypes.byref(rows),
                                  ctypes.byref(ld)))
        return _as_tensor(ptr.value, (rows.value, ld.value), "<f4", self, self.device)

    # ---- in-kernel peer-memory exchange (NEXT #1)
    def mailbox(self) -> tuple[int, int]:
        ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().evox_pso_mailbox(self._h, ctypes.byref(ptr), ctypes.byref(n)))
        return ptr.value, n.value

    def mailbox_ipc(self) -> bytes:
        buf = (ctypes.c_uint8 * 64)()
        _check(lib().evox_pso_mailbox_ipc(self._h, buf))
        return bytes(buf)

    def connect_local(self, mailboxes):
        """Same-process group: `mailboxes` = [PSO.mailbox()[0] of rank r for r in range(world)]."""
        arr = (ctypes.c_void_p * len(mailboxes))(*[int(m) for m in mailboxes])
        _check(lib().evox_pso_connect(self._h, 0, arr))

    def connect_ipc(self, handles):
        """Multi-process group: `handles` = [64-byte PSO.mailbox_ipc() of rank r]."""
        buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles))
        _check(lib().evox_pso_connect(self._h, 1, buf))

    def fin_time(self, reset: bool = False) -> tuple[float, int]:
        """(summed device time in ms of the gbest-publication / exchange kernel, launches)."""
        ms, k = ctypes.c_double(), ctypes.c_int64()
        _check(lib().evox_pso_fin_time(self._h, ctypes.byref(ms), ctypes.byref(k), int(reset)))
        return ms.value, k.value

    def tell(self, fitness):
        """Algorithm.tell with a [rows] float32 CUDA tensor of this rank's fitness."""
        import torch
        if not (isinstance(fitness, torch.Tensor) and fitness.is_cuda
                and fitness.dtype == torch.float32 and fitness.is_contiguous()):
            raise TypeError("fitness must be a contiguous CUDA float32 tensor")
        # order the caller's producer stream before the handle's stream
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(fitness.device))
        self.stream.wait_event(ev)
        _check(lib().evox_pso_tell(self._h, fitness.data_ptr()))


class CSO(_Handle):
    """Competitive swarm optimizer (Table II; R-8)."""
    _prefix = "cso"

    def __init__(self, pop: int, dim: int, lb=-5.12, ub=5.12, phi: float = 0.0, block: int = 0,
                 seed: int = 0, stream=None, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, device: Optional[int] = None, workspace=None,
                 flags: int = 0, peer_timeout_ms: Optional[int] = None):
        self._h = None
        self.pop, self.dim = int(pop), int(dim)
        lbv, ubv = _bounds(lb, ub, self.dim)
        opts, self._keep = _opts(stream, rank, world, device, nccl_id, workspace, flags,
                                 peer_timeout_ms)
        h = ctypes.c_void_p()
        _check(lib().evox_cso_init(self.pop, self.dim, lbv.ctypes.data, ubv.ctypes.data,
                                   float(phi), int(block), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                   ctypes.byref(opts), ctypes.byref(h)))
        self._h = h.value
        self.device = _device_of(device)

    @staticmethod
    def workspace_bytes(pop, dim, world=1, rank=0) -> int:
        b = ctypes.c_size_t()
        _check(lib().evox_cso_workspace_bytes(pop, dim, world, rank, ctypes.byref(b)))
        return b.value

    def step(self, problem, n_gens: int = 1):
        _check(lib().evox_cso_step(self._h, problem_id(problem), int(n_gens)))

    def state_base(self) -> int:
        p = ctypes.c_void_p()
        _check(lib().evox_cso_state(self._h, ctypes.byref(p), None))
        return p.value

    def state_ipc(self) -> bytes:
        buf = (ctypes.c_uint8 * 64)()
        _check(lib().evox_cso_state(self._h, None, buf))
        return bytes(buf)

    def connect_local(self, bases):
        arr = (ctypes.c_void_p * len(bases))(*[int(b) for b in bases])
        _check(lib().evox_cso_connect(self._h, 0, arr))

    def connect_ipc(self, handles):
        buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles))
        _check(lib().evox_cso_connect(self._h, 1, buf))


class DE(_Handle):
    """DE/rand/1/bin (the DE of the paper's experiment; R-14)."""
    _prefix = "de"

    def __init__(self, pop: int, dim: int, lb=-5.12, ub=5.12, F: float = 0.5, CR: float = 0.9,
                 seed: int = 0, stream=None, rank: int = 0, world: int = 1,
                 device: Optional[int] = None, workspace=None, flags: int = 0,
                 peer_timeout_ms: Optional[int] = None):
        self._h = None
        self.pop, self.dim = int(pop), int(dim)
        lbv, ubv = _bounds(lb, ub, self.dim)
        opts, self._keep = _opts(stream, rank, world, device, None, workspace, flags,
                                 peer_timeout_ms)
        h = ctypes.c_void_p()
        _check(lib().evox_de_init(self.pop, self.dim, lbv.ctypes.data, ubv.ctypes.data, float(F),
                                  float(CR), int(seed) & 0xFFFFFFFFFFFFFFFF, ctypes.byref(opts),
                                  ctypes.byref(h)))
        self._h = h.value
        self.device = _device_of(device)

    @staticmethod
    def workspace_bytes(pop, dim) -> int:
        b = ctypes.c_size_t()
        _check(lib().evox_de_workspace_bytes(pop, dim, ctypes.byref(b)))
        return b.value

    def step(self, problem, n_gens: int = 1):
        _check(lib().evox_de_step(self._h, problem_id(problem), int(n_gens)))

    def state_base(self) -> int:
        p = ctypes.c_void_p()
        _check(lib().evox_de_state(self._h, ctypes.byref(p), None))
        return p.value

    def state_ipc(self) -> bytes:
        buf = (ctypes.c_uint8 * 64)()
        _check(lib().evox_de_state(self._h, None, buf))
        return bytes(buf)

    def connect_local(self, bases):
        arr = (ctypes.c_void_p * len(bases))(*[int(b) for b in bases])
        _check(lib().evox_de_connect(self._h, 0, arr))

    def connect_ipc(self, handles):
        buf = ctypes.create_string_buffer(b"".join(bytes(h) for h in handles))
        _check(lib().evox_de_connect(self._h, 1, buf))
