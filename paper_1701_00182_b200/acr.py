"""Reference-facing API of the B200 ACR path (ctypes over libacrgpu.so).

Mirrors the reference's public surface for the H-matrix hot path
(/root/reference/proj/core/include/acr/acr.hpp:15-23,185-224 and errors.hpp:10-60):

    AcrConfig                       acr.hpp:15-23
    acr_factor(system, config)      acr.hpp:222      -> AcrFactorization
    AcrFactorization.solve(f)       acr.hpp:205      (f: (n, dim) or (nrhs, n, dim))
    .factor_bytes() / .inverse_rank_stats() / .level_info()   acr.hpp:207-210
    acr_solve(fact, f)              acr.hpp:223
    DimensionError / SingularBlockError / LeafMemoryError / UsageError   errors.hpp

There is no CPU fallback: if libacrgpu.so is missing or no CUDA device is
present, every call raises.  ``ArithmeticMode.Dense`` (the reference's exact
DenseKernel oracle) is a CPU oracle mode and is rejected here (UsageError).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os

import numpy as np

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # libacrgpu's 16 streams; read at context creation

from . import problems

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.environ.get("ACRGPU_LIB") or os.path.join(_HERE, "libacrgpu.so")  # override: A/B of kernel variants


# ---------------------------------------------------------------- errors (errors.hpp)
class Error(RuntimeError):
    pass


class DimensionError(Error):
    def __init__(self, msg, plane=-1):
        super().__init__(msg)
        self.plane_index = plane


class SingularBlockError(Error):
    def __init__(self, msg, level=-1, plane=-1, rows=(-1, -1)):
        super().__init__(msg)
        self.level = level
        self.plane = plane
        self.rows = rows


class LeafMemoryError(Error):
    pass


class IndefiniteError(Error):
    """pcg: nonpositive search-direction curvature (errors.hpp:45-48)."""


class DivergenceError(Error):
    """iterative_refinement: three consecutive residual increases (errors.hpp:51-54)."""


class UsageError(Error):
    pass


class DeviceError(Error):
    pass


class ArithmeticMode(enum.Enum):
    Dense = 0
    HMatrix = 1


class Admissibility(enum.Enum):
    Standard = 0
    Weak = 1


@dataclasses.dataclass
class AcrConfig:
    """AcrConfig (acr.hpp:15-23).  ``exact_dense_products`` is the documented
    deviation switch, off by default."""

    mode: ArithmeticMode = ArithmeticMode.HMatrix
    eps: float = 1e-3
    eta: float = 2.0
    leaf_size: int = 32
    admissibility: Admissibility = Admissibility.Standard
    stop_planes: int = 1
    leaf_memory_cap: int = 2 << 30
    exact_dense_products: bool = False


@dataclasses.dataclass
class RankStats:
    average_rank: float = 0.0
    largest_rank: int = 0
    dense_leaf_count: int = 0
    lowrank_leaf_count: int = 0
    bytes: int = 0


@dataclasses.dataclass
class LevelInfo:
    level: int
    plane_count: int
    eliminated: int
    bytes: int
    largest_rank: int
    average_rank: float


# ---------------------------------------------------------------- ctypes layer
class _Err(C.Structure):
    _fields_ = [("code", C.c_int), ("level", C.c_int), ("plane", C.c_int), ("row_begin", C.c_int),
                ("row_end", C.c_int), ("msg", C.c_char * 256)]


class _Cfg(C.Structure):
    _fields_ = [("eps", C.c_double), ("eta", C.c_double), ("leaf_size", C.c_int), ("weak", C.c_int),
                ("stop_planes", C.c_int), ("leaf_memory_cap", C.c_long), ("flags", C.c_int)]


class _Sys(C.Structure):
    _fields_ = [("n", C.c_int), ("dim", C.c_int), ("coords", C.POINTER(C.c_double)),
                ("blk_off", C.POINTER(C.c_long)), ("rows", C.POINTER(C.c_int)), ("cols", C.POINTER(C.c_int)),
                ("vals", C.POINTER(C.c_double))]


class _Stats(C.Structure):
    _fields_ = [("average_rank", C.c_double), ("largest_rank", C.c_int), ("dense_leaf_count", C.c_int),
                ("lowrank_leaf_count", C.c_int), ("inverse_bytes", C.c_long), ("factor_bytes", C.c_long)]


class _Level(C.Structure):
    _fields_ = [("level", C.c_int), ("plane_count", C.c_int), ("eliminated", C.c_int), ("bytes", C.c_long),
                ("largest_rank", C.c_int), ("average_rank", C.c_double)]


class _Trace(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("apply_time", C.c_double),
                ("total_time", C.c_double)]


class _Timing(C.Structure):
    _fields_ = [("lift_ms", C.c_double), ("factor_ms", C.c_double), ("solve_ms", C.c_double),
                ("flops_nominal", C.c_double), ("flops_svd", C.c_double), ("flops_qr", C.c_double),
                ("flops_gemm", C.c_double), ("flops_lu", C.c_double), ("factor_launches", C.c_long),
                ("solve_launches", C.c_long)]


class _Msg(C.Structure):
    _fields_ = [("level", C.c_int), ("from_plane", C.c_int), ("to_plane", C.c_int), ("solve_phase", C.c_int),
                ("bytes", C.c_long)]


SYMBOLS = {
    "acrgpu_version": (C.c_char_p, []),
    "acrgpu_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_ctx_destroy": (None, [C.c_void_p]),
    "acrgpu_factor": (C.c_int, [C.c_void_p, C.POINTER(_Sys), C.POINTER(_Cfg), C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_factor_destroy": (None, [C.c_void_p]),
    "acrgpu_system_upload": (C.c_int, [C.c_void_p, C.POINTER(_Sys), C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_system_destroy": (None, [C.c_void_p]),
    "acrgpu_factor_resident": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(_Cfg), C.POINTER(C.c_void_p),
                                         C.POINTER(_Err)]),
    "acrgpu_solve": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(_Err)]),
    "acrgpu_solve_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(_Err)]),
    "acrgpu_stats": (C.c_int, [C.c_void_p, C.POINTER(_Stats)]),
    "acrgpu_level_info": (C.c_int, [C.c_void_p, C.POINTER(_Level), C.c_int]),
    "acrgpu_dinv_ranks": (C.c_long, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_long]),
    "acrgpu_timing_get": (C.c_int, [C.c_void_p, C.POINTER(_Timing)]),
    "acrgpu_messages": (C.c_long, [C.c_void_p, C.POINTER(_Msg), C.c_long]),
    "acrgpu_profile_report": (C.c_long, [C.c_char_p, C.c_long, C.c_int]),
    "acrgpu_profile_select": (None, [C.c_char_p]),
    "acrgpu_structure": (C.c_long, [C.c_int, C.POINTER(C.c_double), C.c_int, C.c_double, C.c_int,
                                     C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_long, C.POINTER(_Err)]),
    "acrgpu_comm_unique_id": (C.c_int, [C.c_char_p, C.POINTER(_Err)]),
    "acrgpu_comm_create": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_comm_create_local": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_comm_create_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                          C.POINTER(_Err)]),
    "acrgpu_comm_destroy": (None, [C.c_void_p]),
    "acrgpu_factor_partitioned": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(_Sys), C.POINTER(_Cfg),
                                            C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_factor_partitioned_resident": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(_Cfg),
                                                     C.POINTER(C.c_void_p), C.POINTER(_Err)]),
    "acrgpu_pcg": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                             C.POINTER(C.c_double), C.POINTER(_Trace), C.POINTER(_Err)]),
    "acrgpu_refine": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_double), C.POINTER(_Trace), C.POINTER(_Err)]),
}

COMM_ID_BYTES = 128

_lib = None


def lib():
    """Load libacrgpu.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise DeviceError(f"libacrgpu.so not built ({_LIB}); run paper_1701_00182_b200.build.build()")
        L = C.CDLL(_LIB)
        for name, (res, args) in SYMBOLS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _raise(err: _Err):
    msg = err.msg.decode(errors="replace")
    code = err.code
    if code == 1:
        raise DimensionError(msg, err.plane)
    if code == 2:
        raise SingularBlockError(msg, err.level, err.plane, (err.row_begin, err.row_end))
    if code == 3:
        raise LeafMemoryError(msg)
    if code == 4:
        raise UsageError(msg)
    if code == 6:
        raise IndefiniteError(msg)
    if code == 7:
        raise DivergenceError(msg)
    if code == 5:
        raise DeviceError(msg)
    raise Error(msg or f"acrgpu error {code}")


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Context:
    """One CUDA device.  Reused across factorizations (device arenas are sized once)."""

    def __init__(self, device: int = -1):
        self.h = C.c_void_p()
        err = _Err()
        if lib().acrgpu_ctx_create(device, C.byref(self.h), C.byref(err)):
            _raise(err)

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().acrgpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


def _cfg(config: AcrConfig) -> _Cfg:
    if config.mode != ArithmeticMode.HMatrix:
        raise UsageError("the GPU path implements ArithmeticMode.HMatrix only (Dense mode is the CPU oracle)")
    return _Cfg(config.eps, config.eta, config.leaf_size,
                1 if config.admissibility == Admissibility.Weak else 0, config.stop_planes,
                config.leaf_memory_cap, 1 if config.exact_dense_products else 0)


class AcrFactorization:
    """Reusable elimination record (acr.hpp:195-219); immutable after construction."""

    def __init__(self, handle, system, config, ctx):
        self.h = handle
        self.config = config
        self.n = system.n
        self.dim = system.dim
        self._ctx = ctx  # keep the context alive

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                lib().acrgpu_factor_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def plane_count(self):
        return self.n

    def plane_dim(self):
        return self.dim

    def solve(self, f):
        """f: (n, dim) -> (n, dim), or (nrhs, n, dim) -> (nrhs, n, dim) in one pass."""
        f = np.asarray(f, dtype=np.float64)
        squeeze = f.ndim == 2
        f3 = f[None] if squeeze else f
        if f3.ndim != 3 or f3.shape[1] != self.n:
            raise DimensionError(f"solve: right-hand side has {f3.shape[1] if f3.ndim == 3 else '?'} planes, "
                                 f"factorization has {self.n}")
        if f3.shape[2] != self.dim:
            raise DimensionError("solve: plane right-hand side dimension mismatch", 0)
        f3 = np.ascontiguousarray(f3)
        u = np.empty_like(f3)
        err = _Err()
        if lib().acrgpu_solve(self.h, f3.shape[0], f3.ctypes.data, u.ctypes.data, C.byref(err)):
            _raise(err)
        return u[0] if squeeze else u

    def solve_device(self, f_ptr: int, u_ptr: int, nrhs: int):
        """Device-resident solve (raw CUDA pointers, layout [nrhs][n][dim])."""
        err = _Err()
        if lib().acrgpu_solve_device(self.h, nrhs, C.c_void_p(f_ptr), C.c_void_p(u_ptr), C.byref(err)):
            _raise(err)

    def _stats(self):
        s = _Stats()
        lib().acrgpu_stats(self.h, C.byref(s))
        return s

    def factor_bytes(self) -> int:
        return int(self._stats().factor_bytes)

    def inverse_rank_stats(self) -> RankStats:
        s = self._stats()
        return RankStats(s.average_rank, s.largest_rank, s.dense_leaf_count, s.lowrank_leaf_count, s.inverse_bytes)

    def level_info(self):
        arr = (_Level * 64)()
        k = lib().acrgpu_level_info(self.h, arr, 64)
        return [LevelInfo(a.level, a.plane_count, a.eliminated, a.bytes, a.largest_rank, a.average_rank)
                for a in arr[:k]]

    def dinv_ranks(self, level: int, plane: int):
        n = lib().acrgpu_dinv_ranks(self.h, level, plane, None, 0)
        if n < 0:
            return None
        out = np.zeros(n, np.int32)
        lib().acrgpu_dinv_ranks(self.h, level, plane, _p(out, C.c_int), n)
        return out

    def messages(self) -> list:
        """Elimination-payload records of a partitioned factorization (MessageRecord,
        parallel.hpp:24-30); empty for a single-rank factorization."""
        k = lib().acrgpu_messages(self.h, None, 0)
        arr = (_Msg * max(k, 1))()
        k = lib().acrgpu_messages(self.h, arr, k)
        return [MessageRecord(a.level, a.from_plane, a.to_plane, int(a.bytes), bool(a.solve_phase)) for a in arr[:k]]

    def timing(self) -> dict:
        t = _Timing()
        lib().acrgpu_timing_get(self.h, C.byref(t))
        return {k: getattr(t, k) for k, _ in _Timing._fields_}


def _sys_struct(system):
    keep = (np.ascontiguousarray(system.coords, np.float64), np.ascontiguousarray(system.blk_off, np.int64),
            np.ascontiguousarray(system.rows, np.int32), np.ascontiguousarray(system.cols, np.int32),
            np.ascontiguousarray(system.vals, np.float64))
    coords, off, rows, cols, vals = keep
    s = _Sys(system.n, system.dim, _p(coords, C.c_double), _p(off, C.c_long), _p(rows, C.c_int), _p(cols, C.c_int),
             _p(vals, C.c_double))
    return s, keep


class DeviceSystem:
    """A system validated and uploaded to HBM once (acrgpu_system_upload)."""

    def __init__(self, system: problems.System, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.system = system
        s, keep = _sys_struct(system)
        self.h = C.c_void_p()
        err = _Err()
        if lib().acrgpu_system_upload(self.ctx.h, C.byref(s), C.byref(self.h), C.byref(err)):
            _raise(err)

    def __del__(self):
        try:
            if getattr(self, "h", None) and self.h.value:
                lib().acrgpu_system_destroy(self.h)
                self.h = None
        except Exception:
            pass


def acr_factor(system, config: AcrConfig | None = None, ctx: Context | None = None):
    """acr::acr_factor (acr.cpp:366-384) on the GPU.  ``system`` is a problems.System
    (host COO, uploaded inside the call) or a DeviceSystem (already resident in HBM)."""
    config = config or AcrConfig()
    cfg = _cfg(config)
    h = C.c_void_p()
    err = _Err()
    if isinstance(system, DeviceSystem):
        ctx = system.ctx
        rc = lib().acrgpu_factor_resident(ctx.h, system.h, C.byref(cfg), C.byref(h), C.byref(err))
        host = system.system
    else:
        ctx = ctx or default_context()
        s, keep = _sys_struct(system)
        rc = lib().acrgpu_factor(ctx.h, C.byref(s), C.byref(cfg), C.byref(h), C.byref(err))
        host = system
    if rc:
        _raise(err)
    return AcrFactorization(h, host, config, ctx)


_EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                          C.POINTER(C.c_long), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.POINTER(C.c_long))


def torch_exchange(group=None):
    """Exchange callable for ``Comm.host`` over torch.distributed point-to-point (any backend
    with CPU tensors, e.g. gloo): per peer, the k-th send matches the peer's k-th receive
    (tag k)."""
    import torch
    import torch.distributed as dist

    def exchange(sends, recvs):
        reqs, keep, tags = [], [], {}
        for dst, mv in sends:
            k = tags.get(("s", dst), 0)
            tags[("s", dst)] = k + 1
            t = torch.frombuffer(bytearray(mv), dtype=torch.uint8) if len(mv) else torch.zeros(0, dtype=torch.uint8)
            keep.append(t)
            reqs.append(dist.isend(t, dst, group=group, tag=k))
        outs = []
        for src, mv in recvs:
            k = tags.get(("r", src), 0)
            tags[("r", src)] = k + 1
            t = torch.empty(len(mv), dtype=torch.uint8)
            outs.append((mv, t))
            reqs.append(dist.irecv(t, src, group=group, tag=k))
        for r in reqs:
            r.wait()
        for mv, t in outs:
            if len(mv):
                mv[:] = t.numpy().tobytes()  # mv: unsigned-byte view of the library's host buffer

    return exchange


class Comm:
    """Plane-partition communicator (execute_parallel_factor, parallel.hpp:60-61).

    ``Comm.local(p)``: p ranks run in-process on one device (checks the partitioned
    data path; the factorization handle holds every rank).  ``Comm.nccl(uid, p, rank)``:
    one rank per process/GPU over NCCL point-to-point; ``uid`` from ``Comm.unique_id()``
    on rank 0, shared out of band (e.g. ``torch.distributed.broadcast_object_list``)."""

    def __init__(self, handle, nranks, rank, local):
        self.h, self.nranks, self.rank, self.local = handle, nranks, rank, local

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(COMM_ID_BYTES)
        err = _Err()
        if lib().acrgpu_comm_unique_id(buf, C.byref(err)):
            _raise(err)
        return buf.raw

    @classmethod
    def local_ranks(cls, nranks: int) -> "Comm":
        h = C.c_void_p()
        err = _Err()
        if lib().acrgpu_comm_create_local(nranks, C.byref(h), C.byref(err)):
            _raise(err)
        return cls(h, nranks, 0, True)

    @classmethod
    def host(cls, exchange, nranks: int, rank: int) -> "Comm":
        """Host-staged communicator: ``exchange(sends, recvs)`` moves the wire images of one
        phase -- ``sends`` a list of (dst rank, memoryview), ``recvs`` a list of (src rank,
        writable memoryview); messages between one pair of ranks must be matched in list
        order (``torch_exchange`` does it with torch.distributed isend/irecv)."""

        def fn(user, nsend, dst, sbuf, sbytes, nrecv, src, rbuf, rbytes):
            try:
                def view(addr, n):
                    return memoryview((C.c_ubyte * n).from_address(addr)).cast("B") if n else memoryview(bytearray(0))

                sends = [(dst[i], view(sbuf[i], sbytes[i])) for i in range(nsend)]
                recvs = [(src[i], view(rbuf[i], rbytes[i])) for i in range(nrecv)]
                exchange(sends, recvs)
                return 0
            except Exception:  # pragma: no cover - surfaced as ACRGPU_E_DEVICE
                import traceback
                traceback.print_exc()
                return 1

        cb = _EXCHANGE_FN(fn)
        h = C.c_void_p()
        err = _Err()
        if lib().acrgpu_comm_create_host(cb, None, nranks, rank, C.byref(h), C.byref(err)):
            _raise(err)
        c = cls(h, nranks, rank, False)
        c._cb = cb  # keep the trampoline alive as long as the communicator
        return c

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int) -> "Comm":
        h = C.c_void_p()
        err = _Err()
        if lib().acrgpu_comm_create(uid, nranks, rank, C.byref(h), C.byref(err)):
            _raise(err)
        return cls(h, nranks, rank, False)

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().acrgpu_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def acr_factor_partitioned(system, comm: Comm, config: AcrConfig | None = None, ctx: Context | None = None):
    """execute_parallel_factor (parallel.cpp:96-297) on GPUs: planes owned per
    plan_schedule(n, comm.nranks); bitwise identical to acr_factor."""
    config = config or AcrConfig()
    cfg = _cfg(config)
    h = C.c_void_p()
    err = _Err()
    if isinstance(system, DeviceSystem):
        ctx = system.ctx
        rc = lib().acrgpu_factor_partitioned_resident(ctx.h, comm.h, system.h, C.byref(cfg), C.byref(h), C.byref(err))
        system = system.system
    else:
        ctx = ctx or default_context()
        s, keep = _sys_struct(system)
        rc = lib().acrgpu_factor_partitioned(ctx.h, comm.h, C.byref(s), C.byref(cfg), C.byref(h), C.byref(err))
    if rc:
        _raise(err)
    f = AcrFactorization(h, system, config, ctx)
    f._comm = comm  # keep the communicator alive
    return f


@dataclasses.dataclass
class MessageRecord:
    """parallel.hpp:24-30."""
    level: int
    from_plane: int
    to_plane: int
    bytes: int
    solve_phase: bool = False


@dataclasses.dataclass
class LevelTraffic:
    """parallel.hpp:32-38."""
    level: int = 0
    messages: int = 0
    bytes: int = 0
    active_workers: int = 0
    idle_workers: int = 0


@dataclasses.dataclass
class MessageLedger:
    """parallel.hpp:40-48: cross-worker traffic per level, factor and solve phases."""
    factor: list
    solve: list
    records: list

    def total_messages(self) -> int:
        return len(self.records)

    def total_bytes(self) -> int:
        return sum(r.bytes for r in self.records)


def message_ledger(fact: AcrFactorization, plan) -> MessageLedger:
    """Aggregate a partitioned factorization's records the way run_parallel does
    (parallel.cpp:356-378).  Factor-phase records come from the device run; the solve
    phase moves one plane vector u_j (8*dim bytes) from the owner of each retained plane
    to the owner of each eliminated neighbour held elsewhere (parallel.cpp:264-274),
    which depends only on the plan."""
    from .plan import eliminated_positions
    levels = len(fact.level_info()) - 1
    factor = [LevelTraffic(level=i) for i in range(levels)]
    solve = [LevelTraffic(level=i) for i in range(levels)]
    for i in range(levels):
        active = len(set(plan.assignment[i]))
        for part in (factor[i], solve[i]):
            part.active_workers = active
            part.idle_workers = plan.p - active
    records = list(fact.messages())
    for i in range(levels):
        own = plan.assignment[i]
        m = len(own)
        is_elim = [False] * m
        for e in eliminated_positions(m):
            is_elim[e] = True
        for j in range(m):
            if is_elim[j]:
                continue
            for nb in (j - 1, j + 1):
                if 0 <= nb < m and is_elim[nb] and own[nb] != own[j]:
                    records.append(MessageRecord(i, j, nb, 8 * fact.dim, True))
    for r in records:
        part = solve[r.level] if r.solve_phase else factor[r.level]
        part.messages += 1
        part.bytes += r.bytes
    return MessageLedger(factor, solve, records)


def acr_solve(fact: AcrFactorization, f):
    return fact.solve(f)


def profile_select(names: str | None) -> None:
    """Time these kernels' launches with CUDA events on their streams: None/"" none, "*" all,
    else a comma-separated list of kernel names (overrides ACRGPU_PROFILE)."""
    lib().acrgpu_profile_select((names or "").encode())


def profile_report(reset: bool = True) -> str:
    """Per-kernel device totals of the launches selected by profile_select / ACRGPU_PROFILE
    (name -> ms, launches, CTAs, nominal flops)."""
    n = lib().acrgpu_profile_report(None, 0, 0)
    buf = C.create_string_buffer(n + 1)
    lib().acrgpu_profile_report(buf, n + 1, 1 if reset else 0)
    return buf.value.decode()


def structure(coords, leaf_size=32, eta=2.0, weak=False):
    """(perm, leaves) of the library's cluster / block cluster tree (no device needed)."""
    coords = np.ascontiguousarray(coords, np.float64)
    dim = coords.shape[0]
    err = _Err()
    n = lib().acrgpu_structure(dim, _p(coords, C.c_double), leaf_size, eta, 1 if weak else 0, None, None, 0,
                               C.byref(err))
    if n < 0:
        _raise(err)
    perm = np.zeros(dim, np.int32)
    leaves = np.zeros((n, 5), np.int32)
    lib().acrgpu_structure(dim, _p(coords, C.c_double), leaf_size, eta, 1 if weak else 0, _p(perm, C.c_int),
                           _p(leaves, C.c_int), n, C.byref(err))
    return perm, leaves


# ---------------------------------------------------------------- Krylov drivers
@dataclasses.dataclass
class IterationTrace:
    """acr::IterationTrace (krylov.hpp:8-14)."""
    converged: bool = False
    iterations: int = 0
    residual_history: list = dataclasses.field(default_factory=list)
    apply_time: float = 0.0
    total_time: float = 0.0


@dataclasses.dataclass
class KrylovResult:
    """acr::KrylovResult (krylov.hpp:16-19): u is (n, dim)."""
    u: np.ndarray
    trace: IterationTrace


def _krylov(entry, system, precond, tol, max_iterations):
    import torch  # device buffers only (plumbing); the iteration runs in libacrgpu
    dsys = system if isinstance(system, DeviceSystem) else DeviceSystem(system, precond._ctx if precond else None)
    host = dsys.system
    f = np.ascontiguousarray(np.asarray(host.rhs, np.float64).reshape(-1, host.n, host.dim)[0])
    dev = torch.device("cuda", torch.cuda.current_device())
    f_d = torch.from_numpy(f).to(dev)
    u_d = torch.empty_like(f_d)
    hist = np.zeros(max(1, max_iterations))
    tr = _Trace()
    err = _Err()
    torch.cuda.synchronize()
    rc = getattr(lib(), entry)(dsys.ctx.h, dsys.h, precond.h if precond is not None else None, float(tol),
                               int(max_iterations), C.c_void_p(f_d.data_ptr()), C.c_void_p(u_d.data_ptr()),
                               _p(hist, C.c_double), C.byref(tr), C.byref(err))
    if rc:
        _raise(err)
    u = u_d.cpu().numpy()
    return KrylovResult(u, IterationTrace(bool(tr.converged), int(tr.iterations),
                                          [float(x) for x in hist[:tr.iterations]], tr.apply_time, tr.total_time))


def pcg(system, precond: AcrFactorization | None, tol: float, max_iterations: int) -> KrylovResult:
    """acr::pcg (krylov.cpp:38-90): preconditioned CG with true-residual stopping on the
    system's first right-hand side; precond None runs plain CG.  Raises IndefiniteError."""
    return _krylov("acrgpu_pcg", system, precond, tol, max_iterations)


def iterative_refinement(system, precond: AcrFactorization, tol: float, max_iterations: int) -> KrylovResult:
    """acr::iterative_refinement (krylov.cpp:92-131): u += M^{-1}(f - A u).  Raises
    DivergenceError after three consecutive residual increases."""
    return _krylov("acrgpu_refine", system, precond, tol, max_iterations)
