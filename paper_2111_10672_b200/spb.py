"""Python mirror of the reference SPB interface over the C ABI.

The reference (/root/reference/proj/include/jigsaw/spb/{spb,model}.hpp) is a
C++ library; its drop-in replacement here is libspb_b200.so
(include/spb_b200.h) plus the C++ adapter (include/spb_b200/jigsaw_spb.hpp).
This module binds the same C ABI with ctypes so tests and the bench read like
the reference's own tests: the same names, argument meanings and error types
(ArgumentError / ProtocolError / ConfigError, errors.hpp:9-25).

There is no CPU fallback: every compute call goes through the CUDA library,
and importing the module fails loudly if the library cannot be loaded.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPB_LIB_PATH", os.path.join(_PKG, "libspb_b200.so"))  # override: tuning variants


class SpbError(Exception):
    """Base of the errors raised by the C ABI."""


class ArgumentError(SpbError, ValueError):
    """jigsaw::ArgumentError (errors.hpp:9-12)."""


class ProtocolError(SpbError, RuntimeError):
    """jigsaw::ProtocolError (errors.hpp:16-19)."""


class ConfigError(SpbError, RuntimeError):
    """jigsaw::ConfigError (errors.hpp:22-25)."""


class CudaError(SpbError, RuntimeError):
    pass


class NcclError(SpbError, RuntimeError):
    pass


_STATUS = {1: ArgumentError, 2: ProtocolError, 3: ConfigError, 4: CudaError, 5: NcclError}

_lib: Optional[C.CDLL] = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads libspb_b200.so (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        from . import build as _build

        _build.build()
    if "SPB_NCCL_LIB" not in os.environ:
        # Share torch's NCCL when it is installed (the engine dlopens NCCL lazily).
        import importlib.util

        spec = importlib.util.find_spec("nvidia.nccl") if importlib.util.find_spec("nvidia") else None
        if spec and spec.submodule_search_locations:
            cand = os.path.join(list(spec.submodule_search_locations)[0], "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["SPB_NCCL_LIB"] = cand
    lib = C.CDLL(path)
    i, ip, vp, f, fp, u64 = C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_float, C.POINTER(C.c_float), C.c_uint64
    sig = {
        "spb_last_error": (C.c_char_p, [vp]),
        "spb_suffix_layers": (i, [i, i, i, ip]),
        "spb_chunk_coverage": (i, [i, i, ip]),
        "spb_chunk_layout": (i, [i, i, ip]),
        "spb_layer_chunks": (i, [i, i, ip]),
        "spb_draw_batch": (i, [u64, i, i, i, i, ip]),
        "spb_rank_workers": (i, [i, i, i, i, ip, ip]),
        "spb_create": (i, [ip, i, i, i, i, C.POINTER(vp)]),
        "spb_destroy": (i, [vp]),
        "spb_set_dataset": (i, [vp, fp, fp, i]),
        "spb_set_params": (i, [vp, vp]),
        "spb_get_params": (i, [vp, vp]),
        "spb_set_optimizer": (i, [vp, f, f, f]),
        "spb_partial_backprop": (i, [vp, ip, i, i, vp, C.POINTER(C.c_longlong), ip]),
        "spb_aggregate": (i, [vp, i, i, vp, ip, ip, vp]),
        "spb_aggregate64": (i, [i, i, i, vp, ip, ip, vp]),
        "spb_layer_shard": (i, [C.c_longlong, i, C.POINTER(C.c_longlong)]),
        "spb_set_gemm_chunk": (i, [i, i]),
        "spb_loss64": (i, [vp, vp, ip, i, C.POINTER(C.c_double)]),
        "spb_train_steps": (i, [vp, u64, i, i, i, fp]),
        "spb_step_host": (i, [vp, fp, fp, i, fp]),
        "spb_loss": (i, [vp, C.POINTER(C.c_double)]),
        "spb_synchronize": (i, [vp]),
        "spb_stream": (vp, [vp]),
        "spb_comm_unique_id": (i, [vp]),
        "spb_comm_init": (i, [vp, vp, i, i]),
        "spb_last_batch": (i, [vp, ip, i]),
        "spb_launches_per_step": (i, [vp, ip]),
        "spb_make_random_chain_mlp": (i, [ip, i, i, u64, fp, fp, vp]),
        "spb_get_grads": (i, [vp, vp]),
        "spb_profile_step": (i, [vp, u64, i, i, i, fp, C.POINTER(C.c_double), ip, fp]),
        "spb_time_train_steps": (i, [vp, u64, i, i, i, fp]),
        "spb_bucket_plan": (i, [i, i, i, i, ip, ip, ip]),
        "spb_set_fused_update": (i, [vp, i]),
        "spb_set_chain": (i, [vp, i]),
        "spb_step_host_async": (i, [vp, fp, fp, i, fp]),
        "spb_trace_steps": (i, [vp, u64, i, i, i, i, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), ip, ip, ip,
                                ip]),
        "spb_comm_mode": (i, [vp, ip]),
        "spb_profile_task": (i, [vp, i, i, i, fp, fp, C.POINTER(C.c_double)]),
        "spb_empirical_variance": (i, [vp, i, i, i, u64, C.POINTER(C.c_double)]),
        "spb_create_conv": (i, [ip, i, i, i, i, i, C.POINTER(vp)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


EXPORTED = [
    "spb_last_error", "spb_suffix_layers", "spb_chunk_coverage", "spb_chunk_layout", "spb_layer_chunks",
    "spb_draw_batch", "spb_rank_workers", "spb_create", "spb_destroy", "spb_set_dataset", "spb_set_params",
    "spb_get_params", "spb_set_optimizer", "spb_partial_backprop", "spb_aggregate", "spb_aggregate64", "spb_loss64", "spb_layer_shard", "spb_set_gemm_chunk", "spb_train_steps",
    "spb_step_host", "spb_loss", "spb_synchronize", "spb_stream", "spb_comm_unique_id", "spb_comm_init",
    "spb_last_batch", "spb_launches_per_step", "spb_make_random_chain_mlp",
    "spb_get_grads", "spb_profile_step", "spb_time_train_steps", "spb_bucket_plan", "spb_set_fused_update",
    "spb_set_chain", "spb_trace_steps", "spb_step_host_async",
    "spb_comm_mode", "spb_profile_task",
    "spb_empirical_variance", "spb_create_conv",
]

PROFILE_CLASSES = ["gemm_fwd", "gemm_wgrad", "gemm_dgrad", "head", "colreduce", "update", "gather", "comm"]


def _check(st: int, ctx=None):
    if st != 0:
        msg = load_library().spb_last_error(ctx).decode()
        raise _STATUS.get(st, SpbError)(msg)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ptrs(blocks: Sequence[Optional[np.ndarray]]):
    arr = (C.POINTER(C.c_float) * max(1, len(blocks)))()
    for i, b in enumerate(blocks):
        arr[i] = _fp(b) if b is not None else C.POINTER(C.c_float)()
    return C.cast(arr, C.c_void_p), arr


# ---- bookkeeping (spb.hpp:39-49) -------------------------------------------

def suffix_layers(j: int, k: int, L: int) -> int:
    out = C.c_int()
    _check(load_library().spb_suffix_layers(j, k, L, C.byref(out)))
    return out.value


def chunk_coverage(m: int, k: int) -> List[int]:
    out = np.zeros(max(m, 1), dtype=np.int32)
    _check(load_library().spb_chunk_coverage(m, k, _ip(out)))
    return out[:m].tolist()


def chunk_layout(k: int, L: int):
    out = np.zeros(2 * max(k, 1), dtype=np.int32)
    _check(load_library().spb_chunk_layout(k, L, _ip(out)))
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(k)]


def layer_chunks(k: int, L: int) -> List[int]:
    out = np.zeros(max(L, 1), dtype=np.int32)
    _check(load_library().spb_layer_chunks(k, L, _ip(out)))
    return out[:L].tolist()


def draw_batch(seed: int, step: int, worker: int, count: int, dataset_size: int) -> np.ndarray:
    """Rng(seed).split(step).split(worker) draws (spb.cpp:127-131,141,187)."""
    out = np.zeros(max(count, 1), dtype=np.int32)
    _check(load_library().spb_draw_batch(seed, step, worker, count, dataset_size, _ip(out)))
    return out[:count]


def rank_workers(k: int, L: int, rank: int, nranks: int) -> List[int]:
    out = np.zeros(k, dtype=np.int32)
    n = C.c_int()
    _check(load_library().spb_rank_workers(k, L, rank, nranks, _ip(out), C.byref(n)))
    return out[: n.value].tolist()


def bucket_plan(k: int, L: int, nranks: int, full_backprop: bool = False):
    """Per layer (index l-1): (kind, root, contributing ranks) of the
    multi-GPU gradient protocol; kind 0 = all-reduce, 1 = broadcast."""
    kind = np.zeros(L, dtype=np.int32)
    root = np.zeros(L, dtype=np.int32)
    mask = np.zeros(L, dtype=np.int32)
    _check(load_library().spb_bucket_plan(k, L, nranks, int(full_backprop), _ip(kind), _ip(root), _ip(mask)))
    return [(int(kind[l]), int(root[l]), [r for r in range(nranks) if (int(mask[l]) >> r) & 1]) for l in range(L)]


def layer_shard(count: int, parts: int) -> int:
    """The sub exchange mode's shard length (spb_layer_shard)."""
    out = C.c_longlong()
    _check(load_library().spb_layer_shard(count, parts, C.byref(out)))
    return out.value


def comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(load_library().spb_comm_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def block_dims(widths: Sequence[int]) -> List[int]:
    return [widths[l + 1] * widths[l] + widths[l + 1] for l in range(len(widths) - 1)]


# ---- reference data types (spb.hpp:20-36, model.hpp:15-19) -----------------

@dataclass
class SpbConfig:
    k: int = 1
    B: int = 1
    P: float = 0.0
    lr_base: float = 0.0
    R: float = 0.0
    V: float = 0.0

    def validate(self):  # spb.cpp:11-14
        if self.k < 1:
            raise ArgumentError("SpbConfig: k must be >= 1")
        if self.B < 1 or self.B % self.k != 0:
            raise ArgumentError("SpbConfig: B must be positive and divisible by k")


@dataclass
class PartialGradient:
    blocks: List[np.ndarray]  # size L; absent blocks are empty
    covered_from: int = 1

    def covers(self, layer_1based: int) -> bool:
        return layer_1based >= self.covered_from


@dataclass
class BackpropStats:
    layer_ops: List[int] = field(default_factory=list)


class StepSchedule(Enum):
    Theorem1 = 0
    Constant = 1


@dataclass
class VarianceEstimate:  # spb.hpp:91-98
    spb: float = 0.0  # E || grad f - g_spb ||^2
    spb_se: float = 0.0
    baseline: float = 0.0  # same, with every worker computing the full gradient
    baseline_se: float = 0.0
    p_hat: List[float] = field(default_factory=list)  # per-chunk single-sample variances p_i
    p_se: List[float] = field(default_factory=list)


@dataclass
class SgdResult:
    avg_loss: List[float] = field(default_factory=list)
    step_size: List[float] = field(default_factory=list)
    avg_subopt: List[float] = field(default_factory=list)
    avg_iterate: List[np.ndarray] = field(default_factory=list)
    iterates: List[List[np.ndarray]] = field(default_factory=list)


# ---- the model ("layer" API, model.hpp:26-60,95-111) -------------------------

class ChainMlp:
    """ChainMlp on one B200: h_l = tanh(W_l h_{l-1} + b_l), affine head,
    per-sample loss 0.5*||out - y||^2 (model.hpp:91-111).

    k / per_worker_batch size the device workspace for SPB steps."""

    kind = "ChainMlp"

    def __init__(self, widths: Sequence[int], inputs, targets, weights, k: int = 1, per_worker_batch: int = 1,
                 device: int = 0):
        lib = load_library()
        self.widths = [int(w) for w in widths]
        if len(self.widths) < 2:
            raise ArgumentError("mlp: need at least one layer")
        X = np.ascontiguousarray(inputs, dtype=np.float32).reshape(len(inputs), -1)
        Y = np.ascontiguousarray(targets, dtype=np.float32).reshape(len(targets), -1)
        if X.shape[0] == 0 or X.shape[0] != Y.shape[0]:
            raise ArgumentError("mlp: dataset shape mismatch")
        self._dims = block_dims(self.widths)
        if len(weights) != len(self._dims) or any(np.size(wb) != d for wb, d in zip(weights, self._dims)):
            raise ArgumentError("mlp: weight block size mismatch")
        w = np.asarray(self.widths, dtype=np.int32)
        ctx = C.c_void_p()
        _check(lib.spb_create(_ip(w), len(self.widths), k, per_worker_batch, device, C.byref(ctx)))
        self._ctx = ctx
        self.k, self.per_worker_batch = k, per_worker_batch
        _check(lib.spb_set_dataset(ctx, _fp(X), _fp(Y), X.shape[0]), ctx)
        self._N = X.shape[0]
        self._initial = [np.asarray(b, dtype=np.float32).copy() for b in weights]
        self.set_params(self._initial)

    def close(self):
        """Releases the device state (and the NCCL communicator, if any)."""
        ctx = getattr(self, "_ctx", None)
        if ctx is not None and _lib is not None:
            _lib.spb_destroy(ctx)
        self._ctx = None

    def __del__(self):
        self.close()

    # LayeredModel accessors (model.hpp:32-36)
    def layer_count(self) -> int:
        return len(self._dims)

    def block_dims(self) -> List[int]:
        return list(self._dims)

    def dataset_size(self) -> int:
        return self._N

    def initial_params(self) -> List[np.ndarray]:
        return [b.copy() for b in self._initial]

    def set_initial_params(self, x):
        self._initial = [np.asarray(b, dtype=np.float32).copy() for b in x]

    def zeros_like(self) -> List[np.ndarray]:
        return [np.zeros(d, dtype=np.float32) for d in self._dims]

    @property
    def ctx(self):
        return self._ctx

    def set_params(self, x):
        blocks = [np.ascontiguousarray(b, dtype=np.float32) for b in x]
        p, _keep = _ptrs(blocks)
        _check(load_library().spb_set_params(self._ctx, p), self._ctx)

    def get_params(self) -> List[np.ndarray]:
        out = self.zeros_like()
        p, _keep = _ptrs(out)
        _check(load_library().spb_get_params(self._ctx, p), self._ctx)
        return out

    def get_grads(self) -> List[np.ndarray]:
        """The aggregated gradient of the last step (or last partial_backprop)."""
        out = self.zeros_like()
        p, _keep = _ptrs(out)
        _check(load_library().spb_get_grads(self._ctx, p), self._ctx)
        return out

    def set_fused_update(self, fused):
        """Single-GPU optimizer placement: False / 0 per-layer update kernels
        (gradients readable with get_grads), True / 1 inside every wgrad
        epilogue, 2 (the default) inside the cheap (<= 512-row) wgrads only."""
        _check(load_library().spb_set_fused_update(self._ctx, int(fused)), self._ctx)

    def set_chain(self, steps: int):
        """Steps captured per CUDA graph by train_steps (1..16): step t+1's
        forward of layer l waits only for W_l of step t, so the exchange /
        update tail of a step overlaps the next forward. Same results."""
        _check(load_library().spb_set_chain(self._ctx, int(steps)), self._ctx)

    def trace_steps(self, seed: int, step0: int, steps: int, full_backprop: bool = False) -> dict:
        """Per-op timeline of `steps` chained iterations replayed from one
        graph (spb_trace_steps): arrays t0 / t1 (ns, relative), cls, stream,
        sub. Advances the parameters by 2 * steps iterations."""
        cap = 1 << 15
        tb = np.zeros(cap, np.int64)
        te = np.zeros(cap, np.int64)
        cl, stv, sb = (np.zeros(cap, np.int32) for _ in range(3))
        n = C.c_int(0)
        lib = load_library()
        lp = C.POINTER(C.c_longlong)
        _check(lib.spb_trace_steps(self._ctx, seed, step0, steps, int(full_backprop), cap, tb.ctypes.data_as(lp),
                                   te.ctypes.data_as(lp), _ip(cl), _ip(stv), _ip(sb), C.byref(n)), self._ctx)
        k = min(n.value, cap)
        t0 = tb[:k].min() if k else 0
        return {"t0": tb[:k] - t0, "t1": te[:k] - t0, "cls": cl[:k], "stream": stv[:k], "sub": sb[:k]}

    def set_optimizer(self, lr: float, momentum: float = 0.0, weight_decay: float = 0.0):
        _check(load_library().spb_set_optimizer(self._ctx, lr, momentum, weight_decay), self._ctx)

    def loss(self, x=None) -> float:
        """ChainMlp::loss (model.cpp:139-143) at x (default: current params)."""
        if x is not None:
            self.set_params(x)
        out = C.c_double()
        _check(load_library().spb_loss(self._ctx, C.byref(out)), self._ctx)
        return out.value

    def train_steps(self, seed: int, step0: int, steps: int, full_backprop: bool = False, losses: bool = False):
        buf = np.zeros(max(steps, 1), dtype=np.float32) if losses else None
        _check(load_library().spb_train_steps(self._ctx, seed, step0, steps, int(full_backprop),
                                              _fp(buf) if buf is not None else None), self._ctx)
        return buf[:steps] if buf is not None else None

    def _check_host_rows(self, X_rows, Y_rows):
        """The C side copies hosted_rows * n_0 and hosted_rows * n_L floats
        straight from these pointers (possibly later, on a copy stream): the
        arrays must be exactly that, float32 and C-contiguous. No silent
        conversion -- a temporary copy could be freed before an asynchronous
        copy reads it."""
        rows = self.hosted_workers * self.per_worker_batch
        for name, a, cols in (("X_rows", X_rows, self._row_width()), ("Y_rows", Y_rows, self.widths[-1])):
            if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous:
                raise ArgumentError(f"{name}: need a C-contiguous float32 numpy array")
            if a.size != rows * cols or (a.ndim == 2 and a.shape != (rows, cols)):
                raise ArgumentError(f"{name}: need shape ({rows}, {cols}), got {a.shape}")

    def _row_width(self) -> int:
        return self.widths[0]

    @property
    def hosted_workers(self) -> int:
        """Workers whose rows this rank's steps consume (all k on one GPU)."""
        return getattr(self, "_hosted", self.k)

    def step_host(self, X_rows: np.ndarray, Y_rows: np.ndarray, full_backprop: bool = False) -> float:
        self._check_host_rows(X_rows, Y_rows)
        loss = np.zeros(1, dtype=np.float32)
        _check(load_library().spb_step_host(self._ctx, _fp(X_rows), _fp(Y_rows), int(full_backprop), _fp(loss)),
               self._ctx)
        return float(loss[0])

    def step_host_async(self, X_rows: np.ndarray, Y_rows: np.ndarray, loss_out: np.ndarray, full_backprop: bool = False):
        """spb_step_host_async: enqueue one step on host rows (pinned for an
        asynchronous copy); loss_out (float32, >= 1 element) receives the
        loss. The arrays must stay alive and unchanged until synchronize()."""
        self._check_host_rows(X_rows, Y_rows)
        if not isinstance(loss_out, np.ndarray) or loss_out.dtype != np.float32 or loss_out.size < 1:
            raise ArgumentError("loss_out: need a float32 numpy array with >= 1 element")
        _check(load_library().spb_step_host_async(self._ctx, _fp(X_rows), _fp(Y_rows), int(full_backprop),
                                                  _fp(loss_out)), self._ctx)

    def profile_step(self, seed: int, step: int, full_backprop: bool = False):
        """One eager step with per-class CUDA-event timings (see spb_profile_step)."""
        n = len(PROFILE_CLASSES)
        ms = np.zeros(n, dtype=np.float32)
        work = np.zeros(n, dtype=np.float64)
        launches = np.zeros(n, dtype=np.int32)
        step_ms = np.zeros(1, dtype=np.float32)
        _check(load_library().spb_profile_step(self._ctx, seed, step, int(full_backprop), n, _fp(ms),
                                               work.ctypes.data_as(C.POINTER(C.c_double)), _ip(launches),
                                               _fp(step_ms)), self._ctx)
        return {c: dict(ms=float(ms[i]), work=float(work[i]), launches=int(launches[i]))
                for i, c in enumerate(PROFILE_CLASSES)}, float(step_ms[0])

    def time_train_steps(self, seed: int, step0: int, steps: int, full_backprop: bool = False) -> float:
        ms = np.zeros(1, dtype=np.float32)
        _check(load_library().spb_time_train_steps(self._ctx, seed, step0, steps, int(full_backprop), _fp(ms)),
               self._ctx)
        return float(ms[0])

    def comm_init(self, unique_id: bytes, rank: int, nranks: int):
        """Joins the NCCL clique; the context then runs only this rank's workers."""
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(load_library().spb_comm_init(self._ctx, C.cast(buf, C.c_void_p), rank, nranks), self._ctx)
        self.rank, self.nranks = rank, nranks
        self._hosted = len(rank_workers(self.k, self.layer_count(), rank, nranks))

    def comm_init_torch(self, dist, rank: int, nranks: int):
        """Rendezvous through an initialised torch.distributed group (plumbing only)."""
        obj = [comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.comm_init(obj[0], rank, nranks)

    @property
    def comm_mode(self):
        """Multi-GPU aggregation mode: "rh", "push", "p2p", "sub" (None before comm_init; "local" for one rank)."""
        v = C.c_int()
        _check(load_library().spb_comm_mode(self._ctx, C.byref(v)), self._ctx)
        return {0: "local", 2: "p2p", 3: "sub", 4: "push", 5: "rh"}.get(v.value)

    def profile_task(self, rows: int, suffix: int, reps: int = 10):
        """(forward_ms, backward_ms, peak_mem_gb) of one worker task that
        backpropagates the top `suffix` layers of a `rows`-sample batch."""
        f = np.zeros(1, dtype=np.float32)
        b = np.zeros(1, dtype=np.float32)
        mem = C.c_double()
        _check(load_library().spb_profile_task(self._ctx, rows, suffix, reps, _fp(f), _fp(b), C.byref(mem)), self._ctx)
        return float(f[0]), float(b[0]), float(mem.value)

    def last_batch(self, rows: int) -> np.ndarray:
        out = np.zeros(rows, dtype=np.int32)
        _check(load_library().spb_last_batch(self._ctx, _ip(out), rows), self._ctx)
        return out

    def launches_per_step(self) -> int:
        n = C.c_int()
        _check(load_library().spb_launches_per_step(self._ctx, C.byref(n)), self._ctx)
        return n.value

    def synchronize(self):
        _check(load_library().spb_synchronize(self._ctx), self._ctx)

    def stream_handle(self) -> int:
        return int(load_library().spb_stream(self._ctx) or 0)


def make_random_chain_mlp(widths: Sequence[int], samples: int, seed: int, **kw) -> ChainMlp:
    """make_random_chain_mlp (model.cpp:208-231) data, rounded to fp32, on the GPU.

    The generator is the reference's counter-based stream Rng(seed).split(0x313a)
    (weights U(-1/sqrt(n_in), 1/sqrt(n_in)), inputs N(0,1), targets
    tanh(sum x) + 0.1 N(0,1)), evaluated by the C++ host generator."""
    X, Y, blocks = gen_chain_mlp(widths, samples, seed)
    return ChainMlp(widths, X, Y, blocks, **kw)


class ConvNet(ChainMlp):
    """CIFAR10-shaped convolutional SPB model on one B200 (SURVEY.md 8f-1,
    BASELINE configs[3]): 3x3 convolutions (padding 1, stride 1 or 2) with
    tanh, lowered to the tcgen05 GEMMs by im2col; global average pool; affine
    head; per-sample loss 0.5 ||out - y||^2. The reference has no conv model:
    this mirrors its LayeredModel interface (layer_count, block_dims,
    partial_backprop, loss) and its SPB rules apply unchanged.

    in_shape = (h, w, c); convs = [(c_out, stride), ...]; samples are NHWC
    images; block l = W_l [c_out x 9 c_in] (columns (ky*3+kx)*c_in + ci), b_l."""

    kind = "ConvNet"

    def __init__(self, in_shape, convs, nout: int, inputs, targets, weights, k: int = 1, per_worker_batch: int = 1,
                 device: int = 0):
        lib = load_library()
        self.in_shape = tuple(int(v) for v in in_shape)
        self.convs = [(int(c), int(st)) for c, st in convs]
        self.nout = int(nout)
        self._dims = convnet_block_dims(self.in_shape, self.convs, self.nout)
        h, w, c = self.in_shape
        X = np.ascontiguousarray(inputs, dtype=np.float32).reshape(len(inputs), -1)
        Y = np.ascontiguousarray(targets, dtype=np.float32).reshape(len(targets), -1)
        if X.shape[0] == 0 or X.shape[0] != Y.shape[0] or X.shape[1] != h * w * c or Y.shape[1] != self.nout:
            raise ArgumentError("convnet: dataset shape mismatch")
        if len(weights) != len(self._dims) or any(np.size(wb) != d for wb, d in zip(weights, self._dims)):
            raise ArgumentError("convnet: weight block size mismatch")
        geom = np.asarray([h, w, c] + [v for cs in self.convs for v in cs], dtype=np.int32)
        ctx = C.c_void_p()
        _check(lib.spb_create_conv(_ip(geom), len(self.convs), self.nout, k, per_worker_batch, device, C.byref(ctx)))
        self._ctx = ctx
        self.widths = [c] + [cs[0] for cs in self.convs] + [self.nout]
        self.k, self.per_worker_batch = k, per_worker_batch
        _check(lib.spb_set_dataset(ctx, _fp(X), _fp(Y), X.shape[0]), ctx)
        self._N = X.shape[0]
        self._initial = [np.asarray(b, dtype=np.float32).copy() for b in weights]
        self.set_params(self._initial)

    def _row_width(self) -> int:
        h, w, c = self.in_shape
        return h * w * c


def convnet_block_dims(in_shape, convs, nout: int) -> List[int]:
    c = in_shape[2]
    dims = []
    for co, _ in convs:
        dims.append(co * 9 * c + co)
        c = co
    dims.append(nout * c + nout)
    return dims


def gen_convnet(in_shape, convs, nout: int, samples: int, seed: int):
    """Synthetic CIFAR-shaped data and a random init (numpy, deterministic):
    images uniform in [-1, 1), targets uniform in [-1, 1), weights
    N(0, 1/fan_in), biases 0.01 N(0, 1). Returns X [samples, h*w*c], Y, blocks."""
    rng = np.random.default_rng(seed)
    h, w, c = in_shape
    X = rng.uniform(-1, 1, size=(samples, h * w * c)).astype(np.float32)
    Y = rng.uniform(-1, 1, size=(samples, nout)).astype(np.float32)
    blocks = []
    cin = c
    for co, _ in convs:
        Wl = rng.standard_normal((co, 9 * cin)) / np.sqrt(9 * cin)
        blocks.append(np.concatenate([Wl.ravel(), 0.01 * rng.standard_normal(co)]).astype(np.float32))
        cin = co
    Wl = rng.standard_normal((nout, cin)) / np.sqrt(cin)
    blocks.append(np.concatenate([Wl.ravel(), 0.01 * rng.standard_normal(nout)]).astype(np.float32))
    return X, Y, blocks


def gen_chain_mlp(widths: Sequence[int], samples: int, seed: int):
    """fp32 (X [samples x n_0], Y [samples x n_L], weight blocks) of
    make_random_chain_mlp(widths, samples, seed) (model.cpp:208-231)."""
    w = np.asarray(widths, dtype=np.int32)
    X = np.zeros((samples, widths[0]), dtype=np.float32)
    Y = np.zeros((samples, widths[-1]), dtype=np.float32)
    blocks = [np.zeros(d, dtype=np.float32) for d in block_dims(widths)]
    p, _keep = _ptrs(blocks)
    _check(load_library().spb_make_random_chain_mlp(_ip(w), len(widths), samples, seed, _fp(X), _fp(Y), p))
    return X, Y, blocks


# ---- worker and aggregator (spb.hpp:54-61) -----------------------------------

def partial_backprop(model: ChainMlp, x, batch, suffix: int, stats: Optional[BackpropStats] = None) -> PartialGradient:
    """spb.cpp:51-68 on the GPU: the batch-mean gradient of the last `suffix` layers."""
    L = model.layer_count()
    if x is not None:
        model.set_params(x)
    b = np.ascontiguousarray(batch, dtype=np.int32)
    out = model.zeros_like()
    p, _keep = _ptrs(out)
    ops = None
    if stats is not None:
        if not stats.layer_ops:
            stats.layer_ops = [0] * L
        ops = np.asarray(stats.layer_ops, dtype=np.int64)
    cov = C.c_int()
    _check(load_library().spb_partial_backprop(model.ctx, _ip(b) if b.size else None, int(b.size), suffix, p,
                                               ops.ctypes.data_as(C.POINTER(C.c_longlong)) if ops is not None else None,
                                               C.byref(cov)), model.ctx)
    if stats is not None:
        stats.layer_ops = [int(v) for v in ops]
    blocks = [o if l + 1 >= cov.value else np.zeros(0, dtype=np.float32) for l, o in enumerate(out)]
    return PartialGradient(blocks, cov.value)


_agg_model = None


def _aggregator_ctx():
    global _agg_model
    if _agg_model is None:
        w = np.asarray([1, 1], dtype=np.int32)
        ctx = C.c_void_p()
        _check(load_library().spb_create(_ip(w), 2, 1, 1, 0, C.byref(ctx)))
        _agg_model = ctx
    return _agg_model


def aggregate(grads: Sequence[PartialGradient], k: int) -> List[np.ndarray]:
    """spb.cpp:70-106: per layer, the mean over its contributing workers (GPU)."""
    if k < 1 or len(grads) != k:
        raise ArgumentError("aggregate: need exactly k gradients")
    L = len(grads[0].blocks)
    for g in grads:
        if len(g.blocks) != L:
            raise ProtocolError("aggregate: gradient layer counts differ")
    flat, dims = [], np.zeros(k * L, dtype=np.int32)
    for j, g in enumerate(grads):
        for l in range(L):
            b = g.blocks[l]
            b = None if b is None or np.size(b) == 0 else np.ascontiguousarray(b, dtype=np.float32)
            flat.append(b)
            dims[j * L + l] = 0 if b is None else b.size
    cov = np.asarray([g.covered_from for g in grads], dtype=np.int32)
    sizes = [max(int(dims[j * L + l]) for j in range(k)) for l in range(L)]
    out = [np.zeros(max(s, 1), dtype=np.float32) for s in sizes]
    pin, _k1 = _ptrs(flat)
    pout, _k2 = _ptrs(out)
    ctx = _aggregator_ctx()
    _check(load_library().spb_aggregate(ctx, k, L, pin, _ip(dims), _ip(cov), pout), ctx)
    return [o[:s] for o, s in zip(out, sizes)]


def empirical_variance(model: ChainMlp, cfg: SpbConfig, x, trials: int, seed: int) -> VarianceEstimate:
    """empirical_variance (spb.cpp:212-265) on the GPU, with the reference's
    sampling protocol (kWorkerDrawTag / kChunkDrawTag streams) sample for
    sample. The model's workspace must match (cfg.k, cfg.B)."""
    cfg.validate()
    if trials < 1:
        raise ArgumentError("empirical_variance: trials must be >= 1")
    if x is not None:
        model.set_params(x)
    out = np.zeros(4 + 2 * cfg.k, dtype=np.float64)
    _check(load_library().spb_empirical_variance(model.ctx, cfg.k, cfg.B, trials, seed,
                                                 out.ctypes.data_as(C.POINTER(C.c_double))), model.ctx)
    k = cfg.k
    return VarianceEstimate(float(out[0]), float(out[1]), float(out[2]), float(out[3]),
                            [float(v) for v in out[4:4 + k]], [float(v) for v in out[4 + k:4 + 2 * k]])


def spb_sgd_run(model: ChainMlp, cfg: SpbConfig, iterations: int, schedule: StepSchedule, seed: int,
                record_iterates: bool = False) -> SgdResult:
    """spb_sgd_run (spb.cpp:164-210) with each iteration one device-resident
    SPB step (spb_train_steps). The Theorem1 schedule needs a convex model,
    which a ChainMlp is not (spb.cpp:169-171)."""
    cfg.validate()
    if iterations < 1:
        raise ArgumentError("spb_sgd_run: iterations must be >= 1")
    if schedule == StepSchedule.Theorem1:
        raise ConfigError("Theorem1 schedule requires the convex model")
    if cfg.k != model.k or cfg.B // cfg.k != model.per_worker_batch:
        raise ArgumentError("spb_sgd_run: model workspace was created for a different (k, B)")
    x = model.initial_params()
    model.set_params(x)
    model.set_optimizer(cfg.lr_base)
    xbar = [np.zeros_like(b, dtype=np.float64) for b in x]
    res = SgdResult()
    for s in range(1, iterations + 1):
        model.train_steps(seed, s, 1)
        xs = model.get_params()
        for l in range(len(xbar)):  # spb.cpp:199-200
            xbar[l] += (xs[l] - xbar[l]) / s
        res.step_size.append(cfg.lr_base)
        if record_iterates:
            res.iterates.append(xs)
        # avg_loss f(xbar_s) (spb.cpp:202): evaluated at xbar, then restore x.
        res.avg_loss.append(model.loss([b.astype(np.float32) for b in xbar]))
        model.set_params(xs)
    res.avg_iterate = [b.astype(np.float32) for b in xbar]
    return res
