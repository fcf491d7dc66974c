"""TEST INFRASTRUCTURE ONLY -- ctypes front-end to the CPU checkers.

* ``Oracle``: the C restatement oracle/spb_oracle.c (liboracle.so), built
  from this repo anywhere gcc exists.
* ``Ref``: the unmodified reference SPB core, oracle/_ref/libjigsaw_ref.so,
  compiled from /root/reference by oracle/Makefile (this container only; the
  built .so travels to the GPU box).

Both expose the same methods, named after the reference API
(/root/reference/proj/include/jigsaw/spb/spb.hpp:39-83). Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs import this module: it is the
checker, never the product, and nothing under paper_2111_10672_b200/ uses it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libjigsaw_ref.so")

ST_OK, ST_ARGUMENT, ST_PROTOCOL, ST_CONFIG = 0, 1, 2, 3


class OracleError(Exception):
    def __init__(self, status: int, what: str = ""):
        super().__init__(f"status {status}: {what}")
        self.status = status


def build(ref: bool = False) -> None:
    """Builds liboracle.so (and, when /root/reference exists and ref=True, _ref)."""
    targets = ["liboracle.so"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _ptr_array(blocks: Sequence[Optional[np.ndarray]]):
    arr = (C.POINTER(C.c_double) * len(blocks))()
    for i, b in enumerate(blocks):
        arr[i] = _dp(b) if b is not None else C.POINTER(C.c_double)()
    return arr


def block_dims(widths: Sequence[int]) -> List[int]:
    """model.cpp:99 -- block l = W_l row-major then b_l."""
    return [widths[l + 1] * widths[l] + widths[l + 1] for l in range(len(widths) - 1)]


class _Common:
    lib: C.CDLL
    prefix: str

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, st: int, what: str = ""):
        if st != ST_OK:
            raise OracleError(st, what)

    # ---- bookkeeping (spb.cpp:16-49) ----
    def suffix_layers(self, j: int, k: int, L: int) -> int:
        out = C.c_int()
        self._check(self._f("suffix_layers")(j, k, L, C.byref(out)), "suffix_layers")
        return out.value

    def chunk_coverage(self, m: int, k: int) -> List[int]:
        out = np.zeros(max(m, 1), dtype=np.int32)
        self._check(self._f("chunk_coverage")(m, k, _ip(out)), "chunk_coverage")
        return out[:m].tolist()

    def chunk_layout(self, k: int, L: int):
        out = np.zeros(2 * max(k, 1), dtype=np.int32)
        self._check(self._f("chunk_layout")(k, L, _ip(out)), "chunk_layout")
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(k)]

    def layer_chunks(self, k: int, L: int) -> List[int]:
        out = np.zeros(max(L, 1), dtype=np.int32)
        self._check(self._f("layer_chunks")(k, L, _ip(out)), "layer_chunks")
        return out[:L].tolist()

    def rng_stream(self, key: int, tags: Sequence[int], kind: int, n: int, bound: int = 0) -> np.ndarray:
        t = np.asarray(tags, dtype=np.uint64)
        out = np.zeros(n, dtype=np.uint64)
        self._f("rng_stream")(C.c_uint64(key), t.ctypes.data_as(C.POINTER(C.c_uint64)), len(t), kind,
                              C.c_uint64(bound), n, out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out


class Oracle(_Common):
    """The C restatement (spb_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_mix.restype = C.c_uint64
        L.orc_mix.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_loss.restype = C.c_double
        L.orc_spb_step.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                   C.c_int]
        L.orc_sgd_momentum.argtypes = [C.c_long, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.c_double, C.c_double, C.c_double, C.c_int]
        L.orc_gen_chain_mlp.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_uint64,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]
        L.orc_draw_batch.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]

    def mix(self, a: int, b: int) -> int:
        return int(self.lib.orc_mix(a, b))

    def draw_batch(self, seed: int, step: int, worker: int, count: int, n: int) -> np.ndarray:
        out = np.zeros(count, dtype=np.int32)
        self.lib.orc_draw_batch(seed, step, worker, count, n, _ip(out))
        return out

    def gen_chain_mlp(self, widths: Sequence[int], samples: int, seed: int):
        """make_random_chain_mlp (model.cpp:208-231): returns X, Y, blocks (fp64)."""
        w = np.asarray(widths, dtype=np.int32)
        X = np.zeros((samples, widths[0]), dtype=np.float64)
        Y = np.zeros((samples, widths[-1]), dtype=np.float64)
        blocks = [np.zeros(d, dtype=np.float64) for d in block_dims(widths)]
        self.lib.orc_gen_chain_mlp(_ip(w), len(widths), samples, seed, _dp(X), _dp(Y), _ptr_array(blocks))
        return X, Y, blocks

    def loss(self, widths, X, Y, params) -> float:
        w = np.asarray(widths, dtype=np.int32)
        return float(self.lib.orc_loss(_ip(w), len(widths) - 1, _ptr_array(params), _dp(X), _dp(Y), X.shape[0]))

    def partial_backprop(self, widths, X, Y, params, batch, suffix: int, layer_ops=None):
        """spb.cpp:51-68. Returns (blocks with None for absent layers, covered_from)."""
        L = len(widths) - 1
        w = np.asarray(widths, dtype=np.int32)
        b = np.ascontiguousarray(batch, dtype=np.int32)
        dims = block_dims(widths)
        out = [np.zeros(d, dtype=np.float64) for d in dims]
        cov = C.c_int()
        ops_ptr = None
        if layer_ops is not None:
            ops_ptr = layer_ops.ctypes.data_as(C.POINTER(C.c_longlong))
        st = self.lib.orc_partial_backprop(_ip(w), L, _dp(X), _dp(Y), X.shape[0], _ptr_array(params), _ip(b),
                                           len(b), suffix, _ptr_array(out), ops_ptr, C.byref(cov))
        self._check(st, "partial_backprop")
        return [o if l + 1 >= cov.value else None for l, o in enumerate(out)], cov.value

    def aggregate(self, grads: Sequence[Sequence[Optional[np.ndarray]]], covered_from: Sequence[int], k: int):
        """spb.cpp:70-106."""
        if k < 1 or len(grads) != k:
            raise OracleError(ST_ARGUMENT, "aggregate: need exactly k gradients")
        L = len(grads[0])
        flat, dims = [], np.zeros(k * L, dtype=np.int32)
        for j in range(k):
            if len(grads[j]) != L:
                raise OracleError(ST_PROTOCOL, "aggregate: gradient layer counts differ")
            for l in range(L):
                g = grads[j][l]
                flat.append(None if g is None or len(g) == 0 else np.ascontiguousarray(g, dtype=np.float64))
                dims[j * L + l] = 0 if flat[-1] is None else len(flat[-1])
        sizes = [max(int(dims[j * L + l]) for j in range(k)) for l in range(L)]
        out = [np.zeros(max(s, 1), dtype=np.float64) for s in sizes]
        cov = np.asarray(covered_from, dtype=np.int32)
        st = self.lib.orc_aggregate(k, L, _ptr_array(flat), _ip(dims), _ip(cov), _ptr_array(out))
        self._check(st, "aggregate")
        return [o[:s] for o, s in zip(out, sizes)]

    def spb_step(self, widths, X, Y, params, k: int, B: int, lr: float, seed: int, s: int, full: bool = False):
        """One SPB-SGD iteration (spb.cpp:187-196) updating params in place."""
        w = np.asarray(widths, dtype=np.int32)
        st = self.lib.orc_spb_step(_ip(w), len(widths) - 1, _dp(X), _dp(Y), X.shape[0],
                                   C.cast(_ptr_array(params), C.c_void_p), k, B, lr, seed, s, int(full))
        self._check(st, "spb_step")

    def sgd_momentum(self, w, g, buf, lr, momentum, weight_decay, first_step):
        self.lib.orc_sgd_momentum(w.size, _dp(w), _dp(g), _dp(buf), lr, momentum, weight_decay, int(first_step))


class Ref(_Common):
    """The reference's own SPB core (oracle/_ref/libjigsaw_ref.so)."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (build with `make -C oracle ref` where /root/reference exists)")
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_mix.restype = C.c_uint64
        L.ref_rng_mix.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_chain_random.restype = C.c_void_p
        L.ref_chain_random.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_uint64]
        L.ref_chain_new.restype = C.c_void_p
        L.ref_chain_new.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.c_int, C.c_void_p]
        L.ref_chain_free.argtypes = [C.c_void_p]
        for n in ("ref_layer_count", "ref_block_dim", "ref_get_params", "ref_set_params", "ref_loss",
                  "ref_partial_backprop", "ref_step", "ref_sgd_run", "ref_time_steps"):
            getattr(L, n).argtypes = None
        L.ref_layer_count.argtypes = [C.c_void_p]
        L.ref_block_dim.argtypes = [C.c_void_p, C.c_int]
        L.ref_get_params.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_set_params.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_loss.argtypes = [C.c_void_p, C.POINTER(C.c_double)]
        L.ref_partial_backprop.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_void_p,
                                           C.POINTER(C.c_longlong), C.POINTER(C.c_int)]
        L.ref_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_int]
        L.ref_sgd_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64,
                                  C.POINTER(C.c_double)]
        L.ref_time_steps.restype = C.c_double
        L.ref_time_steps.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                     C.c_int, C.c_int]
        L.ref_profile_query.argtypes = [C.c_char_p, C.c_char_p, C.c_double, C.POINTER(C.c_double)]
        for n in ("ref_empirical_variance", "ref_variance_oracle"):
            getattr(L, n).argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_double)]

    def _check(self, st: int, what: str = ""):
        if st != ST_OK:
            raise OracleError(st, what + ": " + self.lib.ref_last_error().decode())

    def mix(self, a: int, b: int) -> int:
        return int(self.lib.ref_rng_mix(a, b))

    def profile_query(self, csv_text: str, model: str, fraction: float) -> dict:
        """ProfileTable::from_csv + the interpolators (profile.cpp:67-171)."""
        out = np.zeros(7, dtype=np.float64)
        self._check(self.lib.ref_profile_query(csv_text.encode(), model.encode(), fraction, _dp(out)), "profile")
        keys = ("forward_ms", "backward_ms", "peak_mem_gb", "grad_size_mb", "batch", "duration_ms", "comm_mb")
        return dict(zip(keys, (float(v) for v in out)))


class RefModel:
    """A reference ChainMlp plus its current iterate (oracle/ref_capi.cpp Handle)."""

    def __init__(self, ref: Ref, widths, X=None, Y=None, params=None, samples=0, seed=0):
        self.ref, self.widths = ref, list(widths)
        w = np.asarray(widths, dtype=np.int32)
        if X is None:
            self.h = ref.lib.ref_chain_random(_ip(w), len(widths), samples, seed)
        else:
            self._X = np.ascontiguousarray(X, dtype=np.float64)
            self._Y = np.ascontiguousarray(Y, dtype=np.float64).reshape(-1)
            ps = [np.ascontiguousarray(p, dtype=np.float64) for p in params]
            self.h = ref.lib.ref_chain_new(_ip(w), len(widths), _dp(self._X), _dp(self._Y), self._X.shape[0],
                                           C.cast(_ptr_array(ps), C.c_void_p))
        if not self.h:
            raise OracleError(ST_ARGUMENT, ref.lib.ref_last_error().decode())
        self.L = len(widths) - 1
        self.dims = block_dims(widths)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_chain_free(self.h)
            self.h = None

    def get_params(self):
        out = [np.zeros(d, dtype=np.float64) for d in self.dims]
        self.ref.lib.ref_get_params(self.h, C.cast(_ptr_array(out), C.c_void_p))
        return out

    def set_params(self, params):
        ps = [np.ascontiguousarray(p, dtype=np.float64) for p in params]
        self.ref.lib.ref_set_params(self.h, C.cast(_ptr_array(ps), C.c_void_p))

    def loss(self) -> float:
        out = C.c_double()
        self.ref._check(self.ref.lib.ref_loss(self.h, C.byref(out)), "loss")
        return out.value

    def partial_backprop(self, batch, suffix: int, layer_ops=None):
        b = np.ascontiguousarray(batch, dtype=np.int32)
        out = [np.zeros(d, dtype=np.float64) for d in self.dims]
        cov = C.c_int()
        ops = layer_ops.ctypes.data_as(C.POINTER(C.c_longlong)) if layer_ops is not None else None
        st = self.ref.lib.ref_partial_backprop(self.h, _ip(b), len(b), suffix, C.cast(_ptr_array(out), C.c_void_p),
                                               ops, C.byref(cov))
        self.ref._check(st, "partial_backprop")
        return [o if l + 1 >= cov.value else None for l, o in enumerate(out)], cov.value

    def step(self, k: int, B: int, lr: float, seed: int, s: int, full: bool = False, threads: int = 1):
        self.ref._check(self.ref.lib.ref_step(self.h, k, B, lr, seed, s, int(full), threads), "step")

    def sgd_run(self, k: int, B: int, lr: float, iters: int, seed: int):
        avg = np.zeros(iters, dtype=np.float64)
        self.ref._check(self.ref.lib.ref_sgd_run(self.h, k, B, lr, iters, seed, _dp(avg)), "sgd_run")
        return avg

    def empirical_variance(self, k: int, B: int, trials: int, seed: int) -> dict:
        """empirical_variance (spb.cpp:212-265) at the current iterate."""
        out = np.zeros(4 + 2 * k, dtype=np.float64)
        self.ref._check(self.ref.lib.ref_empirical_variance(self.h, k, B, trials, seed, _dp(out)), "empirical_variance")
        return dict(spb=out[0], spb_se=out[1], baseline=out[2], baseline_se=out[3], p_hat=out[4:4 + k],
                    p_se=out[4 + k:])

    def variance_oracle(self, k: int, B: int, trials: int, seed: int) -> dict:
        """The reference's independent brute-force oracle (oracle.cpp:240-326)."""
        out = np.zeros(4 + 2 * k, dtype=np.float64)
        self.ref._check(self.ref.lib.ref_variance_oracle(self.h, k, B, trials, seed, _dp(out)), "variance_oracle")
        return dict(spb=out[0], spb_se=out[1], harmonic_sum=out[2], harmonic_sum_se=out[3], p_hat=out[4:4 + k],
                    p_se=out[4 + k:])

    def time_steps(self, k, B, lr, seed, s0, steps, full=False, threads=1) -> float:
        return float(self.ref.lib.ref_time_steps(self.h, k, B, lr, seed, s0, steps, int(full), threads))


def ref_aggregate(ref: Ref, grads, covered_from, k: int):
    """aggregate (spb.cpp:70-106) through the reference."""
    L = len(grads[0])
    flat, dims = [], np.zeros(k * L, dtype=np.int32)
    for j in range(k):
        for l in range(L):
            g = grads[j][l]
            flat.append(None if g is None or len(g) == 0 else np.ascontiguousarray(g, dtype=np.float64))
            dims[j * L + l] = 0 if flat[-1] is None else len(flat[-1])
    sizes = [max(int(dims[j * L + l]) for j in range(k)) for l in range(L)]
    out = [np.zeros(max(s, 1), dtype=np.float64) for s in sizes]
    cov = np.asarray(covered_from, dtype=np.int32)
    st = ref.lib.ref_aggregate(k, L, _ptr_array(flat), _ip(dims), _ip(cov), _ptr_array(out))
    ref._check(st, "aggregate")
    return [o[:s] for o, s in zip(out, sizes)]


def fp32_round(a: np.ndarray) -> np.ndarray:
    """Rounds fp64 data to fp32 and back, so CPU and GPU see identical inputs."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)
