"""TEST INFRASTRUCTURE ONLY -- a batched fp64 (numpy/BLAS) restatement of one
SPB iteration, for parity checks at sizes the per-sample reference cannot
finish in seconds (the benchmarked cfg3: 16 x 4096 + 1, k = 8, B_w = 128).

It computes the same mathematical quantities as the reference, only grouped
into matrix products instead of the reference's per-sample loop:

* forward, ChainMlp::sample_loss / mlp_forward (model.cpp:108-128):
  h_l = tanh(W_l h_{l-1} + b_l), affine last layer, loss 0.5 ||out - y||^2;
* worker j backpropagates suffix_layers(j, k, L) = ceil(j L / k) layers
  (spb.cpp:16-21), i.e. down to stop_j = L - s_j + 1
  (add_sample_gradient model.cpp:145-186: gW += delta (x) h_{l-1}, gb += delta,
  delta <- (W_l^T delta) * (1 - h_{l-1}^2) while l > stop);
* partial_backprop (spb.cpp:51-68) is the batch mean of the per-sample
  suffix gradients, and aggregate (spb.cpp:70-106) averages layer l over its
  m_l contributors {k - m_l + 1 .. k} (chunk_coverage spb.cpp:23-29), so the
  aggregate of layer l is (1 / (m_l B_w)) * sum over the contributors' rows;
* full backprop (baseline_estimate spb.cpp:149-160) is m_l = k everywhere;
* the update x -= lr g (spb.cpp:196), or the paper's momentum SGD + weight
  decay with PyTorch semantics (parity unpinned by the reference).

Only the summation order differs from the reference (BLAS blocking instead of
batch order), which moves fp64 results by ~1e-15 relative -- far below the
1e-5 / 1e-4 parity bars this checker is used for. It is pinned against the
compiled reference (oracle/_ref) and the C restatement in
tests/test_oracle.py::test_batched_oracle_matches_reference.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


def suffix_layers(j: int, k: int, L: int) -> int:
    """spb.cpp:16-21."""
    return (j * L + k - 1) // k


def contributors(k: int, L: int, full: bool = False) -> List[int]:
    """m_l for l = 1..L: the number of workers whose suffix covers layer l."""
    m = []
    for l in range(1, L + 1):
        m.append(k if full else sum(1 for j in range(1, k + 1) if L - suffix_layers(j, k, L) + 1 <= l))
    return m


def split_block(block: np.ndarray, n_out: int, n_in: int):
    """Block l = W_l row-major [n_out x n_in] followed by b_l (model.hpp:93-94)."""
    W = block[: n_out * n_in].reshape(n_out, n_in)
    b = block[n_out * n_in: n_out * n_in + n_out]
    return W, b


def forward(widths: Sequence[int], X: np.ndarray, params: Sequence[np.ndarray]):
    """Activations H_0 .. H_{L-1} and the head output for the rows of X."""
    L = len(widths) - 1
    H = [np.asarray(X, dtype=np.float64)]
    for l in range(1, L):
        W, b = split_block(params[l - 1], widths[l], widths[l - 1])
        H.append(np.tanh(H[-1] @ W.T + b))
    W, b = split_block(params[L - 1], widths[L], widths[L - 1])
    return H, H[-1] @ W.T + b


def loss(widths, X, Y, params) -> float:
    """ChainMlp::loss (model.cpp:139-143): mean of 0.5 ||out - y||^2."""
    _, out = forward(widths, X, params)
    d = out - np.asarray(Y, dtype=np.float64).reshape(out.shape)
    return float(0.5 * np.mean(np.sum(d * d, axis=1)))


def aggregate_step(widths: Sequence[int], X: np.ndarray, Y: np.ndarray, params: Sequence[np.ndarray], k: int,
                   bw: int, full: bool = False) -> List[np.ndarray]:
    """The aggregated SPB gradient of one iteration. X / Y hold the k workers'
    batches concatenated in worker order (rows (j-1)*bw .. j*bw-1 = worker j)."""
    L = len(widths) - 1
    rows = k * bw
    X = np.asarray(X, dtype=np.float64).reshape(rows, widths[0])
    Y = np.asarray(Y, dtype=np.float64).reshape(rows, widths[L])
    m = contributors(k, L, full)
    H, out = forward(widths, X, params)
    grads: List[np.ndarray] = [None] * L  # type: ignore[list-item]
    r0 = (k - m[L - 1]) * bw
    delta = out[r0:] - Y[r0:]  # delta_L over layer L's contributor rows
    for l in range(L, 0, -1):
        r0 = (k - m[l - 1]) * bw
        d = delta[-(rows - r0):]  # contributor rows of layer l (a tail of the rows)
        h = H[l - 1][r0:]
        scale = 1.0 / (m[l - 1] * bw)
        gW = (d.T @ h) * scale
        gb = d.sum(axis=0) * scale
        grads[l - 1] = np.concatenate([gW.ravel(), gb])
        if l > 1:
            q0 = (k - m[l - 2]) * bw  # rows that continue below layer l
            W, _ = split_block(params[l - 1], widths[l], widths[l - 1])
            dq = delta[-(rows - q0):] if rows - q0 > 0 else delta[:0]
            hq = H[l - 1][q0:]
            delta = (dq @ W) * (1.0 - hq * hq)
    return grads


def sgd_update(params: List[np.ndarray], grads: Sequence[np.ndarray], lr: float, momentum: float = 0.0,
               weight_decay: float = 0.0, bufs: List[np.ndarray] | None = None) -> None:
    """x -= lr g (spb.cpp:196, axpy :120-123) when momentum = wd = 0; otherwise
    PyTorch SGD: g' = g + wd w; buf = mu buf + g' (buf starts at 0); w -= lr buf."""
    for l, g in enumerate(grads):
        if momentum == 0.0 and weight_decay == 0.0:
            params[l] -= lr * g
            continue
        gp = g + weight_decay * params[l]
        bufs[l] *= momentum
        bufs[l] += gp
        params[l] -= lr * bufs[l]
