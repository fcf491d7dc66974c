"""Generates tests/golden/*.npz from the UNMODIFIED reference SPB core.

Run in the build container (needs /root/reference and oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py

Every fixture feeds the reference fp32-rounded data (stored back as fp64) so
the fp32 B200 path and the fp64 reference see identical inputs; only the
arithmetic differs. Inputs come from make_random_chain_mlp (model.cpp:208-231)
with the recorded (widths, samples, seed); outputs come from the reference's
own partial_backprop (spb.cpp:51-68), aggregate (spb.cpp:70-106) and SPB-SGD
iteration (spb.cpp:187-196, via oracle/ref_capi.cpp ref_step). Large blocks
are stored as deterministic samples plus per-layer norms to keep the files
small.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, Ref, RefModel, fp32_round, ref_aggregate  # noqa: E402

SAMPLE = 4096  # stored entries per large block


def sample_idx(n: int, seed: int) -> np.ndarray:
    if n <= SAMPLE:
        return np.arange(n)
    return np.sort(np.random.default_rng(seed).choice(n, SAMPLE, replace=False))


def model_from(orc: Oracle, ref: Ref, widths, samples, seed):
    X, Y, W = orc.gen_chain_mlp(widths, samples, seed)
    X, Y, W = fp32_round(X), fp32_round(Y), [fp32_round(b) for b in W]
    return RefModel(ref, widths, X, Y, W), X, Y, W


def pack_blocks(prefix: str, blocks, out: dict, seed: int):
    for l, b in enumerate(blocks):
        if b is None:
            out[f"{prefix}_absent_{l}"] = np.array(1)
            continue
        idx = sample_idx(b.size, seed + l)
        out[f"{prefix}_idx_{l}"] = idx.astype(np.int64)
        out[f"{prefix}_val_{l}"] = b[idx]
        out[f"{prefix}_norm_{l}"] = np.array(np.linalg.norm(b))
        out[f"{prefix}_size_{l}"] = np.array(b.size)


def main():
    orc, ref = Oracle(), Ref()

    # G1: test_spb.cpp:93-124 instance -- partial backprop per suffix.
    widths, N, seed = [3, 4, 4, 4, 1], 24, 5
    m, X, Y, W = model_from(orc, ref, widths, N, seed)
    batch = np.array([0, 3, 5, 7, 11, 13], dtype=np.int32)
    out = dict(widths=np.array(widths), samples=np.array(N), seed=np.array(seed), batch=batch)
    for suffix in range(1, len(widths)):
        ops = np.zeros(len(widths) - 1, dtype=np.int64)
        g, cov = m.partial_backprop(batch, suffix, ops)
        out[f"cov_{suffix}"] = np.array(cov)
        out[f"ops_{suffix}"] = ops
        pack_blocks(f"pb{suffix}", g, out, 100)
    out["loss"] = np.array(m.loss())
    np.savez_compressed(os.path.join(HERE, "g1_partial_backprop.npz"), **out)

    # G2: SPB-SGD trajectory, k=3 on {3,5,4,1}: params after each step.
    widths, N, seed, k, B, lr, sseed, steps = [3, 5, 4, 1], 32, 1, 3, 6, 0.05, 11, 5
    m, X, Y, W = model_from(orc, ref, widths, N, seed)
    out = dict(widths=np.array(widths), samples=np.array(N), seed=np.array(seed), k=np.array(k), B=np.array(B),
               lr=np.array(lr), step_seed=np.array(sseed), steps=np.array(steps))
    for s in range(1, steps + 1):
        m.step(k, B, lr, sseed, s)
        pack_blocks(f"x{s}", m.get_params(), out, 200)
        for j in range(1, k + 1):
            out[f"batch_{s}_{j}"] = orc.draw_batch(sseed, s, j, B // k, N)
    np.savez_compressed(os.path.join(HERE, "g2_sgd_trajectory.npz"), **out)

    # G3: ragged widths -- one SPB aggregate and one full-backprop mean.
    widths, N, seed, k, bw, sseed = [37, 33, 20, 1], 100, 9, 4, 5, 3
    m, X, Y, W = model_from(orc, ref, widths, N, seed)
    L = len(widths) - 1
    grads, covs = [], []
    for j in range(1, k + 1):
        b = orc.draw_batch(sseed, 1, j, bw, N)
        g, cov = m.partial_backprop(b, ref.suffix_layers(j, k, L))
        grads.append(g)
        covs.append(cov)
    agg = ref_aggregate(ref, grads, covs, k)
    out = dict(widths=np.array(widths), samples=np.array(N), seed=np.array(seed), k=np.array(k), bw=np.array(bw),
               step_seed=np.array(sseed), covered_from=np.array(covs))
    pack_blocks("agg", agg, out, 300)
    np.savez_compressed(os.path.join(HERE, "g3_ragged_aggregate.npz"), **out)

    # G4: cfg1 (784-512-512-1, N=4096, k=4, B_w=128): the aggregate of step 1
    # and the params after 10 SPB-SGD steps (lr 1e-2, step seed 11).
    widths, N, seed, k, bw, lr, sseed, steps = [784, 512, 512, 1], 4096, 7, 4, 128, 1e-2, 11, 10
    m, X, Y, W = model_from(orc, ref, widths, N, seed)
    L = len(widths) - 1
    grads, covs = [], []
    for j in range(1, k + 1):
        b = orc.draw_batch(sseed, 1, j, bw, N)
        g, cov = m.partial_backprop(b, ref.suffix_layers(j, k, L))
        grads.append(g)
        covs.append(cov)
    agg = ref_aggregate(ref, grads, covs, k)
    out = dict(widths=np.array(widths), samples=np.array(N), seed=np.array(seed), k=np.array(k), bw=np.array(bw),
               lr=np.array(lr), step_seed=np.array(sseed), steps=np.array(steps), covered_from=np.array(covs))
    pack_blocks("agg", agg, out, 400)
    for s in range(1, steps + 1):
        m.step(k, k * bw, lr, sseed, s)
    pack_blocks("x10", m.get_params(), out, 500)
    out["loss10"] = np.array(m.loss())
    np.savez_compressed(os.path.join(HERE, "g4_cfg1.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
