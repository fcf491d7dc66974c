"""Tuning experiment: TMEM accumulation chunk (k-blocks per chunk) per GEMM kind
vs fp32-faithfulness at the full cfg3 depth and step time.

    python tools/chunk_experiment.py build_variants/*/libspb_b200.so

For each library variant (built with SPB_NVCC_EXTRA=-DSPB_CHUNK_KB_{FWD,DGRAD,WGRAD}=n),
in its own process: the step-1 SPB aggregate of cfg3 (4096 x 16 + 1, k = 8,
B_w = 128) vs oracle/batched.py (per-layer relative error), and the SPB step
time (10 graph steps after 3 warm-up, momentum + wd)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = "/tmp/chunk_ref.npz"


def child(lib):
    os.environ["SPB_LIB_PATH"] = lib
    from paper_2111_10672_b200 import spb

    widths, k, bw, N, seed = [4096] * 16 + [1], 8, 128, 8192, 11
    X, Y, W = spb.gen_chain_mlp(widths, N, 7)
    m = spb.ChainMlp(widths, X, Y, W, k=k, per_worker_batch=bw)
    m.set_optimizer(0.0)
    m.set_fused_update(0)
    m.train_steps(seed, 1, 1)
    g = m.get_grads()
    ref = np.load(REF)
    errs = [float(np.linalg.norm(g[l] - ref[f"g{l}"]) / np.linalg.norm(ref[f"g{l}"])) for l in range(16)]
    m.set_params(W)
    m.set_optimizer(0.01, 0.9, 1e-4)
    m.set_fused_update(2)
    m.train_steps(seed, 1, 3)
    m.synchronize()
    ms = m.time_train_steps(seed, 4, 10) / 10
    print(json.dumps({"lib": lib, "ms_per_step": ms, "max_err": max(errs), "errs": errs}), flush=True)


def main(libs):
    if not os.path.exists(REF):
        from oracle import batched
        from oracle.oracle import Oracle
        from paper_2111_10672_b200 import spb

        widths, k, bw, N, seed = [4096] * 16 + [1], 8, 128, 8192, 11
        X, Y, W = spb.gen_chain_mlp(widths, N, 7)
        o = Oracle()
        rows = np.concatenate([o.draw_batch(seed, 1, j, bw, N) for j in range(1, k + 1)])
        g = batched.aggregate_step(widths, X[rows].astype(np.float64), Y[rows].astype(np.float64),
                                   [b.astype(np.float64) for b in W], k, bw)
        np.savez(REF, **{f"g{l}": g[l] for l in range(16)})
    for lib in libs:
        subprocess.run([sys.executable, __file__, "--child", lib])


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2])
    else:
        main(sys.argv[1:])
