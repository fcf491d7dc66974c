"""cfg5 (BASELINE configs[4]): SPB vs full-backprop scaling sweep over layer
widths 1k-8k (ChainMlp, 16 layers + scalar head, k = 8 workers x 128 rows),
with the saved backward FLOPs and exchange bytes of each point.

    python tools/sweep.py                        # 1 GPU
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/sweep.py                           # N GPUs (one process each)

Rank 0 prints one JSON line per width. Timed over 10 steps after 3 warm-up
steps: short bursts (the SM clock has not yet settled under the power cap),
~5 % faster than bench.py's longer timed regions on the same box.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402  (timing helpers, spb_savings)
from paper_2111_10672_b200 import spb  # noqa: E402

WIDTHS = [1024, 2048, 4096, 8192]
K, BW, N, STEPS, WARM = 8, 128, 4096, 10, 3


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    for n in WIDTHS:
        widths = [n] * 16 + [1]
        X, Y, W = spb.gen_chain_mlp(widths, N, 7)
        m = spb.ChainMlp(widths, X, Y, W, k=K, per_worker_batch=BW, device=local)
        del X, Y, W
        if world > 1:
            m.comm_init_torch(dist, rank, world)
        m.set_optimizer(0.01, 0.9, 1e-4)
        res = {}
        for full in (False, True):
            m.set_params(m.initial_params())
            m.train_steps(11, 1, WARM, full_backprop=full)
            m.synchronize()
            bench.barrier(dist)
            ms = m.time_train_steps(11, 1 + WARM, STEPS, full_backprop=full)
            bench.barrier(dist)
            ms = bench.max_over_ranks(dist, ms) / STEPS
            res["full" if full else "spb"] = {"ms_per_step": round(ms, 4), "samples_per_s": round(K * BW / (ms * 1e-3), 1)}
        mode = m.comm_mode if world > 1 else "local"
        m.close()
        if rank == 0:
            line = {"workload": f"cfg5: ChainMlp 16x{n} + scalar head, k={K} x {BW} rows", "n_gpus": world,
                    "aggregation": mode, **res,
                    "spb_speedup": round(res["full"]["ms_per_step"] / res["spb"]["ms_per_step"], 4),
                    "savings": bench.spb_savings(widths, K, BW, world)}
            print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
