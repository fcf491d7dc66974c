"""Multi-GPU cfg3 step breakdown (tuning aid): graph-replay ms/step, then one
eager step's per-class CUDA-event times, per rank, for each exchange mode.

    python tools/multi_profile.py [world] [modes, e.g. p2p,sub,push,rh] [widths]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(rank, world, port, mode, widths_s):
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPB_COMM"] = mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, rest = widths_s.split("x")
    depth, head = rest.split("+")
    widths = [int(n)] * int(depth) + [int(head)]
    X, Y, W = spb.gen_chain_mlp(widths, 8192, 7)
    m = spb.ChainMlp(widths, X, Y, W, k=8, per_worker_batch=128, device=rank)
    m.comm_init_torch(dist, rank, world)
    m.set_optimizer(0.01, 0.9, 1e-4)
    m.train_steps(11, 1, 5)
    ms = m.time_train_steps(11, 6, 20)
    prof, step_ms = m.profile_step(11, 30)
    dist.barrier()
    cls = " ".join(f"{c}={v['ms']:.3f}/{v['launches']}" for c, v in prof.items() if v["launches"])
    print(f"[{mode} r{rank}] graph {ms:.3f} ms/step | eager {step_ms:.3f} ms: {cls}", flush=True)
    dist.barrier()
    m.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["p2p", "sub"]
    widths = sys.argv[3] if len(sys.argv) > 3 else "4096x16+1"
    for i, nv in enumerate(modes):
        mp.start_processes(run, args=(world, 29700 + 10 * i + world, nv, widths), nprocs=world, start_method="spawn")
