"""Step-by-step multi-GPU bring-up with progress prints (debug aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(rank, world, port, mode):
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    def log(*a):
        print(f"[r{rank} {time.time():.1f}]", *a, flush=True)

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    widths = [96, 80, 72, 64, 56, 48, 40, 32, 1]
    X, Y, W = spb.gen_chain_mlp(widths, 512, 5)
    m = spb.ChainMlp(widths, X, Y, W, k=8, per_worker_batch=16, device=rank)
    log("ctx ok")
    m.comm_init_torch(dist, rank, world)
    log("comm ok")
    m.set_optimizer(0.05)
    prof, ms = m.profile_step(11, 1)
    log("eager step ok", ms, prof["comm"])
    m.train_steps(11, 2, 1)
    m.synchronize()
    log("graph step ok")
    m.train_steps(11, 3, 5)
    m.synchronize()
    log("5 graph steps ok")
    dist.barrier()
    m.close()
    log("closed")
    dist.destroy_process_group()
    log("pg destroyed")


if __name__ == "__main__":
    import torch.multiprocessing as mp

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    mp.start_processes(run, args=(world, 29600 + world, "x"), nprocs=world, start_method="spawn")
