"""NCCL all-reduce / reduce-scatter / all-gather bandwidth on this box (torch.distributed, fp32)."""
import os
import time

import torch
import torch.distributed as dist


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    for mb in (64, 256, 1024):
        n = mb * (1 << 20) // 4
        x = torch.ones(n, device="cuda")
        for _ in range(3):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(10):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / 10
        alg = mb / 1024 / t
        if rank == 0:
            print(f"all_reduce {mb:5d} MB: {t * 1e3:7.3f} ms  algbw {alg:6.1f} GB/s  busbw {alg * 2 * (world - 1) / world:6.1f} GB/s",
                  flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
