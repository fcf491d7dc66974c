"""Diagnostics: the ConvNet on N GPUs (tests/test_gpu_multi.py's shapes),
per-layer error against the CPU conv oracle after each of 3 steps, and
cross-rank equality. python tools/conv_multi_debug.py WORLD MODE"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CSHAPE, CCONVS, CNOUT = (8, 8, 3), [(8, 1), (12, 2), (16, 1)], 3
N, K, BW, LR, SEED, DSEED = 512, 8, 16, 0.05, 11, 5


def run(rank, world, port, mode, out):
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPB_COMM"] = mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y, W = spb.gen_convnet(CSHAPE, CCONVS, CNOUT, N, DSEED)
    m = spb.ConvNet(CSHAPE, CCONVS, CNOUT, X, Y, W, k=K, per_worker_batch=BW, device=rank)
    m.comm_init_torch(dist, rank, world)
    m.set_optimizer(LR)
    res = []
    for s in range(1, 4):
        m.train_steps(SEED, s, 1)
        res.append(m.get_params())
    np.save(os.path.join(out, f"r{rank}.npy"), np.array(res, dtype=object), allow_pickle=True)
    dist.barrier()
    m.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    from oracle.conv_oracle import ConvOracle
    from oracle.oracle import Oracle
    from paper_2111_10672_b200 import spb

    world, mode = int(sys.argv[1]), sys.argv[2]
    out = os.path.join(ROOT, "gpurun_out", "conv_debug")
    os.makedirs(out, exist_ok=True)
    mp.start_processes(run, args=(world, 29931, mode, out), nprocs=world, start_method="spawn")
    X, Y, W = spb.gen_convnet(CSHAPE, CCONVS, CNOUT, N, DSEED)
    o = ConvOracle(CSHAPE, CCONVS, CNOUT)
    orc = Oracle()
    B = [w.astype(np.float64) for w in W]
    got = [np.load(os.path.join(out, f"r{r}.npy"), allow_pickle=True) for r in range(world)]
    for s in range(1, 4):
        o.spb_step(B, X.astype(np.float64), Y.astype(np.float64), K, BW, LR, SEED, s, orc)
        for l in range(o.L):
            errs = [float(np.linalg.norm(got[r][s - 1][l] - B[l]) / np.linalg.norm(B[l])) for r in range(world)]
            same = all(np.array_equal(got[r][s - 1][l], got[0][s - 1][l]) for r in range(world))
            print(f"step {s} layer {l}: rel err per rank {['%.2e' % e for e in errs]} rank-identical {same}")
