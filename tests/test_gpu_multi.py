"""Multi-GPU SPB step (needs >= 2 GPUs; skipped otherwise).

Each rank runs its balanced worker set on its own B200. Aggregation paths:
p2p (copy-engine pulls of gradient shards, sharded update, pulls of the
updated weights), rh (the same on a recursive-halving / -doubling schedule),
push (gradient rows stored to their owners by the wgrad epilogue) and sub
(NCCL reduce-scatter among each layer's contributing ranks only, over
contributor sub-communicators, sharded update, weight broadcast to every
rank).
Weights after 3 steps must equal the single-process CPU oracle's SPB-SGD
iterates (1e-4) and be bit-identical across ranks; batch indices must be
bit-exact.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(fn, world, *rest):
    """mp.start_processes(fn, args=(world, port, *rest)) on a fresh port,
    retried when another process grabbed the port first (EADDRINUSE)."""
    import torch.multiprocessing as mp

    for attempt in range(4):
        try:
            return mp.start_processes(fn, args=(world, _free_port(), *rest), nprocs=world, start_method="spawn")
        except Exception as ex:  # noqa: BLE001
            if "EADDRINUSE" not in str(ex) or attempt == 3:
                raise


WIDTHS, N, K, BW, LR, SEED, DSEED = [96, 80, 72, 64, 56, 48, 40, 32, 1], 512, 8, 16, 0.05, 11, 5


def _rank(rank, world, port, out_dir, full, mode="p2p", mu=0.0, wd=0.0, chain=None, steps=2):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPB_COMM"] = mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y, W = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    m = spb.ChainMlp(WIDTHS, X, Y, W, k=K, per_worker_batch=BW, device=rank)
    m.comm_init_torch(dist, rank, world)
    assert m.comm_mode == mode
    m.set_optimizer(LR, mu, wd)
    if chain is not None:
        m.set_chain(chain)
    m.train_steps(SEED, 1, 1, full_backprop=full)
    idx = m.last_batch(len(spb.rank_workers(K, len(WIDTHS) - 1, rank, world)) * BW)
    m.train_steps(SEED, 2, steps, full_backprop=full)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), idx, *m.get_params())
    dist.barrier()
    m.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["rh", "push", "p2p", "sub"])
@pytest.mark.parametrize("full", [False, True])
def test_multi_gpu_step_matches_oracle(tmp_path, orc, full, mode):
    world = min(_gpus(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")

    from paper_2111_10672_b200 import spb

    _launch(_rank, world, str(tmp_path), full, mode)
    L = len(WIDTHS) - 1
    X, Y, W = orc.gen_chain_mlp(WIDTHS, N, DSEED)
    Xf, Yf, Wf = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    X, Y, P = Xf.astype(np.float64), Yf.astype(np.float64), [b.astype(np.float64) for b in Wf]
    for s in range(1, 4):
        orc.spb_step(WIDTHS, X, Y, P, K, K * BW, LR, SEED, s, full=full)
    outs = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    for r in range(world):
        ws = spb.rank_workers(K, L, r, world)
        want = np.concatenate([orc.draw_batch(SEED, 1, j, BW, N) for j in ws])
        assert np.array_equal(outs[r]["arr_0"], want)
        for l in range(L):
            got = outs[r][f"arr_{l + 1}"]
            assert np.linalg.norm(got - P[l]) / np.linalg.norm(P[l]) <= 1e-4
            assert np.array_equal(got, outs[0][f"arr_{l + 1}"])


def _rank_momentum(rank, world, port, out_dir, mode):
    _rank(rank, world, port, out_dir, False, mode, 0.9, 1e-3)


def test_multi_gpu_momentum_sharded_modes_agree(tmp_path):
    """Momentum + weight decay: every mode keeps each element's momentum
    buffer on the rank owning its shard; after 3 steps their weights must
    agree with the sub mode's (NCCL reductions) to fp32 rounding, and be
    bit-identical across ranks."""
    world = min(_gpus(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")

    res = {}
    for mode in ("rh", "push", "p2p", "sub"):
        d = tmp_path / mode
        d.mkdir()
        _launch(_rank_momentum, world, str(d), mode)
        res[mode] = [np.load(d / f"r{r}.npz") for r in range(world)]
    L = len(WIDTHS) - 1
    for l in range(L):  # push and p2p sum the same contributions in the same order
        for r in range(world):
            assert np.array_equal(res["push"][r][f"arr_{l + 1}"], res["p2p"][r][f"arr_{l + 1}"])
    for mode in ("rh", "push", "p2p"):
        for l in range(L):
            a, b = res[mode][0][f"arr_{l + 1}"], res["sub"][0][f"arr_{l + 1}"]
            assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
            for r in range(world):
                assert np.array_equal(res[mode][r][f"arr_{l + 1}"], a)


def _rank_chain(rank, world, port, out_dir, mode, chain):
    _rank(rank, world, port, out_dir, False, mode, 0.9, 1e-3, chain=chain, steps=7)


@pytest.mark.parametrize("mode", ["push", "p2p", "rh"])
def test_multi_gpu_chained_graph_bitwise(tmp_path, mode):
    """Cross-step pipelining (spb_set_chain): with 7 iterations captured in one
    graph, iteration t+1's forward of layer l waits only for W_l of
    iteration t (its exchange and update) while the rest of iteration t's
    exchange still runs. Weights must be bit-identical to one graph per
    iteration and across ranks."""
    world = min(_gpus(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")

    res = {}
    for chain in (1, 8):
        d = tmp_path / f"c{chain}"
        d.mkdir()
        _launch(_rank_chain, world, str(d), mode, chain)
        res[chain] = [np.load(d / f"r{r}.npz") for r in range(world)]
    for l in range(len(WIDTHS) - 1):
        a = res[1][0][f"arr_{l + 1}"]
        for r in range(world):
            assert np.array_equal(res[8][r][f"arr_{l + 1}"], a)
            assert np.array_equal(res[1][r][f"arr_{l + 1}"], a)


CSHAPE, CCONVS, CNOUT = (8, 8, 3), [(8, 1), (12, 2), (16, 1)], 3


def _rank_conv(rank, world, port, out_dir, mode):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPB_COMM"] = mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y, W = spb.gen_convnet(CSHAPE, CCONVS, CNOUT, N, DSEED)
    m = spb.ConvNet(CSHAPE, CCONVS, CNOUT, X, Y, W, k=K, per_worker_batch=BW, device=rank)
    m.comm_init_torch(dist, rank, world)
    assert m.comm_mode == mode
    m.set_optimizer(LR)
    m.train_steps(SEED, 1, 3)
    np.savez(os.path.join(out_dir, f"c{rank}.npz"), *m.get_params())
    dist.barrier()
    m.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["rh", "p2p", "sub"])
def test_multi_gpu_convnet_matches_oracle(tmp_path, orc, mode):
    """The ConvNet (cfg4 shape family) on 2-4 GPUs: 3 SPB steps equal the
    single-process fp64 conv oracle (1e-4) and are bit-identical across ranks."""
    world = min(_gpus(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")

    from oracle.conv_oracle import ConvOracle
    from paper_2111_10672_b200 import spb

    _launch(_rank_conv, world, str(tmp_path), mode)
    X, Y, W = spb.gen_convnet(CSHAPE, CCONVS, CNOUT, N, DSEED)
    o = ConvOracle(CSHAPE, CCONVS, CNOUT)
    B = [w.astype(np.float64) for w in W]
    for s in range(1, 4):
        o.spb_step(B, X.astype(np.float64), Y.astype(np.float64), K, BW, LR, SEED, s, orc)
    outs = [np.load(os.path.join(tmp_path, f"c{r}.npz")) for r in range(world)]
    for l in range(o.L):
        got = outs[0][f"arr_{l}"]
        assert np.linalg.norm(got - B[l]) / np.linalg.norm(B[l]) <= 1e-4
        for r in range(world):
            assert np.array_equal(outs[r][f"arr_{l}"], got)


def _rank_one_worker(rank, world, port, out_dir, mode):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["SPB_COMM"] = mode
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y, W = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    m = spb.ChainMlp(WIDTHS, X, Y, W, k=world, per_worker_batch=BW, device=rank)
    m.comm_init_torch(dist, rank, world)
    assert m.comm_mode == mode
    m.set_optimizer(LR, 0.9, 1e-3)
    m.train_steps(SEED, 1, 3)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), *m.get_params())
    dist.barrier()
    m.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["sub", "p2p"])
def test_multi_gpu_one_worker_per_gpu(tmp_path, orc, mode):
    """north_star's layout at small scale: k = world workers, ONE per GPU, so a
    layer's contributing ranks are a strict suffix of the ranks and the sub
    mode reduces each layer over its own contributor sub-communicator. Weights
    after 3 momentum + wd steps match the CPU oracle's restatement (1e-4) and
    are rank-identical."""
    world = min(_gpus(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")
    from oracle import batched
    from paper_2111_10672_b200 import spb

    _launch(_rank_one_worker, world, str(tmp_path), mode)
    Xf, Yf, Wf = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    X, Y = Xf.astype(np.float64), Yf.astype(np.float64)
    P = [b.astype(np.float64) for b in Wf]
    bufs = [np.zeros_like(p) for p in P]
    for s in range(1, 4):
        rows = np.concatenate([orc.draw_batch(SEED, s, j, BW, N) for j in range(1, world + 1)])
        g = batched.aggregate_step(WIDTHS, X[rows], Y[rows], P, world, BW)
        batched.sgd_update(P, g, LR, 0.9, 1e-3, bufs)
    outs = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    for l in range(len(WIDTHS) - 1):
        for r in range(world):
            got = outs[r][f"arr_{l}"]
            assert np.linalg.norm(got - P[l]) / np.linalg.norm(P[l]) <= 1e-4
            assert np.array_equal(got, outs[0][f"arr_{l}"])


def test_contexts_on_two_devices_in_one_process(orc):
    """One process driving contexts on two GPUs (the reference's threads
    each own a model; the drop-in binds a context to the caller's device):
    per-device kernel attributes and the ones box are set up on each device,
    and the same SPB steps give bit-identical weights on both, equal to the
    CPU oracle (1e-4)."""
    if _gpus() < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2111_10672_b200 import spb

    X, Y, W = spb.gen_chain_mlp(WIDTHS, N, DSEED)
    outs = []
    for dev in (1, 0):  # device 1 first: its kernels are configured before device 0's
        m = spb.ChainMlp(WIDTHS, X, Y, W, k=K, per_worker_batch=BW, device=dev)
        try:
            m.set_optimizer(LR)
            m.train_steps(SEED, 1, 3)
            outs.append(m.get_params())
        finally:
            m.close()
    X64, Y64 = X.astype(np.float64), Y.astype(np.float64)
    P = [b.astype(np.float64) for b in W]
    for s in range(1, 4):
        orc.spb_step(WIDTHS, X64, Y64, P, K, K * BW, LR, SEED, s)
    for l in range(len(WIDTHS) - 1):
        assert np.array_equal(outs[0][l], outs[1][l])
        assert np.linalg.norm(outs[0][l] - P[l]) / np.linalg.norm(P[l]) <= 1e-4
