"""The N>1 protocol on CPU with torch.distributed gloo (world sizes 2, 4 and 8).

Every rank hosts the workers spb_rank_workers(k, L, rank, N) assigns it and
computes its local per-layer contribution with the CPU oracle (the mean of
each hosted contributor's partial_backprop block divided by the layer's
GLOBAL contributor count, i.e. what the device wgrad epilogue produces with
alpha_l = 1/(m_l * B_w)), then runs an exchange mode's protocol: sub (each layer reduced among its
contributing ranks only (spb_bucket_plan), the owners' sharded update, weight
broadcast to every rank) or push (the MLP default from 3 to 8 ranks: gradient
rows stored to their block-row owners, owner-side sum in rank order, update,
rows fetched by every rank). The weights must be rank-identical and equal the single-process
oracle's SPB step (aggregate spb.cpp:70-106 + x -= lr g).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


WIDTHS, N, K, BW, LR, SEED, DSEED = [11, 9, 8, 7, 6, 5, 4, 3, 1], 64, 8, 3, 0.05, 11, 4


def test_bucket_plan_shapes():
    from paper_2111_10672_b200 import spb

    L = 16
    for world in (1, 2, 4, 8):
        plan = spb.bucket_plan(8, L, world)
        for l, (kind, root, ranks) in enumerate(plan, 1):
            assert ranks, "every layer has a contributor (worker k backpropagates all layers)"
            assert (kind == 1) == (len(ranks) == 1)
            if kind == 1:
                assert root == ranks[0]
        full = spb.bucket_plan(8, L, world, full_backprop=True)
        assert all(r == list(range(world)) for _, _, r in full)
    plan8 = spb.bucket_plan(8, L, 8)
    assert [len(r) for _, _, r in plan8] == [1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8]


def _sub_worker(rank, world, port, out_dir, k):
    """The sub exchange mode (engine.cu enqueue_sub_layer): per layer, the
    contributing ranks reduce (a reduce-scatter, here all-reduce + own shard)
    over their own group only, each updates its shard (spb_layer_shard), and
    every member broadcasts its updated shard to all ranks."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle.oracle import Oracle
    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    L = len(WIDTHS) - 1
    X, Y, W = orc.gen_chain_mlp(WIDTHS, N, DSEED)
    chunks = spb.layer_chunks(k, L)
    local = [np.zeros_like(b) for b in W]
    for j in spb.rank_workers(k, L, rank, world):
        g, cov = orc.partial_backprop(WIDTHS, X, Y, W, orc.draw_batch(SEED, 1, j, BW, N), spb.suffix_layers(j, k, L))
        for l in range(cov, L + 1):
            local[l - 1] += g[l - 1] / chunks[l - 1]
    plan = spb.bucket_plan(k, L, world)
    sets = sorted({tuple(r) for _, _, r in plan if len(r) > 1})
    groups = {s: dist.new_group(list(s)) for s in sets}  # collectively, same order everywhere
    P = [b.copy() for b in W]
    moved = 0.0
    for l in range(L, 0, -1):
        _, _, ranks = plan[l - 1]
        cnt = local[l - 1].size
        sh = spb.layer_shard(cnt, len(ranks))
        bounds = [(min(cnt, i * sh), min(cnt, (i + 1) * sh)) for i in range(len(ranks))]
        if rank in ranks:
            t = torch.from_numpy(local[l - 1].copy())
            if len(ranks) > 1:
                dist.all_reduce(t, group=groups[tuple(ranks)])
                moved += t.numel()
            a, b = bounds[ranks.index(rank)]
            P[l - 1][a:b] = W[l - 1][a:b] - LR * t.numpy()[a:b]
        for i, r in enumerate(ranks):
            a, b = bounds[i]
            if b > a:
                t = torch.from_numpy(np.ascontiguousarray(P[l - 1][a:b]))
                dist.broadcast(t, src=r)
                P[l - 1][a:b] = t.numpy()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *P, np.array([moved]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 8), (4, 8), (8, 8), (2, 2), (4, 4)])
def test_sub_protocol_matches_single_process_step(tmp_path, world, k, orc):
    """Contributor sub-communicators (the sub mode): the
    weights after one step equal the single-process SPB step, on every rank;
    with one worker per rank (k = world) ranks outside a layer's contributor
    set move no gradient bytes for it."""
    mp.start_processes(_sub_worker, args=(world, _free_port(), str(tmp_path), k), nprocs=world, start_method="spawn")
    L = len(WIDTHS) - 1
    X, Y, W = orc.gen_chain_mlp(WIDTHS, N, DSEED)
    P = [b.copy() for b in W]
    orc.spb_step(WIDTHS, X, Y, P, k, k * BW, LR, SEED, 1)
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for r in range(world):
        for l in range(L):
            got = outs[r][f"arr_{l}"]
            np.testing.assert_allclose(got, P[l], rtol=1e-12, atol=1e-15)
            assert np.array_equal(got, outs[0][f"arr_{l}"])  # rank-identical weights
    if k == world:  # rank 0 (worker 1) contributes to the top layers only
        from paper_2111_10672_b200 import spb

        top = spb.suffix_layers(1, k, L)
        dims = spb.block_dims(WIDTHS)
        assert float(outs[0][f"arr_{L}"][0]) <= sum(dims[L - top:])


def _push_worker(rank, world, port, out_dir, k):
    """The push exchange mode (exchange.cu enqueue_push_layer, the MLP default
    from 3 to 8 ranks): layer l's rows are owned block-wise (rank o: rows
    [o * rpo, (o + 1) * rpo), rpo = ceil(n_l / N)); every contributing rank
    stores its gradient rows (weights and bias) into their owners' staging
    (here point-to-point sends), the owner sums the contributing ranks' rows
    in ascending rank order and updates them, and every rank fetches the
    other owners' updated rows (here broadcasts)."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle.oracle import Oracle
    from paper_2111_10672_b200 import spb

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    L = len(WIDTHS) - 1
    X, Y, W = orc.gen_chain_mlp(WIDTHS, N, DSEED)
    chunks = spb.layer_chunks(k, L)
    local = [np.zeros_like(b) for b in W]
    for j in spb.rank_workers(k, L, rank, world):
        g, cov = orc.partial_backprop(WIDTHS, X, Y, W, orc.draw_batch(SEED, 1, j, BW, N), spb.suffix_layers(j, k, L))
        for l in range(cov, L + 1):
            local[l - 1] += g[l - 1] / chunks[l - 1]
    plan = spb.bucket_plan(k, L, world)
    P = [b.copy() for b in W]
    for l in range(L, 0, -1):
        _, _, ranks = plan[l - 1]
        n_out, n_in = WIDTHS[l], WIDTHS[l - 1]
        rpo = -(-n_out // world)
        rows = [(min(n_out, o * rpo), min(n_out, (o + 1) * rpo)) for o in range(world)]

        def block(flat, o):  # owner o's weight rows, then its bias entries
            a, b = rows[o]
            return np.concatenate([flat[a * n_in:b * n_in], flat[n_out * n_in + a:n_out * n_in + b]])

        staged = {}
        for o in range(world):  # 1. contributors store their rows to the owners
            for r in ranks:
                if r == o or rank not in (r, o):
                    continue
                if rank == r:
                    dist.send(torch.from_numpy(block(local[l - 1], o)), dst=o)
                else:
                    buf = torch.empty(block(local[l - 1], o).shape, dtype=torch.float64)
                    dist.recv(buf, src=r)
                    staged[r] = buf.numpy()
        a, b = rows[rank]  # 2. the owner sums in rank order and updates its rows
        if b > a:
            acc = np.zeros_like(block(local[l - 1], rank))
            for r in ranks:
                acc = acc + (block(local[l - 1], rank) if r == rank else staged[r])
            new = block(W[l - 1], rank) - LR * acc
            P[l - 1][a * n_in:b * n_in] = new[:(b - a) * n_in]
            P[l - 1][n_out * n_in + a:n_out * n_in + b] = new[(b - a) * n_in:]
        for o in range(world):  # 3. every rank fetches the other owners' rows
            a, b = rows[o]
            if b <= a:
                continue
            t = torch.from_numpy(block(P[l - 1], o))
            dist.broadcast(t, src=o)
            P[l - 1][a * n_in:b * n_in] = t.numpy()[:(b - a) * n_in]
            P[l - 1][n_out * n_in + a:n_out * n_in + b] = t.numpy()[(b - a) * n_in:]
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *P)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k", [(2, 8), (4, 8), (8, 8), (4, 4)])
def test_push_protocol_matches_single_process_step(tmp_path, world, k, orc):
    """The push mode's row ownership and owner-side summation at world sizes
    2 / 4 / 8 (8 = one SPB worker per rank, the north_star layout): weights
    after one step equal the single-process SPB step on every rank, and are
    rank-identical."""
    mp.start_processes(_push_worker, args=(world, _free_port(), str(tmp_path), k), nprocs=world, start_method="spawn")
    L = len(WIDTHS) - 1
    X, Y, W = orc.gen_chain_mlp(WIDTHS, N, DSEED)
    P = [b.copy() for b in W]
    orc.spb_step(WIDTHS, X, Y, P, k, k * BW, LR, SEED, 1)
    outs = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    for r in range(world):
        for l in range(L):
            np.testing.assert_allclose(outs[r][f"arr_{l}"], P[l], rtol=1e-12, atol=1e-15)
            assert np.array_equal(outs[r][f"arr_{l}"], outs[0][f"arr_{l}"])


def test_layer_shard_partition():
    from paper_2111_10672_b200 import spb

    for cnt in (1, 3, 4, 5, 97, 4096, 16781344):
        for parts in range(1, 9):
            sh = spb.layer_shard(cnt, parts)
            assert sh % 4 == 0 and parts * sh >= cnt and (parts - 1) * sh < cnt + 4 * parts
