"""NVLink peer-copy bandwidth between the GPUs of one box (tuning aid):
one-way and bidirectional copies of a 1 GiB buffer, timed with CUDA events.

    python tools/p2p_bench.py
"""
import torch


def timed(fn, streams, reps=5):
    fn()
    for s in streams:
        s.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in streams]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in streams]
    for s, e in zip(streams, e0):
        e.record(s)
    for _ in range(reps):
        fn()
    for s, e in zip(streams, e1):
        e.record(s)
    for s in streams:
        s.synchronize()
    return max(a.elapsed_time(b) for a, b in zip(e0, e1)) / reps


def main():
    n = torch.cuda.device_count()
    size = 1 << 30
    bufs = [torch.empty(size, dtype=torch.uint8, device=f"cuda:{i}") for i in range(n)]
    dst = [torch.empty(size, dtype=torch.uint8, device=f"cuda:{i}") for i in range(n)]
    st = [torch.cuda.Stream(device=f"cuda:{i}") for i in range(n)]
    print("peer access 0->1:", torch.cuda.can_device_access_peer(0, 1))

    def one_way():
        with torch.cuda.stream(st[0]):
            dst[1].copy_(bufs[0], non_blocking=True)

    ms = timed(one_way, [st[0]])
    print(f"one-way 0->1      {ms:.3f} ms  {size / ms / 1e6:.1f} GB/s")

    def bidir():
        with torch.cuda.stream(st[0]):
            dst[1].copy_(bufs[0], non_blocking=True)
        with torch.cuda.stream(st[1]):
            dst[0].copy_(bufs[1], non_blocking=True)

    ms = timed(bidir, [st[0], st[1]])
    print(f"bidir 0<->1       {ms:.3f} ms  {size / ms / 1e6:.1f} GB/s per direction")
    # Pull vs push with explicit streams (cudaMemcpyAsync on the stream of the
    # device that executes the copy): torch's cross-device copy_ always runs
    # on the source device (a push).
    from cuda.bindings import runtime as rt

    def ce_copy(exec_dev, dst_t, src_t, nbytes, reps=5):
        torch.cuda.set_device(exec_dev)
        s = torch.cuda.Stream(device=f"cuda:{exec_dev}")
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        kind = rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice
        rt.cudaMemcpyAsync(dst_t.data_ptr(), src_t.data_ptr(), nbytes, kind, s.cuda_stream)
        a.record(s)
        for _ in range(reps):
            rt.cudaMemcpyAsync(dst_t.data_ptr(), src_t.data_ptr(), nbytes, kind, s.cuda_stream)
        b.record(s)
        s.synchronize()
        return a.elapsed_time(b) / reps

    for nbytes in (16 << 20, 64 << 20, 1 << 30):
        ms_push = ce_copy(0, dst[1], bufs[0], nbytes)
        ms_pull = ce_copy(1, dst[1], bufs[0], nbytes)
        print(f"{nbytes >> 20:5d} MiB 0->1  push (dev0 CE) {nbytes / ms_push / 1e6:7.1f} GB/s   "
              f"pull (dev1 CE) {nbytes / ms_pull / 1e6:7.1f} GB/s")
    # The p2p aggregation pattern: every GPU pulls a shard from every peer at
    # once, one stream per (GPU, peer); timed per stream with CUDA events.
    kind = rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice
    for i in range(n):
        torch.cuda.set_device(i)
        for p in range(n):
            if p != i:
                rt.cudaDeviceEnablePeerAccess(p, 0)  # already-enabled pairs just return an error code
    for total in (64 << 20, 256 << 20):
        shard = total // n
        reps = 10
        streams = {(i, p): torch.cuda.Stream(device=f"cuda:{i}") for i in range(n) for p in range(n) if p != i}
        evs = {}
        for i in range(n):
            torch.cuda.synchronize(i)
        for i in range(n):
            torch.cuda.set_device(i)
            for p in range(n):
                if p == i:
                    continue
                s = streams[(i, p)]
                a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_ev.record(s)
                for _ in range(reps):
                    rt.cudaMemcpyAsync(dst[i].data_ptr() + p * shard, bufs[p].data_ptr() + i * shard, shard, kind,
                                       s.cuda_stream)
                b_ev.record(s)
                evs[(i, p)] = (a_ev, b_ev)
        for i in range(n):
            torch.cuda.synchronize(i)
        worst = max(a_ev.elapsed_time(b_ev) for a_ev, b_ev in evs.values()) / reps
        print(f"all-pull x{n}: {shard >> 20} MiB from each of {n - 1} peers: {worst * 1e3:.1f} us/round (slowest "
              f"stream)  {(n - 1) * shard / worst / 1e6:.1f} GB/s inbound per GPU")
    if n >= 4:
        def ring():
            for i in range(n):
                with torch.cuda.stream(st[i]):
                    dst[(i + 1) % n].copy_(bufs[i], non_blocking=True)

        ms = timed(ring, st)
        print(f"ring x{n} (i->i+1) {ms:.3f} ms  {size / ms / 1e6:.1f} GB/s per GPU out")

        part = size // (n - 1)

        def fan_out():  # each GPU sends 1/(n-1) GiB to every other GPU
            for i in range(n):
                with torch.cuda.stream(st[i]):
                    for j in range(1, n):
                        t = (i + j) % n
                        dst[t][(j - 1) * part:j * part].copy_(bufs[i][:part], non_blocking=True)

        ms = timed(fan_out, st)
        print(f"all-to-all x{n}    {ms:.3f} ms  {part * (n - 1) / ms / 1e6:.1f} GB/s per GPU out")


if __name__ == "__main__":
    main()
