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
