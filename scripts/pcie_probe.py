"""Pinned host <-> device copy rates on this box (the ceiling of bench.py's e2e leg).

    python scripts/pcie_probe.py

96 MB pinned buffers (the bench's largest boundary is 205 MB): H2D alone, D2H
alone, and both directions at once on two streams.  Prints GB/s per case.
"""
import torch


def rate(fn, nbytes, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    n = 24 << 20  # 96 MB of fp32
    h_in = torch.empty(n, pin_memory=True).fill_(1.0)
    h_out = torch.empty(n, pin_memory=True)
    d_a = torch.empty(n, device="cuda")
    d_b = torch.ones(n, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def h2d():
        d_a.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_b, non_blocking=True)

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    print(f"H2D pinned  {rate(h2d, 4 * n):6.1f} GB/s")
    print(f"D2H pinned  {rate(d2h, 4 * n):6.1f} GB/s")
    print(f"both dirs   {rate(both, 8 * n):6.1f} GB/s total (each direction 4*n bytes)")
    # the e2e leg's blocking upload: x.to(device) from a pinned tensor
    print(f"H2D .to()   {rate(lambda: h_in.to('cuda'), 4 * n):6.1f} GB/s")


if __name__ == "__main__":
    main()
