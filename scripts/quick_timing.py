"""Quick CUDA-event timing of compress / decompress launches (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402


def time_fn(fn, reps=50, flush=None):
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    shapes = [("C1 gpt2-small 8x1024x768", (8, 1024, 768)), ("C3 gpt2-med 8x1024x1024", (8, 1024, 1024)),
              ("resnet 64x2048x7x7", (64, 2048, 7, 7)), ("resnet 64x256x56x56", (64, 256, 56, 56))]
    g = torch.Generator(device=dev).manual_seed(0)
    for name, shape in shapes:
        x = torch.randn(shape, device=dev, generator=g).reshape(-1)
        d = x.numel()
        for r in (10, 100, 1000):
            k = P.select_k(d, r)
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
            wsb = L.gp_topk_workspace_bytes(d, 0)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            L.gp_workspace_init(ws.data_ptr(), wsb, st)
            out = torch.empty(d, device=dev)
            err = torch.zeros(1, dtype=torch.int32, device=dev)

            def comp():
                assert L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, st) == 0

            def decomp():
                assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(), st) == 0

            for _ in range(3):
                comp()
                decomp()
            tc, tcb = time_fn(comp, flush=flush)
            td, tdb = time_fn(decomp, flush=flush)
            byts = d * 4 + k * 12
            print(f"{name:28s} r={r:5d} d={d:9d} k={k:8d} compress {tc:8.2f} us ({byts / tc / 1e3:7.1f} GB/s, best {tcb:7.2f})"
                  f"  decompress {td:8.2f} us ({byts / td / 1e3:7.1f} GB/s, best {tdb:7.2f})", flush=True)


if __name__ == "__main__":
    main()
