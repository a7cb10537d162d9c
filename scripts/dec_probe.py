"""Decompress cold/warm decomposition vs plain memset/copy kernels (development aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402
from scripts.graph_timing import graph_time  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
    for shape in [(64, 2048, 7, 7), (64, 512, 28, 28), (64, 256, 56, 56)]:
        x = torch.randn(shape, device=dev).reshape(-1)
        d = x.numel()
        for r in (10, 1000):
            k = P.select_k(d, r)
            st = torch.cuda.current_stream().cuda_stream
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
            wsb = L.gp_topk_workspace_bytes(d, 0)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            L.gp_workspace_init(ws.data_ptr(), wsb, st)
            out = torch.empty(d, dtype=torch.float32, device=dev)
            out2 = torch.empty(d, dtype=torch.float32, device=dev)
            err = torch.zeros(1, dtype=torch.int32, device=dev)

            def fl():
                flush.sum()

            def comp():
                L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb,
                                         torch.cuda.current_stream().cuda_stream)

            def dec():
                L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream)

            def zero():
                out2.zero_()

            def copy():
                out2.copy_(x)

            comp()
            t_fl = graph_time([fl])
            res = {
                "fl+dec": graph_time([fl, dec]) - t_fl,
                "fl+comp+dec - fl+comp": graph_time([fl, comp, dec]) - graph_time([fl, comp]),
                "dec warm": graph_time([dec]),
                "fl+zero": graph_time([fl, zero]) - t_fl,
                "zero warm": graph_time([zero]),
                "fl+copy": graph_time([fl, copy]) - t_fl,
                "comp+zero - comp": graph_time([comp, zero]) - graph_time([comp]),
            }
            print(f"{str(shape):20s} r={r:5d} " + "  ".join(f"{k_}={v:6.2f}" for k_, v in res.items()), flush=True)


if __name__ == "__main__":
    main()
