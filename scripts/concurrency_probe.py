"""Two independent compresses: sequential at full grid vs concurrent at half grid on two streams (graphs)."""
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
    s_main = torch.cuda.current_stream()
    side = [torch.cuda.Stream(dev) for _ in range(3)]
    for shape in [(64, 2048, 7, 7), (64, 1024, 14, 14), (64, 512, 28, 28), (64, 256, 56, 56)]:
        for r in (10, 100, 1000):
            n = 4
            xs = [torch.relu(torch.randn(shape, device=dev)).reshape(-1) for _ in range(n)]
            d = xs[0].numel()
            k = P.select_k(d, r)
            frames = [torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev) for _ in range(n)]
            wsb = L.gp_topk_workspace_bytes(d, 0)
            wss = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(n)]
            for ws in wss:
                L.gp_workspace_init(ws.data_ptr(), wsb, s_main.cuda_stream)

            def comp(i, ctas):
                st = torch.cuda.current_stream().cuda_stream
                assert L.gp_topk_compress_frame_ctas(xs[i].data_ptr(), 0, d, k, frames[i].data_ptr(),
                                                     wss[i].data_ptr(), wsb, st, ctas) == 0

            def fl():
                flush.sum()

            def run(nstreams, ctas):  # 4 compresses over nstreams streams
                def f():
                    cur = torch.cuda.current_stream()
                    for s in side:
                        s.wait_stream(cur)
                    for i in range(n):
                        j = i % nstreams
                        if j == 0:
                            comp(i, ctas)
                        else:
                            with torch.cuda.stream(side[j - 1]):
                                comp(i, ctas)
                    for s in side:
                        cur.wait_stream(s)
                return f

            t0 = graph_time([fl])
            res = {"1x148": graph_time([fl, run(1, 0)]) - t0, "2x74": graph_time([fl, run(2, 74)]) - t0,
                   "3x49": graph_time([fl, run(3, 49)]) - t0, "4x37": graph_time([fl, run(4, 37)]) - t0}
            print(f"{str(shape):20s} r={r:5d} 4 compresses: " + "  ".join(f"{a}={b:7.2f}" for a, b in res.items()),
                  flush=True)


if __name__ == "__main__":
    main()
