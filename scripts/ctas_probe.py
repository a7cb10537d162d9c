"""C1-class compress latency vs cooperative grid size (CUDA graphs, L2 flushed)."""
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
    for shape in [(262144,), (1048576,), (4194304,), (8, 1024, 768)]:
        x = torch.randn(shape, device=dev).reshape(-1)
        d = x.numel()
        k = P.select_k(d, 100)
        frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
        wsb = L.gp_topk_workspace_bytes(d, 0)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        L.gp_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
        res = []
        t0 = graph_time([lambda: flush.sum()])
        for ctas in (8, 16, 32, 64, 148):
            def comp(c=ctas):
                L.gp_topk_compress_frame_ctas(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb,
                                              torch.cuda.current_stream().cuda_stream, c)
            t = graph_time([lambda: flush.sum(), comp]) - t0
            res.append(f"{ctas}:{t:6.2f}")
        print(f"d={d:9d} ({d * 4 / 2**20:5.1f} MB) compress us by CTAs  " + "  ".join(res), flush=True)


if __name__ == "__main__":
    main()
