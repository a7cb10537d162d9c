"""Is the C1 compress's cold penalty instruction fetch?  C1 (8x1024x768 fp32, r=100) compress after a
512 MB L2 flush, with and without a 1,000-element compress (same kernel code, negligible data) between
the flush and the timed launch.  Development probe."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_12707_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
sp = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn(8 * 1024 * 768, device=dev, generator=g)
t = torch.randn(1 << 16, device=dev, generator=g)
flush = torch.ones(128 << 20, device=dev)
d, k = x.numel(), x.numel() // 100
dt, kt = t.numel(), t.numel() // 100
frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
ft = torch.empty(16 + 12 * kt, dtype=torch.uint8, device=dev)
wsb = L.gp_topk_workspace_bytes(d, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
ws2 = torch.empty(wsb, dtype=torch.uint8, device=dev)
L.gp_workspace_init(ws.data_ptr(), wsb, sp)
L.gp_workspace_init(ws2.data_ptr(), wsb, sp)
for variant in ("flush", "flush+tiny", "flush", "flush+tiny"):
    ts = []
    for i in range(23):
        flush.sum()
        if variant == "flush+tiny":
            L.gp_topk_compress_frame(t.data_ptr(), 0, dt, kt, ft.data_ptr(), ws2.data_ptr(), wsb, sp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, sp)
        e1.record()
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{variant:12s} C1 compress {statistics.median(ts):6.2f} us", flush=True)
