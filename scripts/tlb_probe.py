"""What makes writes right after the 512 MB L2 flush slow?  Times a 25 MB zero_ and the C1 decompress
(1) right after the flush, (2) after the flush plus a one-element-per-2-MB read of the output buffer
(warms the TLB, moves ~13 sectors), (3) with no flush.  Development probe."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_12707_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
sp = torch.cuda.current_stream().cuda_stream
d = 8 * 1024 * 768
k = d // 100
x = torch.randn(d, device=dev)
frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
wsb = L.gp_topk_workspace_bytes(d, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
L.gp_workspace_init(ws.data_ptr(), wsb, sp)
L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, sp)
out = torch.empty(d, device=dev)
err = torch.zeros(1, dtype=torch.int32, device=dev)
flush = torch.ones(128 << 20, device=dev)
stride = (2 << 20) // 4
probe = torch.empty(out[::stride].numel(), device=dev)


def timed(fn, pre):
    ts = []
    for i in range(23):
        pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


def dec():
    L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 2, err.data_ptr(), sp)


for name, fn in (("zero_ 25 MB", lambda: out.zero_()), ("C1 decompress", dec)):
    a = timed(fn, lambda: flush.sum())
    b = timed(fn, lambda: (flush.sum(), probe.copy_(out[::stride])))
    c = timed(fn, lambda: None)
    print(f"{name:14s} after flush {a:6.2f} us | flush + TLB touch {b:6.2f} us | no flush {c:6.2f} us", flush=True)
