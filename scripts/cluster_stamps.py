"""Per-phase timestamps of the single-cluster compress (gp_cluster.cu CL_STAMP
slots: 0 start, 1 loaded, 2+3p / 3+3p / 4+3p = radix pass p histogrammed /
past its cluster barrier / digit found, 20 counted, 21 past the count
barrier, 22 written), CTA 0 and the max over CTAs, after a 512 MB L2 flush."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
L = _lib.lib()
L.gp_debug_stamps.argtypes = [ctypes.c_void_p]
L.gp_debug_stamps.restype = None
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
dbg = torch.zeros(1024 * 32, dtype=torch.int64, device=dev)
for dt, d, r in (("fp32", 16384, 100), ("fp32", 262144, 100), ("fp32", 786432, 100), ("fp32", 786432, 10),
                 ("bf16", 1572864, 100)):
    x = torch.randn(d, device=dev)
    code = 0
    if dt == "bf16":
        x, code = x.bfloat16(), 1
    k = P.select_k(d, r)
    frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
    wsb = L.gp_topk_workspace_bytes(d, code)
    ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    for it in range(3):
        dbg.zero_()
        flush.sum()
        L.gp_debug_stamps(dbg.data_ptr())
        assert L.gp_topk_compress_frame(x.data_ptr(), code, d, k, frame.data_ptr(), ws.data_ptr(), wsb, s) == 0
        L.gp_debug_stamps(None)
        torch.cuda.synchronize()
    st = dbg.view(1024, 32).cpu()
    ncta = int((st[:, 0] != 0).sum())
    t0 = int(st[:ncta, 0].min())
    slots = [i for i in range(32) if int(st[0, i]) != 0]
    row = " ".join(f"{i}:{(int(st[0, i]) - t0) / 1e3:.2f}/{(int(st[:ncta, i].max()) - t0) / 1e3:.2f}" for i in slots)
    print(f"{dt} d={d} r={r} ctas={ncta} | slot:cta0/max us | {row}", flush=True)
