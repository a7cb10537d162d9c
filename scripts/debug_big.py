import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import compressor_oracle as O
from paper_2410_12707_b200 import _lib
L = _lib.lib()
print("lib", _lib.LIB_PATH)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(33)
x = torch.randn(64, 256, 56, 56, device=dev, generator=g)
for kind in ("activation", "gradient"):
    xx = (torch.relu(x) if kind == "activation" else x * 1e-3).reshape(-1).contiguous()
    host = xx.cpu().numpy()
    d = xx.numel()
    for r in (10.0, 100.0, 1000.0):
        for ctas in (0, 37):
            k = max(1, int(np.floor(d / r)))
            wsb = L.gp_topk_workspace_bytes(d, 0)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            sp = torch.cuda.current_stream().cuda_stream
            L.gp_workspace_init(ws.data_ptr(), wsb, sp)
            frame = torch.empty(16 + 12 * k, dtype=torch.uint8, device=dev)
            assert L.gp_topk_compress_frame_ctas(xx.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, sp, ctas) == 0
            err = torch.zeros(1, dtype=torch.int32, device=dev)
            out = torch.empty(d, device=dev)
            L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(), sp)
            torch.cuda.synchronize()
            got = frame.cpu().numpy().tobytes()
            want = O.compress_frame(host, r, method="threshold")
            gi = np.frombuffer(got, dtype="<i8", count=k, offset=16)
            wi = np.frombuffer(want, dtype="<i8", count=k, offset=16)
            nd = int((gi != wi).sum())
            print(kind, r, ctas, "ws", wsb, "hdr", np.frombuffer(got[:16], "<u8").tolist(), "flag", int(err.item()),
                  "same" if got == want else f"DIFF idx_mismatch={nd} first={np.argmax(gi != wi) if nd else -1}", flush=True)
