"""One mode-2 cluster compress of a 262,144-element fp32 vector at r = 100 (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
import paper_2410_12707_b200 as P  # noqa: E402
from paper_2410_12707_b200 import _lib  # noqa: E402

L = _lib.lib()
L.gp_set_cluster_path(2)
d = int(sys.argv[1]) if len(sys.argv) > 1 else 262_144
x = torch.randn(d, device="cuda")
for _ in range(3):
    p = P.topk_compress(x, 100.0)
torch.cuda.synchronize()
print("ok", p.values.numel())
