"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool).

* The `checked` library variant (-DGP_CHECKED: device-side bounds and
  invariant checks that trap with the failing condition) runs every kernel path
  of scripts/sanitize_cases.py in a subprocess; a trap fails the process.
* Guard canaries (memcheck's question): frames and outputs are carved out of
  larger buffers whose guard bytes around them must be untouched.
* Workspace state (initcheck's question): after every call the workspace's
  state region is zero again, as the C-ABI contract says.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2410_12707_b200 import _lib
from oracle import compressor_oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
CHECKED = ROOT / "paper_2410_12707_b200" / "_lib" / "variants" / "checked" / "libadatopk.so"
GUARD = 4096


def test_checked_build_runs_every_kernel_path(cuda):
    from paper_2410_12707_b200 import build

    build.build(out_dir=CHECKED.parent, defines=["-DGP_CHECKED"])  # incremental: rebuilds only if stale
    env = dict(os.environ, GP_LIB=str(CHECKED))
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "sanitize_cases.py"), "--small"], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ALL CASES OK" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
    assert "GP_CHECK failed" not in r.stdout + r.stderr


def _guarded(nbytes, device):
    buf = torch.full((nbytes + 2 * GUARD,), 0xA5, dtype=torch.uint8, device=device)
    return buf, buf[GUARD:GUARD + nbytes]


def _guards_intact(buf):
    return bool((buf[:GUARD] == 0xA5).all()) and bool((buf[-GUARD:] == 0xA5).all())


@pytest.mark.parametrize("ratio", [1.0, 3.0, 10.0, 100.0, 10000.0])
@pytest.mark.parametrize("d", [1, 33, 100_003, 3_000_017])
def test_guard_canaries_and_workspace_left_zeroed(cuda, d, ratio):
    L = _lib.lib()
    g = torch.Generator(device=cuda).manual_seed(d)
    x = torch.randn(d, device=cuda, generator=g)
    k = O.select_k(d, ratio)
    sp = torch.cuda.current_stream().cuda_stream
    wsb = L.gp_topk_workspace_bytes(d, 0)
    ws = torch.zeros(wsb, dtype=torch.uint8, device=cuda)
    fbuf, frame = _guarded(16 + 12 * k, cuda)
    obuf, outb = _guarded(4 * d, cuda)
    out = outb.view(torch.float32)
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    assert L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, frame.data_ptr(), ws.data_ptr(), wsb, sp) == 0
    assert L.gp_topk_decompress_frame(frame.data_ptr(), k, d, out.data_ptr(), 0, 0, err.data_ptr(), sp) == 0
    torch.cuda.synchronize()
    assert _guards_intact(fbuf) and _guards_intact(obuf)
    assert int(err.item()) == 0
    assert frame.cpu().numpy().tobytes() == O.compress_frame(x.cpu().numpy(), ratio, method="threshold")
    # the state region (everything the kernel must find zeroed) is zero again
    state = ws[:_state_bytes(wsb)]
    assert int(torch.count_nonzero(state)) == 0


def _state_bytes(wsb):
    """Extent of the workspace state region (gp_compress.cu workspace_state_bytes): control words,
    level histograms, fine histogram sized for the largest vector the buffer could hold."""
    def up(v):
        return (v + 255) & ~255
    n, fb = wsb // 8, 16
    while fb < 20 and (n >> (fb + 5)) != 0:
        fb += 1
    return up(256) + up(8 * 256 * 4) + up((1 << fb) * 4)
