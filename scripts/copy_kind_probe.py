"""Are gp_copy_async device-to-device copies done by copy engines or by SM copy kernels?

    ncu --metrics gpu__time_duration.sum python scripts/copy_kind_probe.py

Copies 64 MB on GPU 0 (local) and GPU 0 -> GPU 1 (peer, if present) through
gp_copy_async, timing each with CUDA events; a copy done by an SM kernel shows
up in ncu's launch list, a copy-engine copy does not.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2410_12707_b200 import _lib  # noqa: E402


def timed(fn, nbytes, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    L = _lib.lib()
    n = 64 << 20
    a = torch.ones(n, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    s = torch.cuda.current_stream(0).cuda_stream
    print(f"local D2D   {timed(lambda: L.gp_copy_async(b.data_ptr(), a.data_ptr(), n, s), n):7.1f} GB/s", flush=True)
    if torch.cuda.device_count() > 1:
        torch.cuda.set_device(0)
        c = torch.empty(n, dtype=torch.uint8, device="cuda:1")
        try:
            torch.cuda.can_device_access_peer(0, 1)
            torch.zeros(1, device="cuda:1")
        except Exception as e:  # noqa: BLE001
            print("peer", e)
        print(f"peer 0->1   {timed(lambda: L.gp_copy_async(c.data_ptr(), a.data_ptr(), n, s), n):7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
