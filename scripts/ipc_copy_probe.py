"""Copy-engine pushes into a peer's CUDA-IPC-mapped buffer (the bench's N>1 transport), two ranks.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ipc_copy_probe.py

Times, on every rank at once (both directions, as in the ring): one 256 MB copy; the same bytes
as 24 copies of the bench's frame sizes on 1 and 7 streams; a 256 MB copy from a buffer
allocated after the IPC mapping was opened.  Prints GB/s per direction on rank 0.
"""
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2410_12707_b200.peer import PeerRing  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    cpu = dist.new_group(backend="gloo")
    nb = 256 << 20
    early = torch.ones(nb, dtype=torch.uint8, device=dev)
    ring = PeerRing(nb, dev, cpu)
    late = torch.ones(nb, dtype=torch.uint8, device=dev)
    shapes = [(64, 256, 56, 56), (64, 512, 28, 28), (64, 1024, 14, 14), (64, 2048, 7, 7)]
    sizes = []
    for s in shapes:
        d = math.prod(s)
        for _ in range(2):
            for r in (10, 100, 1000):
                sizes.append(16 + 12 * (d // r))
    scale = nb / sum(sizes)
    sizes = [int(x * scale) // 256 * 256 for x in sizes]
    streams = [torch.cuda.Stream(dev) for _ in range(7)]
    cur = torch.cuda.current_stream(dev)

    def timed(fn):
        res = []
        for _ in range(4):
            dist.barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            for st in streams:
                st.wait_stream(cur)
            moved = fn()
            for st in streams:
                cur.wait_stream(st)
            e1.record(cur)
            e1.synchronize()
            res.append(moved / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        t = torch.tensor([min(res[1:])], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def one(src):
        ring.copy(ring.peer_recv(0), src.data_ptr(), nb, streams[0])
        return nb

    def frames(ns):
        def f():
            off, tot = 0, 0
            for i, sz in enumerate(sizes):
                ring.copy(ring.peer_recv(0) + off, early.data_ptr() + off, sz, streams[i % ns])
                off += sz
                tot += sz
            return tot
        return f

    srcs = [torch.ones(sz, dtype=torch.uint8, device=dev) for sz in sizes]
    # the same frames spread over a 12 GB footprint (the bench holds ~10 GB of inputs, outputs, workspaces)
    spread, fill = [], []
    for sz in sizes:
        spread.append(torch.ones(sz, dtype=torch.uint8, device=dev))
        fill.append(torch.empty(480 << 20, dtype=torch.uint8, device=dev))

    def frames_spread(ns):
        def f():
            off, tot = 0, 0
            for i, sz in enumerate(sizes):
                ring.copy(ring.peer_recv(0) + off, spread[i].data_ptr(), sz, streams[i % ns])
                off += sz
                tot += sz
            return tot
        return f

    def frames_sep(ns):
        def f():
            off, tot = 0, 0
            for i, sz in enumerate(sizes):
                ring.copy(ring.peer_recv(0) + off, srcs[i].data_ptr(), sz, streams[i % ns])
                off += sz
                tot += sz
            return tot
        return f

    out = {"one 256 MB copy (buffer allocated before the mapping)": timed(lambda: one(early)),
           "24 frame-sized copies from 24 separate tensors, 1 stream": timed(frames_sep(1)),
           "24 frame-sized copies from 24 separate tensors, 7 streams": timed(frames_sep(7)),
           "24 frames spread over 12 GB, 7 streams": timed(frames_spread(7)),
           "one 256 MB copy (buffer allocated after the mapping)": timed(lambda: one(late)),
           "24 frame-sized copies, 1 stream": timed(frames(1)),
           "24 frame-sized copies, 7 streams": timed(frames(7))}
    if rank == 0:
        for k, v in out.items():
            print(f"{k:55s} {v:7.1f} GB/s per direction", flush=True)
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
