"""PeerRing copy-engine bandwidth across processes (CUDA IPC), 2+ ranks (development aid).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/peer_probe.py

Every rank copies into its successor's receive buffer at once (both directions
busy at N=2): one 256 MB copy; the bench step's 24 frames on 1 / 4 streams;
the same 24 frames in 8 MB pieces.  GB/s per rank = bytes / time, max over ranks.
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2410_12707_b200 import select_k  # noqa: E402
from paper_2410_12707_b200.peer import PeerRing  # noqa: E402

SHAPES = [(64, 256, 56, 56), (64, 512, 28, 28), (64, 1024, 14, 14), (64, 2048, 7, 7)]


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cpu = dist.new_group(backend="gloo")
    sizes = []
    for s in SHAPES:
        d = 1
        for v in s:
            d *= v
        for _ in range(2):
            for r in (10, 100, 1000):
                sizes.append(16 + 12 * select_k(d, r))
    sizes.sort(reverse=True)
    total = sum(sizes)
    cap = max(total, 256 << 20) + 4096 * len(sizes)
    ring = PeerRing(cap, dev, cpu)
    src = torch.empty(cap, dtype=torch.uint8, device=dev)
    streams = [torch.cuda.Stream(dev) for _ in range(8)]

    def timed(plan, n_streams, reps=5):
        """plan: list of (offset, nbytes); copies round-robin over n_streams."""
        best = 1e30
        for _ in range(reps):
            dist.barrier()
            torch.cuda.synchronize()
            cur = torch.cuda.current_stream()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            for st in streams[:n_streams]:
                st.wait_stream(cur)
            for i, (off, nb) in enumerate(plan):
                ring.copy(ring.peer_recv(0) + off, src.data_ptr() + off, nb, streams[i % n_streams])
            for st in streams[:n_streams]:
                cur.wait_stream(st)
            b.record(cur)
            b.synchronize()
            t = torch.tensor([a.elapsed_time(b)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = min(best, float(t.item()))
        nbytes = sum(nb for _, nb in plan)
        return nbytes / (best * 1e-3) / 1e9, best

    frames, off = [], 0
    for nb in sizes:
        frames.append((off, nb))
        off += (nb + 255) // 256 * 256
    pieces = []
    for o, nb in frames:
        for p in range(0, nb, 8 << 20):
            pieces.append((o + p, min(8 << 20, nb - p)))
    rows = [("one 256 MB copy, 1 stream", [(0, 256 << 20)], 1),
            ("one 256 MB copy as 4 x 64 MB, 4 streams", [(i * (64 << 20), 64 << 20) for i in range(4)], 4),
            (f"24 frames ({total / 1e6:.0f} MB), 1 stream", frames, 1),
            ("24 frames, 4 streams", frames, 4),
            ("24 frames in 8 MB pieces, 1 stream", pieces, 1),
            ("24 frames in 8 MB pieces, 4 streams", pieces, 4)]
    for name, plan, ns in rows:
        gbs, ms = timed(plan, ns)
        if rank == 0:
            print(f"{name:45s} {gbs:7.1f} GB/s per rank ({ms:.3f} ms)", flush=True)
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
