"""Multi-rank message path (executor.py:207-297 restated over torch.distributed).

CPU: world_size-2 gloo processes exchange reference wire frames through
StageLink with an oracle codec — checks the protocol (frame sizing from
(d, ratio) alone, grouped send/recv in a ring, pass-through at ratio <= 1).
GPU (-m gpu, >= 2 devices): the same exchange over NCCL with the sm_100a codec,
checked bit-exactly against the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

from oracle import compressor_oracle as O
from paper_2410_12707_b200 import transport as T
from paper_2410_12707_b200.compressor import CompressionPlan


class OracleCodec:
    """CPU codec producing the reference frame with the oracle (test only)."""

    def compress(self, x, ratio, frame=None):
        f = torch.frombuffer(bytearray(O.compress_frame(x.reshape(-1).numpy(), ratio)), dtype=torch.uint8)
        if frame is not None:
            frame.copy_(f)
            return frame
        return f

    def decompress(self, frame, out, ratio):
        vals, idx, d = O.from_bytes(frame.numpy().tobytes())
        out.reshape(-1).copy_(torch.from_numpy(O.topk_decompress(vals.astype(np.float32), idx, d)))
        return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(rank, shapes):
    g = torch.Generator().manual_seed(100 + rank)
    return [torch.randn(s, generator=g) for s in shapes]


SHAPES = [(4, 33, 7), (1000,), (3, 512)]
RATIOS = [10.0, 1.0, 97.0]


def _ring_worker(rank, world, port, backend, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        if backend == "nccl":
            torch.cuda.set_device(rank)
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
            dev = torch.device("cuda", rank)
            link = T.StageLink(dev)
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
            dev = torch.device("cpu")
            link = T.StageLink(dev, codec=OracleCodec())
        xs = [x.to(dev) for x in _inputs(rank, SHAPES)]
        outs = [torch.empty(s, device=dev) for s in SHAPES]
        nxt, prv = (rank + 1) % world, (rank - 1) % world
        got = link.exchange([(x, r, nxt) for x, r in zip(xs, RATIOS)],
                            [(o, r, prv) for o, r in zip(outs, RATIOS)])
        # expected: the oracle applied to the previous rank's inputs
        src = _inputs(prv, SHAPES)
        ok = True
        for x, o, r in zip(src, got, RATIOS):
            flat = x.reshape(-1).numpy()
            if r <= 1.0:
                exp = flat
            else:
                vals, idx, d = O.topk_compress(flat, r)
                exp = O.topk_decompress(vals, idx, d)
            ok &= np.array_equal(o.reshape(-1).cpu().numpy().view(np.uint32), exp.view(np.uint32))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, bool(ok)))
    except Exception as e:  # surface failures to the parent
        q.put((rank, repr(e)))


def _run(world, backend):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ring_worker, args=(r, world, port, backend, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    return res


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ring_exchange_gloo(world):
    """Every rank sends to rank+1 and receives from rank-1 in one grouped
    exchange: world 2, 4 and 8 (the 8-stage pipeline's link count)."""
    res = _run(world, "gloo")
    assert res == {r: True for r in range(world)}, res


def _corrupt_worker(rank, world, port, q):
    """A received frame whose header disagrees with the receiver's (d, k), or
    whose index leaves [0, d), raises at the end of the exchange."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = torch.empty(1000)
        got = []
        for case in ("header", "index"):
            if rank == 0:
                frame = bytearray(O.compress_frame(np.arange(1000, dtype=np.float32), 10.0))
                if case == "header":
                    frame[8:16] = (50).to_bytes(8, "little")  # k = 50, the receiver expects 100
                else:
                    frame[16:24] = (5000).to_bytes(8, "little")  # index 5000 >= d
                dist.send(torch.frombuffer(frame, dtype=torch.uint8), 1)
            else:
                buf = torch.empty(T.frame_bytes(1000, 10.0), dtype=torch.uint8)
                dist.recv(buf, 0)
                try:
                    CheckingOracleCodec().decompress(buf, out, 10.0)
                    got.append("no error")
                except (ValueError, O.IndexOutOfRange) as e:
                    got.append(type(e).__name__)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, got))
    except Exception as e:
        q.put((rank, repr(e)))


class CheckingOracleCodec(OracleCodec):
    """The oracle codec with the receiver-side frame checks the device codec does."""

    def decompress(self, frame, out, ratio):
        d, k = out.numel(), O.select_k(out.numel(), ratio)
        hd, hk = (int(v) for v in np.frombuffer(frame.numpy().tobytes()[:16], dtype="<u8"))
        if (hd, hk) != (d, k):
            raise ValueError(f"frame header {(hd, hk)} != receiver's {(d, k)}")
        return super().decompress(frame, out, ratio)


def test_corrupted_frame_raises_gloo():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_corrupt_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res[1] == ["ValueError", "IndexOutOfRange"], res


def test_frame_bytes_and_passthrough():
    assert T.frame_bytes(100, 100) == 16 + 12
    assert T.frame_bytes(6291456, 100) == 16 + 12 * 62914
    x = torch.randn(3, 4)
    payload, shape = T.maybe_compress(x, ("a", "b"), None)
    assert payload is x and shape is None
    plan = CompressionPlan(base_ratio=10, per_link={("a", "b"): 10.0})
    payload, shape = T.maybe_compress(x, ("b", "a"), plan)  # link not in plan -> ratio 1.0
    assert payload is x and shape is None
    assert T.maybe_decompress(x, None) is x


@pytest.mark.gpu
def test_ring_exchange_nccl_world2(cuda):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run under gpurun --gpus 2)")
    res = _run(2, "nccl")
    assert res == {0: True, 1: True}, res


def _peer_worker(rank, world, port, q, pull=False, shared=False):
    """Frames through PeerRing: push = copy engines into the successor's IPC
    buffer; pull = compress into the own exported buffer, the successor's
    decompress reads it over NVLink.  Event handoff either way.  `shared`: every
    rank on cuda:0 (CUDA IPC between processes of one GPU), gloo only."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import ctypes

        import paper_2410_12707_b200 as P
        from paper_2410_12707_b200 import _lib
        from paper_2410_12707_b200.peer import PeerRing

        dev = torch.device("cuda", 0 if shared else rank)
        torch.cuda.set_device(dev)
        if shared:
            dist.init_process_group("gloo", rank=rank, world_size=world)
            cpu = None
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
            cpu = dist.new_group(backend="gloo")
        L = _lib.lib()
        d, r = 300_007, 50.0
        k = P.select_k(d, r)
        fb = 16 + 12 * k
        ring = PeerRing(fb, dev, cpu, pull=pull)
        st = torch.cuda.current_stream(dev)
        cs = torch.cuda.Stream(dev)
        out = torch.empty(d, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        ok = True
        for rnd in range(4):  # both buffer parities, twice
            g = torch.Generator().manual_seed(1000 * rnd + rank)
            x = torch.randn(d, generator=g).to(dev)
            frame = torch.empty(fb, dtype=torch.uint8, device=dev)
            wsb = L.gp_topk_workspace_bytes(d, 0)
            ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
            if pull:  # the successor must be done with this parity before it is overwritten
                ring.wait_consumed(st)
            dst = ring.recv(rnd) if pull else frame.data_ptr()
            assert L.gp_topk_compress_frame(x.data_ptr(), 0, d, k, dst, ws.data_ptr(), wsb, st.cuda_stream) == 0
            if not pull:
                ring.wait_consumed(cs)
                done = torch.cuda.Event()
                done.record(st)
                cs.wait_event(done)
                ring.copy(ring.peer_recv(rnd), frame.data_ptr(), fb, cs)
                st.wait_stream(cs)
            ring.signal_sent(st)
            dist.barrier(group=cpu)
            ring.wait_sent(st)
            src = ring.peer_recv(rnd) if pull else ring.recv(rnd)
            assert L.gp_topk_decompress_frame(src, k, d, out.data_ptr(), 0, 0, err.data_ptr(), st.cuda_stream) == 0
            ring.signal_consumed(st)
            torch.cuda.synchronize(dev)
            prv = (rank - 1) % world
            src = torch.randn(d, generator=torch.Generator().manual_seed(1000 * rnd + prv)).numpy()
            vals, idx, _ = O.topk_compress(src, r)
            ok &= int(err.item()) == 0
            ok &= np.array_equal(out.cpu().numpy().view(np.uint32), O.topk_decompress(vals, idx, d).view(np.uint32))
        dist.barrier()
        ring.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok)))
    except Exception as e:
        q.put((rank, repr(e)))


@pytest.mark.gpu
@pytest.mark.parametrize("shared", [False, True], ids=["2gpu", "1gpu"])
@pytest.mark.parametrize("pull", [False, True], ids=["push", "pull"])
def test_peer_ring_world2(cuda, pull, shared):
    """2gpu: one rank per GPU over NVLink.  1gpu: both ranks on cuda:0 (two
    processes, CUDA IPC on one device): the same ring code, events and frame
    checks, runnable on a one-GPU box."""
    if not shared and torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run under gpurun --gpus 2)")
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_worker, args=(r, 2, port, q, pull, shared)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def _peer_frames_worker(rank, world, port, q, shared=False):
    """The bench's N>1 step shape: several frames per step pushed into the
    successor's buffer by the copy engines, each with its own interprocess
    event recorded inside a captured CUDA graph, and the successor's
    decompress graph -- on its own stream, overlapping the compress graph --
    waiting per frame.  Fresh data every step, so a frame decompressed before
    its copy landed (the same parity's frame of two steps earlier) is caught."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import paper_2410_12707_b200 as P
        from paper_2410_12707_b200 import _lib
        from paper_2410_12707_b200.peer import PeerRing

        dev = torch.device("cuda", 0 if shared else rank)
        torch.cuda.set_device(dev)
        if shared:
            dist.init_process_group("gloo", rank=rank, world_size=world)
            cpu = None
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
            cpu = dist.new_group(backend="gloo")
        L = _lib.lib()
        specs = [(200_003, 50.0), (350_011, 10.0), (120_007, 100.0)]
        ks = [P.select_k(d, r) for d, r in specs]
        fbs = [16 + 12 * k for k in ks]
        offs = [sum((fb + 255) // 256 * 256 for fb in fbs[:i]) for i in range(len(fbs))]
        ring = PeerRing(sum((fb + 255) // 256 * 256 for fb in fbs), dev, cpu)
        ring.enable_frame_events(len(specs), cpu)
        xs = [torch.empty(d, device=dev) for d, _ in specs]
        frames = [torch.empty(fb, dtype=torch.uint8, device=dev) for fb in fbs]
        outs = [torch.empty(d, device=dev) for d, _ in specs]
        wsb = max(L.gp_topk_workspace_bytes(d, 0) for d, _ in specs)
        ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
        L.gp_workspace_init(ws.data_ptr(), wsb, torch.cuda.current_stream(dev).cuda_stream)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        st, cs, sd, side = (torch.cuda.Stream(dev) for _ in range(4))

        def comp(par):
            cur = torch.cuda.current_stream(dev)
            cs.wait_stream(cur)
            for i, (d, _) in enumerate(specs):
                assert L.gp_topk_compress_frame(xs[i].data_ptr(), 0, d, ks[i], frames[i].data_ptr(), ws.data_ptr(),
                                                wsb, cur.cuda_stream) == 0
                done = torch.cuda.Event()
                done.record(cur)
                cs.wait_event(done)
                ring.copy(ring.peer_recv(par) + offs[i], frames[i].data_ptr(), fbs[i], cs)
                ring.signal_frame_sent(par, i, cs)
            cur.wait_stream(cs)

        def dec(par):
            cur = torch.cuda.current_stream(dev)
            for i, (d, _) in enumerate(specs[::-1]):  # not the send order
                i = len(specs) - 1 - i
                ring.wait_frame_sent(par, i, cur)
                assert L.gp_topk_decompress_frame(ring.recv(par) + offs[i], ks[i], specs[i][0], outs[i].data_ptr(),
                                                  0, 0, err.data_ptr(), cur.cuda_stream) == 0

        graphs = {}
        ok = True
        prv = (rank - 1) % world
        for step_no in range(8):
            par = step_no & 1
            st.wait_stream(sd)
            ring.wait_consumed(st)
            with torch.cuda.stream(st):
                for i, (d, _) in enumerate(specs):
                    xs[i].copy_(torch.randn(d, generator=torch.Generator().manual_seed(97 * step_no + 13 * i + rank)))
                if step_no < 2:  # eager first (kernel attributes), then capture this parity's graphs
                    comp(par)
                else:
                    graphs["c", par].replay()
            dist.barrier(group=cpu)
            with torch.cuda.stream(sd):
                if step_no < 2:
                    dec(par)
                else:
                    graphs["d", par].replay()
                ring.signal_consumed(sd)
            torch.cuda.synchronize(dev)
            for i, (d, r) in enumerate(specs):
                src = torch.randn(d, generator=torch.Generator().manual_seed(97 * step_no + 13 * i + prv)).numpy()
                vals, idx, _ = O.topk_compress(src, r)
                ok &= np.array_equal(outs[i].cpu().numpy().view(np.uint32), O.topk_decompress(vals, idx, d).view(np.uint32))
            ok &= int(err.item()) == 0
            if step_no < 2:
                side.wait_stream(st)
                for name, fn in (("c", comp), ("d", dec)):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=side):
                        fn(par)
                    graphs[name, par] = g
                torch.cuda.synchronize(dev)
                dist.barrier(group=cpu)
        dist.barrier()
        ring.close()
        dist.destroy_process_group()
        q.put((rank, bool(ok)))
    except Exception as e:
        q.put((rank, repr(e)))


@pytest.mark.gpu
@pytest.mark.parametrize("shared", [False, True], ids=["2gpu", "1gpu"])
def test_peer_ring_frame_events_in_graphs(cuda, shared):
    """Per-frame interprocess events recorded and waited on inside captured
    CUDA graphs, decompress overlapping the compress phase: every frame of
    every step equals the oracle's (bench.py's N>1 step, GP_BENCH_FRAME_HANDOFF)."""
    if not shared and torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (run under gpurun --gpus 2)")
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_peer_frames_worker, args=(r, 2, port, q, shared)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


def test_opdata_envelope_cpu():
    """The OpData envelope (opdag.py:67-86) ahead of every pipeline message:
    iteration, micro-batch, link, kind, compress_cfg and shape; a receiver
    expecting anything else raises."""
    f = T.envelope_fields(3, 5, 1, 2, T.KIND_GRADIENT, True, 1234, (2, 64, 128))
    assert f[:9] == [T.ENVELOPE_MAGIC, 3, 5, 1, 2, 1, 1, 1234, 3] and f[9:12] == [2, 64, 128]
    buf = torch.zeros(T.ENVELOPE_BYTES + 16, dtype=torch.uint8)
    T.write_envelope(buf, f)
    T.check_envelope(buf, f)
    with pytest.raises(ValueError, match="envelope"):
        T.check_envelope(buf, T.envelope_fields(3, 6, 1, 2, T.KIND_GRADIENT, True, 1234, (2, 64, 128)))
