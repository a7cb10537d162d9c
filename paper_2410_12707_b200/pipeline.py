"""GPT-2 pipeline training with AdaTopK-compressed stage boundaries.

The reference runs a GPipe fill-drain iteration on in-process workers
(pkg/src/geopipe/executor.py:376-411): every micro-batch forward, then every
micro-batch backward, messages compressed per cross-device link
(`_send_activation` :248-274, `_send_gradient` :276-297), then SGD.  Here each
stage is one GPU process (torch.distributed, NCCL); activations go forward and
gradients go backward as AdaTopK wire frames produced by the sm_100a kernels
(`transport.FrameCodec`), with per-link ratios from `adatopk_plan` (Eq. 6) or
`uniform_plan`.  Stage compute is plain PyTorch (bf16 autocast matmuls, fp32
residual stream, so boundary tensors are fp32).

The partition is OP-Fence's contiguous FLOP-proportional split
(opfence.py:285-315,412-424) of the operator chain [embeddings, blocks, LM
head] over identical devices, so the stage holding the head gets fewer blocks.  `virtual_stages` runs S stages inside one process (one GPU)
with the same compress/decompress at every boundary; it is used for the loss
parity test against the CPU oracle codec and as the N=1 point.
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field
from typing import Optional

import torch
import torch.distributed as dist
import torch.nn as nn
import torch.nn.functional as F

from .compressor import CompressionPlan, adatopk_plan, adatopk_plan_device, select_k, uniform_plan
from .transport import (ENVELOPE_BYTES, KIND_ACTIVATION, KIND_GRADIENT, FrameCodec, check_envelope, envelope_fields,
                        frame_bytes, write_envelope)

_P2P_BATCHED = os.environ.get("GP_P2P_BATCHED", "1") == "1"  # batched single-op P2P (0: plain isend/irecv)


@dataclass(frozen=True)
class GPT2Config:
    n_layer: int
    n_embd: int
    n_head: int
    vocab: int = 50257
    n_ctx: int = 1024


GPT2_SMALL = GPT2Config(12, 768, 12)
GPT2_MEDIUM = GPT2Config(24, 1024, 16)
GPT2_XL = GPT2Config(48, 1600, 25)
GPT2_TINY = GPT2Config(4, 128, 4, vocab=512, n_ctx=64)  # tests


class Block(nn.Module):
    def __init__(self, cfg: GPT2Config, sdpa: bool = True):
        super().__init__()
        h = cfg.n_embd
        self.n_head = cfg.n_head
        self.sdpa = sdpa
        self.ln1 = nn.LayerNorm(h)
        self.qkv = nn.Linear(h, 3 * h)
        self.proj = nn.Linear(h, h)
        self.ln2 = nn.LayerNorm(h)
        self.fc = nn.Linear(h, 4 * h)
        self.out = nn.Linear(4 * h, h)

    def forward(self, x):
        b, t, h = x.shape
        q, k, v = self.qkv(self.ln1(x)).split(h, dim=2)
        q, k, v = (z.view(b, t, self.n_head, h // self.n_head).transpose(1, 2) for z in (q, k, v))
        if self.sdpa:
            y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        else:  # deterministic path for parity tests
            att = (q @ k.transpose(-2, -1)) / math.sqrt(h // self.n_head)
            att = att.masked_fill(torch.ones(t, t, dtype=torch.bool, device=x.device).triu(1), float("-inf"))
            y = att.softmax(-1) @ v
        x = x + self.proj(y.transpose(1, 2).reshape(b, t, h))
        return x + self.out(F.gelu(self.fc(self.ln2(x)), approximate="tanh"))


class Stage(nn.Module):
    """Layers [a, b) of GPT-2, plus the embeddings (first) / final LN + head (last).

    Every module is initialised from a seed keyed by its layer, so the weights
    do not depend on the partition (as executor.py:161-178 keys parameters by
    op name, not placement).
    """

    def __init__(self, cfg: GPT2Config, a: int, b: int, first: bool, last: bool, sdpa: bool = True, seed: int = 0):
        super().__init__()
        self.first, self.last = first, last
        if first:
            torch.manual_seed(seed * 7919 + 1)
            self.wte = nn.Embedding(cfg.vocab, cfg.n_embd)
            self.wpe = nn.Embedding(cfg.n_ctx, cfg.n_embd)
        blocks = []
        for i in range(a, b):
            torch.manual_seed(seed * 7919 + 100 + i)
            blocks.append(Block(cfg, sdpa))
        self.blocks = nn.ModuleList(blocks)
        if last:
            torch.manual_seed(seed * 7919 + 2)
            self.ln_f = nn.LayerNorm(cfg.n_embd)
            # the head GEMM's N padded to a multiple of 64 (GPT-2's 50257 makes
            # the bf16 GEMM 11x slower on B200: 7.5 vs 0.66 ms, scripts/head_probe.py);
            # the extra logits are sliced off before the loss, so the model is unchanged
            self.vocab = cfg.vocab
            self.head = nn.Linear(cfg.n_embd, (cfg.vocab + 63) // 64 * 64, bias=False)

    def forward(self, x, targets=None):
        if self.first:
            pos = torch.arange(x.shape[1], device=x.device)
            x = self.wte(x) + self.wpe(pos)
        for blk in self.blocks:
            x = blk(x)
        if self.last:
            logits = self.head(self.ln_f(x))[..., :self.vocab].float()
            return F.cross_entropy(logits.reshape(-1, self.vocab), targets.reshape(-1))
        return x


def op_flops(cfg: GPT2Config) -> tuple:
    """Forward FLOPs per token of one transformer block and of the LM head (the
    per-operator workload estimate the split is weighted by): a block's four
    projections (12 h^2 weights, 2 FLOPs each) plus attention (4 T h); the head
    2 h V."""
    h = cfg.n_embd
    return 24.0 * h * h + 4.0 * cfg.n_ctx * h, 2.0 * h * cfg.vocab


def proportional_split(weights: list, n_blocks: int) -> list:
    """Contiguous split of items with `weights` into n_blocks blocks of ~equal
    load: OP-Fence's greedy rule (opfence.py:285-315, equal shares for identical
    devices).  Block j closes once its cumulative load reaches (j+1)/n of the
    total, or earlier when half of the next item's load would overshoot that
    target; every block gets at least one item.  Returns [start, end) pairs."""
    total = float(sum(weights))
    bounds, i, acc, n = [], 0, 0.0, len(weights)
    for j in range(n_blocks):
        target = total * (j + 1) / n_blocks
        start = i
        while i < n and n - i > n_blocks - j - 1:
            w = weights[i]
            if i > start and (acc >= target or (acc + w / 2.0 > target and j < n_blocks - 1)):
                break
            acc += w
            i += 1
        bounds.append((start, i))
    if i < n:  # the last block takes whatever is left
        bounds[-1] = (bounds[-1][0], n)
    return bounds


def partition(n_layer: int, n_stages: int, cfg: Optional[GPT2Config] = None):
    """Contiguous layer ranges [a, b) per stage.

    Without `cfg`: an equal split of the layer chain.  With `cfg`: OP-Fence's
    FLOP-proportional split (opfence.py:412-424) of the operator chain
    [embeddings, block 0 .. block n-1, LM head]: the head weighs several blocks
    (GPT-2 medium: 3.5), so the last stage gets fewer blocks.
    """
    if cfg is None:
        bounds = [round(i * n_layer / n_stages) for i in range(n_stages + 1)]
        return [(bounds[i], bounds[i + 1]) for i in range(n_stages)]
    blk, head = op_flops(cfg)
    weights = [1.0] + [blk] * n_layer + [head]  # item 0: embeddings (negligible FLOPs)
    out = []
    for a, b in proportional_split(weights, n_stages):
        # item i >= 1 is block i - 1; the embeddings and the head stay with stages 0 / S-1
        out.append((max(a - 1, 0) if a > 0 else 0, min(max(b - 1, 0), n_layer)))
    out[0] = (0, out[0][1])
    out[-1] = (out[-1][0], n_layer)
    return out


def make_stage(cfg: GPT2Config, s: int, n_stages: int, device, seed: int = 0, sdpa: bool = True) -> Stage:
    a, b = partition(cfg.n_layer, n_stages, cfg)[s]
    return Stage(cfg, a, b, s == 0, s == n_stages - 1, sdpa, seed).to(device)


def link_plan(n_stages: int, mode: str, ratio: float, link_times: Optional[list] = None) -> CompressionPlan:
    """Per-link ratios for the chain 0-1-...-(S-1), both directions.

    `mode` "adatopk": Eq. 6 over link communication times R (seconds), each FP
    link's R mirrored onto its BP link (the reference's CLI keys FP links only,
    SURVEY.md §7.10); "uniform": every link at `ratio`; "none": no plan.
    """
    if mode == "none" or n_stages < 2:
        return None
    links = [(s, s + 1) for s in range(n_stages - 1)] + [(s + 1, s) for s in range(n_stages - 1)]
    if mode == "uniform":
        return uniform_plan(links, ratio)
    R = {}
    for s in range(n_stages - 1):
        t = link_times[s] if link_times is not None else 1.0
        R[(s, s + 1)] = t
        R[(s + 1, s)] = t
    return adatopk_plan(None, R, ratio)


def two_cluster_link_times(n_stages: int, boundary_bytes: int, fast=(1e-5, 1 / 100e9), slow=(5e-3, 1 / 1.25e9)):
    """Simulated heterogeneous links (alpha + beta*M): two clusters of S/2
    stages, fast links inside, one slow link between them (the style of the
    reference's scenarios/fig7_clusters.json)."""
    mid = n_stages // 2 - 1
    return [(slow if s == mid else fast)[0] + (slow if s == mid else fast)[1] * boundary_bytes
            for s in range(n_stages - 1)]


def eq3_pipeline_time(C: list, R: list, n_b: int) -> float:
    """Eq. 3, planner.py:90-104: sum_d (C_d + R_d) + (n_b - 1) * max_d max(C_d, R_d)."""
    return sum(c + r for c, r in zip(C, R)) + (n_b - 1) * max(max(c, r) for c, r in zip(C, R))


def eq7_pipeline_time(C: list, R: list, n_b: int, base_ratio: float, r_dev: list,
                      scale_bottleneck_receive: bool = False) -> float:
    """Eq. 7, planner.py:113-147.  Published closed form: sum_d (C_d + 3 R_d / r_d)
    + 3 (n_b - 1) * max_d max(C_d, R_d) / r; with scale_bottleneck_receive the
    bubble is (n_b - 1) * max_d max(C_d, 3 R_d / r_d) (the reference's variant)."""
    front = sum(c + 3.0 * r / rd for c, r, rd in zip(C, R, r_dev))
    if scale_bottleneck_receive:
        return front + max(max(c, 3.0 * r / rd) for c, r, rd in zip(C, R, r_dev)) * (n_b - 1)
    return front + 3.0 * (n_b - 1) * max(max(c, r) for c, r in zip(C, R)) / base_ratio


def des_chain_fp_time(C: list, M: list, n_b: int) -> float:
    """FP makespan of a stage chain under the reference's discrete-event model
    (simulator.py:108-268, phases=("fp",)): one op at a time per device, one
    message in flight per directed link (FIFO: a send starts at max(producer
    finish, link free) and occupies the link for the message time), every FP
    task of micro-batch m on stage s after its input message arrives.  On a
    chain each device receives its tasks in micro-batch order, so the event loop
    reduces to this flow-shop recurrence.  C[s] = stage s's time per
    micro-batch, M[s] = the message time on the link into stage s (M[0]
    unused).  tests/test_pipeline.py checks it against the reference's
    `simulate` on random chains."""
    S = len(C)
    dev_free = [0.0] * S
    link_free = [0.0] * S
    makespan = 0.0
    for _ in range(n_b):
        finish = 0.0
        for s in range(S):
            ready = 0.0
            if s > 0:
                send = max(finish, link_free[s])
                link_free[s] = ready = send + M[s]
            finish = max(ready, dev_free[s]) + C[s]
            dev_free[s] = finish
        makespan = max(makespan, finish)
    return makespan


def measure_link_times(shape, device, reps: int = 5, chain: Optional[list] = None, as_tensor: bool = False):
    """Measured dense boundary transfer time (s) of every FP link, stage s -> s+1.

    Stage s runs on rank chain[s] (identity by default).  Each rank sends a
    dense boundary tensor to its successor stage while receiving from its
    predecessor (one batched NCCL group, so the links run at once, as in the
    pipeline); the receiver times its receive with CUDA events (median of
    `reps`).  An all-reduce gives every rank the same vector, so every rank
    derives the same per-link plan (both ends of a link agree on k).  This is
    R_i of Eq. 6 measured instead of the alpha-beta estimate of the reference
    CLI (cli.py:51-59).  `as_tensor`: return the float64
    CUDA tensor (no host copy) for an on-device plan.
    """
    rank, S = dist.get_rank(), dist.get_world_size()
    chain = list(chain) if chain is not None else list(range(S))
    s = chain.index(rank)
    x = torch.randn(shape, device=device)
    buf = torch.empty(shape, device=device)
    t = torch.zeros(max(S - 1, 1), dtype=torch.float64, device=device)
    samples = []
    for _ in range(reps + 1):
        dist.barrier()
        ops = []
        if s < S - 1:
            ops.append(dist.P2POp(dist.isend, x, chain[s + 1]))
        if s > 0:
            ops.append(dist.P2POp(dist.irecv, buf, chain[s - 1]))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        b.record()
        torch.cuda.synchronize()
        samples.append(a.elapsed_time(b) * 1e-3)
    if s > 0:
        samples = sorted(samples[1:])
        t[s - 1] = samples[len(samples) // 2]
    dist.all_reduce(t)
    return t if as_tensor else t.tolist()


def measured_link_plan(n_stages: int, ratio: float, link_times: list, boundary: int, device) -> CompressionPlan:
    """Eq. 6 on the device from measured link times (FP time mirrored onto BP)."""
    links = [(s, s + 1) for s in range(n_stages - 1)] + [(s + 1, s) for s in range(n_stages - 1)]
    R = torch.tensor(list(link_times) + list(link_times), dtype=torch.float64, device=device)
    dl = torch.full((len(links),), boundary, dtype=torch.int64, device=device)
    r, _k, status = adatopk_plan_device(R, ratio, dl)
    st = int(status.item())
    if st != 0:
        from .errors import raise_for_status
        raise_for_status(st, "gp_adatopk_plan")
    return CompressionPlan(base_ratio=ratio, per_link={lk: float(v) for lk, v in zip(links, r.tolist())})


@dataclass
class PipelineStats:
    step_ms: float = 0.0
    loss: float = float("nan")
    compress_calls: int = 0
    wire_bytes: int = 0
    dense_bytes: int = 0


def _amp(device):
    """bf16 autocast for the stage matmuls on a GPU; plain fp32 on CPU ranks (tests)."""
    if torch.device(device).type == "cuda":
        return torch.autocast("cuda", dtype=torch.bfloat16)
    import contextlib
    return contextlib.nullcontext()


class VirtualPipeline:
    """All S stages in one process/GPU, compressing at every boundary (fill-drain)."""

    def __init__(self, cfg: GPT2Config, n_stages: int, plan: Optional[CompressionPlan], device, codec=None,
                 lr: float = 1e-4, seed: int = 0, sdpa: bool = True):
        self.cfg, self.S, self.plan, self.device = cfg, n_stages, plan, device
        self.codec = codec if codec is not None else FrameCodec(device)
        self.stages = [make_stage(cfg, s, n_stages, device, seed, sdpa) for s in range(n_stages)]
        self.opts = [torch.optim.AdamW(st.parameters(), lr=lr) for st in self.stages]
        self.stats = PipelineStats()

    def _link(self, x: torch.Tensor, src: int, dst: int) -> torch.Tensor:
        r = self.plan.ratio_for(src, dst) if self.plan is not None else 1.0
        self.stats.dense_bytes += x.numel() * x.element_size()
        if r <= 1.0:
            self.stats.wire_bytes += x.numel() * x.element_size()
            return x.detach().clone()
        frame = self.codec.compress(x.detach().contiguous(), r)
        self.stats.compress_calls += 1
        self.stats.wire_bytes += frame.numel() - 16
        out = torch.empty_like(x)
        self.codec.decompress(frame, out, r)
        return out

    def step(self, tokens: torch.Tensor, targets: torch.Tensor, n_micro: int) -> float:
        S = self.S
        mbs = tokens.chunk(n_micro)
        tgs = targets.chunk(n_micro)
        acts = [[None] * S for _ in range(n_micro)]  # (input leaf, output) per stage
        losses = []
        for m in range(n_micro):  # fill: every micro-batch forward
            x = mbs[m]
            for s in range(S):
                inp = x if s == 0 else x.requires_grad_(True)
                with _amp(self.device):
                    y = self.stages[s](inp, tgs[m] if s == S - 1 else None)
                acts[m][s] = (inp, y)
                if s < S - 1:
                    x = self._link(y, s, s + 1)
            losses.append(y)
        for m in range(n_micro):  # drain: every micro-batch backward
            grad = None
            for s in range(S - 1, -1, -1):
                inp, y = acts[m][s]
                if s == S - 1:
                    (y / n_micro).backward()
                else:
                    y.backward(grad)
                if s > 0:
                    grad = self._link(inp.grad, s, s - 1)
        for o in self.opts:
            o.step()
            o.zero_grad(set_to_none=True)
        loss = float(torch.stack([l.detach() for l in losses]).mean())
        self.stats.loss = loss
        return loss


class DevicePlan:
    """Per-link k kept on the device (north_star item 4): Eq. 6 + select_k run
    in the plan kernel (gp_adatopk_plan) into `k`, a CUDA int64 tensor, and the
    compress kernels read their k from it, so re-planning every step needs no
    host round trip.  Frames are sized for a host-known capacity per link,
    `k_cap = select_k(d, ratio_floor)`; a planned k above it is clamped on the
    device (`clamped` counts such links, read whenever the caller syncs) --
    with measured NVSwitch links Eq. 6 gives every link r ~ 3r, far above the
    floor.  The receiver reads k from each frame's header."""

    def __init__(self, links: list, boundary: int, base_ratio: float, device, ratio_floor: Optional[float] = None):
        self.links = list(links)
        self.index = {lk: i for i, lk in enumerate(self.links)}
        self.boundary, self.base_ratio, self.device = int(boundary), float(base_ratio), device
        self.k_cap = select_k(self.boundary, ratio_floor if ratio_floor is not None else base_ratio)
        n = len(self.links)
        self.k = torch.full((n,), self.k_cap, dtype=torch.int64, device=device)
        self.r = torch.zeros(n, dtype=torch.float64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.clamped = torch.zeros(1, dtype=torch.int64, device=device)
        self._dl = torch.full((n,), self.boundary, dtype=torch.int64, device=device)

    def replan(self, R: torch.Tensor) -> None:
        """Eq. 6 from link times R (float64 CUDA tensor, one per link), stream-ordered, no host sync."""
        from .compressor import _lib, _stream_handle
        import ctypes

        P = ctypes.POINTER
        R = R.to(device=self.device, dtype=torch.float64).contiguous()
        st = _lib.lib().gp_adatopk_plan(
            ctypes.cast(R.data_ptr(), P(ctypes.c_double)), len(self.links), self.base_ratio,
            ctypes.cast(self._dl.data_ptr(), P(ctypes.c_int64)), ctypes.cast(self.r.data_ptr(), P(ctypes.c_double)),
            ctypes.cast(self.k.data_ptr(), P(ctypes.c_int64)), ctypes.cast(self.status.data_ptr(), P(ctypes.c_int32)),
            _stream_handle(self.device))
        if st != 0:
            from .errors import raise_for_status
            raise_for_status(st, "gp_adatopk_plan")
        self.clamped += (self.k > self.k_cap).sum()
        torch.clamp_(self.k, max=self.k_cap)

    def k_slot(self, link) -> torch.Tensor:
        i = self.index[link]
        return self.k[i:i + 1]


class _Timeline:
    """CUDA-event spans of one pipeline step on this rank, exported in the
    reference's Chrome trace format (simulator.py:75-95: complete "X" events,
    microseconds) so a measured step can be laid next to the simulated one."""

    def __init__(self):
        self.t0 = torch.cuda.Event(enable_timing=True)
        self.t0.record()
        self.spans = []

    def span(self, name: str, cat: str):
        tl = self

        class _Span:
            def __enter__(self):
                self.a = torch.cuda.Event(enable_timing=True)
                self.a.record()

            def __exit__(self, *exc):
                b = torch.cuda.Event(enable_timing=True)
                b.record()
                tl.spans.append((name, cat, self.a, b))
                return False

        return _Span()

    def events(self, pid, tid) -> list:
        torch.cuda.synchronize()
        return [{"name": n, "cat": c, "ph": "X", "ts": round(self.t0.elapsed_time(a) * 1e3, 3),
                 "dur": round(a.elapsed_time(b) * 1e3, 3), "pid": pid, "tid": tid} for n, c, a, b in self.spans]


class _NoSpan:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class _HostWork:
    """A gloo P2P request on a host staging buffer; `wait()` copies a received buffer to the device."""

    def __init__(self, work, host, dst=None):
        self.work, self.host, self.dst = work, host, dst

    def wait(self):
        self.work.wait()
        if self.dst is not None:
            self.dst.copy_(self.host)
        return True


class DistPipeline:
    """One stage per rank (torch.distributed); fill-drain with compressed P2P.

    `chain` maps pipeline stages to ranks (stage s runs on rank chain[s]; the
    default is the identity); the OP-Fence schedule supplies it as its
    device_chain (opfence.py:347-435).  `device` (default: the current CUDA
    device) and `codec` make the same fill-drain logic runnable on CPU ranks
    over gloo with a host codec, which the multi-rank CPU tests use.  With a
    `dev_plan` the boundaries use device-resident k (DevicePlan).  The codec's
    validation flag is read once at the end of every step.
    """

    def __init__(self, cfg: GPT2Config, plan: Optional[CompressionPlan], micro_batch: int, seq_len: int,
                 lr: float = 1e-4, seed: int = 0, chain: Optional[list] = None, device=None, codec=None,
                 dev_plan: Optional[DevicePlan] = None, bounds: Optional[list] = None, sdpa: bool = True):
        self.rank, self.S = dist.get_rank(), dist.get_world_size()
        self.chain = list(chain) if chain is not None else list(range(self.S))
        if sorted(self.chain) != list(range(self.S)):
            raise ValueError(f"chain {self.chain} is not a permutation of the {self.S} ranks")
        self.s = self.chain.index(self.rank)  # this rank's stage
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cfg, self.plan, self.mb, self.T = cfg, plan, micro_batch, seq_len
        self.dev_plan = dev_plan
        if bounds is None:
            self.stage = make_stage(cfg, self.s, self.S, self.device, seed, sdpa)
        else:
            a, b = bounds[self.s]
            self.stage = Stage(cfg, a, b, self.s == 0, self.s == self.S - 1, sdpa, seed).to(self.device)
        self.opt = torch.optim.AdamW(self.stage.parameters(), lr=lr)
        self.codec = codec if codec is not None else FrameCodec(self.device)
        self.shape = (micro_batch, seq_len, cfg.n_embd)
        self.step_no = 0    # the iteration in every message envelope (OpData.local_iter)
        # device flag of the envelope checks: the codec's own (read by its check()), or, for a codec
        # without one (host baselines), the pipeline's
        self._err = getattr(self.codec, "err", None)
        if self._err is None and self.device.type == "cuda":
            self._err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.messages = []  # (direction, src_stage, dst_stage, micro_batch) in send order (tests)

    def _amp(self):
        return _amp(self.device)

    def _ratio(self, src, dst):
        return self.plan.ratio_for(src, dst) if self.plan is not None else 1.0

    def _p2p(self, op, buf, peer_stage):
        peer = self.chain[peer_stage]
        if self.device.type == "cuda" and dist.get_backend() == "gloo":
            # CUDA tensors over gloo (several ranks sharing one GPU in the
            # tests): the frame is staged through host memory
            if op is dist.isend:
                h = buf.cpu()
                return _HostWork(dist.isend(h, peer), h)
            h = torch.empty(buf.shape, dtype=buf.dtype)
            return _HostWork(dist.irecv(h, peer), h, buf)
        if _P2P_BATCHED and self.device.type == "cuda":
            return dist.batch_isend_irecv([dist.P2POp(op, buf, peer)])[0]
        return op(buf, peer)

    def _payload_bytes(self, link) -> tuple:
        """(compressed, payload bytes) of a message on `link` (the receiver sizes its buffer from these)."""
        d = math.prod(self.shape)
        if self.dev_plan is not None and link in self.dev_plan.index:
            return True, 16 + 12 * self.dev_plan.k_cap
        r = self._ratio(*link)
        return (False, 4 * d) if r <= 1.0 else (True, frame_bytes(d, r))

    def _send(self, x: torch.Tensor, dst: int, m: int, kind: int):
        """Send stage self.s's tensor to stage dst (link keys are stage indices) as one
        buffer: the OpData envelope (transport.envelope_fields), then the payload --
        a reference wire frame written in place by the compress kernel, or the dense
        tensor (ratio <= 1, executor.py:210-212)."""
        link = (self.s, dst)
        x = x.detach().contiguous()
        compressed, nbytes = self._payload_bytes(link)
        buf = torch.empty(ENVELOPE_BYTES + nbytes, dtype=torch.uint8, device=self.device)
        write_envelope(buf, envelope_fields(self.step_no, m, self.s, dst, kind, compressed, nbytes, x.shape))
        body = buf[ENVELOPE_BYTES:]
        if self.dev_plan is not None and link in self.dev_plan.index:
            self.codec.compress_dk(x, self.dev_plan.k_slot(link), self.dev_plan.k_cap, frame=body)
        elif compressed:
            self.codec.compress(x, self._ratio(*link), frame=body)
        else:
            body.view(x.dtype).copy_(x.reshape(-1))
        return self._p2p(dist.isend, buf, dst), buf

    def _recv(self, src: int, m: int, kind: int) -> torch.Tensor:
        link = (src, self.s)
        out = torch.empty(self.shape, device=self.device)
        compressed, nbytes = self._payload_bytes(link)
        buf = torch.empty(ENVELOPE_BYTES + nbytes, dtype=torch.uint8, device=self.device)
        self._p2p(dist.irecv, buf, src).wait()
        # the envelope the sender must have written for this (iteration, micro-batch, link, kind)
        check_envelope(buf, envelope_fields(self.step_no, m, src, self.s, kind, compressed, nbytes, self.shape),
                       self._err)
        body = buf[ENVELOPE_BYTES:]
        if self.dev_plan is not None and link in self.dev_plan.index:
            return self.codec.decompress_dk(body, out, self.dev_plan.k_cap)
        if not compressed:
            out.reshape(-1).copy_(body.view(out.dtype))
            return out
        return self.codec.decompress(body, out, self._ratio(*link))

    def forward_only(self, tokens: torch.Tensor, targets: torch.Tensor, n_micro: int):
        """The FP half of a step (fill phase, no backward): what Eq. 3 / Eq. 7 model."""
        s, S = self.s, self.S
        mbs, tgs = tokens.chunk(n_micro), targets.chunk(n_micro)
        pending = []
        with torch.no_grad():
            for m in range(n_micro):
                inp = mbs[m] if s == 0 else self._recv(s - 1, m, KIND_ACTIVATION)
                with self._amp():
                    y = self.stage(inp, tgs[m] if s == S - 1 else None)
                if s < S - 1:
                    pending.append(self._send(y, s + 1, m, KIND_ACTIVATION))
        for w, _buf in pending:
            w.wait()
        self.step_no += 1

    def stage_fp_time(self, tokens: torch.Tensor, targets: torch.Tensor, reps: int = 5) -> float:
        """C_d: this stage's forward time for one micro-batch (s, CUDA events, median)."""
        x = tokens[: self.mb] if self.s == 0 else torch.randn(self.shape, device=self.device)
        tg = targets[: self.mb] if self.s == self.S - 1 else None
        ts = []
        with torch.no_grad():
            for _ in range(reps + 1):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                with self._amp():
                    self.stage(x, tg)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e-3)
        ts = sorted(ts[1:])
        return ts[len(ts) // 2]

    def step(self, tokens: torch.Tensor, targets: torch.Tensor, n_micro: int, check: bool = True,
             trace: bool = False):
        """One GPipe fill-drain iteration (executor.py:376-411): every micro-batch
        forward (activations to the next stage, _send_activation :248-274), then
        every micro-batch backward (gradients to the previous stage,
        _send_gradient :276-297), then the optimizer step.  `trace=True` keeps
        this step's CUDA-event spans in `self.last_trace` (Chrome trace events,
        pid = stage)."""
        s, S = self.s, self.S
        mbs, tgs = tokens.chunk(n_micro), targets.chunk(n_micro)
        pending, saved, losses = [], [], []
        tl = _Timeline() if trace and self.device.type == "cuda" else None

        def span(name, cat):
            return tl.span(name, cat) if tl is not None else _NoSpan()

        for m in range(n_micro):  # fill
            with span(f"recv act mb{m}", "recv"):
                inp = mbs[m] if s == 0 else self._recv(s - 1, m, KIND_ACTIVATION).requires_grad_(True)
            with span(f"stage{s} mb{m}", "fp"), self._amp():
                y = self.stage(inp, tgs[m] if s == S - 1 else None)
            saved.append((inp, y))
            if s < S - 1:
                with span(f"{s}->{s + 1} mb{m}", "send"):
                    pending.append(self._send(y, s + 1, m, KIND_ACTIVATION))
                self.messages.append(("fp", s, s + 1, m))
            else:
                losses.append(y.detach())
        for m in range(n_micro):  # drain
            inp, y = saved[m]
            if s == S - 1:
                with span(f"stage{s} mb{m}", "bp"):
                    (y / n_micro).backward()
            else:
                with span(f"recv grad mb{m}", "recv"):
                    g = self._recv(s + 1, m, KIND_GRADIENT)
                with span(f"stage{s} mb{m}", "bp"):
                    y.backward(g)
            if s > 0:
                with span(f"{s}->{s - 1} mb{m}", "send"):
                    pending.append(self._send(inp.grad, s - 1, m, KIND_GRADIENT))
                self.messages.append(("bp", s, s - 1, m))
        for w, _buf in pending:
            w.wait()
        with span(f"stage{s} optimizer", "opt"):
            self.opt.step()
            self.opt.zero_grad(set_to_none=True)
        if tl is not None:
            self.last_trace = tl.events(pid=s, tid=f"stage{s} (rank {self.rank})")
        loss = torch.stack(losses).mean() if losses else torch.zeros((), device=self.device)
        dist.broadcast(loss, self.chain[S - 1])
        self.step_no += 1
        if check and self.dev_plan is not None:
            st = int(self.dev_plan.status.item())  # the on-device Eq. 6's status (InvalidRatio / NoCommunication)
            if st:
                from .errors import raise_for_status
                raise_for_status(st, "gp_adatopk_plan")
        if check and hasattr(self.codec, "check"):
            self.codec.check()  # one flag read per step: a corrupt received frame raises here
        elif check and self._err is not None and int(self._err.item()):
            self._err.zero_()
            raise ValueError("a received message's OpData envelope differs from the receiver's expectation")
        return float(loss)


MODELS = {"small": GPT2_SMALL, "medium": GPT2_MEDIUM, "xl": GPT2_XL}


def gather_chrome_trace(pipe: "DistPipeline") -> Optional[str]:
    """Every rank's `last_trace` in one Chrome trace (the reference's format,
    simulator.py:75-95); returned on every rank.  Ranks start their step clocks
    at the barrier before the traced step, so the stages line up to within the
    barrier's skew."""
    import json

    mine = getattr(pipe, "last_trace", [])
    allv = [None] * dist.get_world_size()
    dist.all_gather_object(allv, mine)
    events = [e for v in allv for e in (v or [])]
    return json.dumps({"traceEvents": events, "displayTimeUnit": "ms"}, sort_keys=True)


def _stage_links(S: int) -> list:
    return [(s, s + 1) for s in range(S - 1)] + [(s + 1, s) for s in range(S - 1)]


def run_pipeline(model: str = "medium", plan_mode: str = "uniform", ratio: float = 100.0, micro_batch: int = None,
                 n_micro: int = None, seq_len: int = 1024, steps: int = 3, warmup: int = 1, codec=None,
                 codec_name: str = "sm_100a FrameCodec", trace_path=None) -> dict:
    """Time GPipe steps of GPT-2 with one stage per rank (or one stage on one GPU).

    plan_mode:
      "uniform"  every FP/BP link at `ratio` (uniform_plan, compressor.py:132-139);
      "measured" link times measured on the NVLink fabric, Eq. 6 + select_k on the
                 device (DevicePlan): the compress kernels read k from device
                 memory, the receivers read it from the frame headers;
      "adatopk"  configs[3]: the reference's unchanged OP-Fence schedule over a
                 simulated two-cluster network (opfence_plan) gives the stage ->
                 GPU chain and the block ranges, the reference CLI's
                 cross_link_times gives R_i (mirrored onto BP links), and Eq. 6
                 (adatopk_plan) the per-link ratios.
    Returns samples/s = global batch / median step time (CUDA events, each step
    the max over ranks) after `warmup` untimed steps.  Call after
    torch.distributed is initialised when WORLD_SIZE > 1.
    """
    cfg = MODELS[model]
    mb = micro_batch or (8 if model != "xl" else 4)
    world = dist.get_world_size() if dist.is_initialized() else 1
    n_micro = n_micro or max(4, 2 * world)
    dev = torch.device("cuda", torch.cuda.current_device())
    boundary = mb * seq_len * cfg.n_embd
    lt, chain, bounds, dev_plan, plan, ofp = None, None, None, None, None, None
    if world > 1 and plan_mode == "measured":
        R = measure_link_times((mb, seq_len, cfg.n_embd), dev, as_tensor=True)
        dev_plan = DevicePlan(_stage_links(world), boundary, ratio, dev)
        dev_plan.replan(torch.cat([R, R]))  # FP time mirrored onto the BP link
    elif world > 1 and plan_mode == "adatopk":
        from .opfence_plan import opfence_partition

        ofp = opfence_partition(cfg.n_layer, cfg.n_embd, cfg.vocab, world, mb, seq_len, n_micro)
        chain, bounds = ofp.chain, ofp.bounds
        plan = adatopk_plan(None, dict(ofp.link_R), ratio)
        lt = [ofp.link_R[(s, s + 1)] for s in range(world - 1)]
    elif world > 1:
        plan = link_plan(world, plan_mode, ratio, None)
    if world > 1:
        pipe = DistPipeline(cfg, plan, mb, seq_len, chain=chain, bounds=bounds, dev_plan=dev_plan, codec=codec)
    else:
        pipe = VirtualPipeline(cfg, 1, None, dev)
    gb = mb * n_micro
    times, loss = [], float("nan")
    for i in range(warmup + steps):
        tok, tgt = synthetic_batch(cfg, gb, seq_len, dev, seed=i)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        loss = pipe.step(tok, tgt, n_micro)
        b.record()
        torch.cuda.synchronize()
        if i >= warmup:
            times.append(a.elapsed_time(b))
    if world > 1:  # per step, the slowest rank
        tt = torch.tensor(times, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        times = tt.tolist()
    t = sorted(times)[len(times) // 2]  # median step
    trace_file = None
    if trace_path and world > 1:  # one more step with CUDA-event spans, as a Chrome trace
        tok, tgt = synthetic_batch(cfg, gb, seq_len, dev, seed=warmup + steps)
        dist.barrier()
        torch.cuda.synchronize()
        pipe.step(tok, tgt, n_micro, trace=True)
        doc = gather_chrome_trace(pipe)
        if dist.get_rank() == 0:
            import pathlib

            pathlib.Path(trace_path).parent.mkdir(parents=True, exist_ok=True)
            pathlib.Path(trace_path).write_text(doc)
        trace_file = str(trace_path)
    links = {}
    if dev_plan is not None:
        ks, rs = dev_plan.k.tolist(), dev_plan.r.tolist()
        lt = [float(v) for v in R.tolist()]
        for (s, d), k, r in zip(dev_plan.links, ks, rs):
            links[f"{s}->{d}"] = {"ratio": round(r, 3), "k": k, "wire_bytes": 16 + 12 * k,
                                  "frame_capacity_bytes": 16 + 12 * dev_plan.k_cap}
    elif plan is not None:
        for (s, d), r in sorted(plan.per_link.items()):
            links[f"{s}->{d}"] = {"ratio": round(r, 3), "k": select_k(boundary, r),
                                  "wire_bytes": 16 + 12 * select_k(boundary, r)}
    model_check = None
    if world > 1 and (plan is not None or dev_plan is not None) and codec is None:
        model_check = _fp_model_check(pipe, cfg, mb, seq_len, n_micro, ratio, dev,
                                      lt if plan_mode in ("measured", "adatopk") else None, chain)
    del pipe
    torch.cuda.empty_cache()
    out = {"metric": "GPT-2 compressed-pipeline samples/s", "value": round(gb / (t * 1e-3), 3), "unit": "samples/s",
           "n_gpus": world, "model": model, "layers": cfg.n_layer, "hidden": cfg.n_embd, "micro_batch": mb,
           "n_micro": n_micro, "global_batch": gb, "seq_len": seq_len, "ms_per_step": round(t, 2),
           "step_ms": [round(v, 2) for v in times], "warmup": warmup,
           "loss": round(loss, 4), "plan": plan_mode if world > 1 else "none (1 stage, no boundary)",
           "codec": codec_name, "base_ratio": ratio, "boundary_elems": boundary, "dense_boundary_bytes": boundary * 4,
           "links": links, "link_times_s": [round(v, 7) for v in lt] if lt is not None else None,
           "link_times_source": {"measured": "dense boundary P2P, CUDA events, median (measure_link_times); "
                                             "Eq. 6 + select_k on the device, k read by the kernels",
                                 "adatopk": "reference cli.cross_link_times over the simulated two-cluster "
                                            "network (alpha + beta*M per cross-device FP edge)"}.get(plan_mode),
           "fp_model": model_check, "trace": trace_file,
           "schedule": "GPipe fill-drain (executor.py:389-404), bf16 autocast, fp32 boundaries",
           "data": "synthetic tokens, random init"}
    if ofp is not None:
        out["partition"] = ("reference OP-Fence (opfence.opfence_schedule over opdag.build_dag + "
                            "costmodel.estimate_dag_costs, baseline/_ref), blocks rounded to their add2 node")
        out["opfence"] = ofp.to_dict()
    else:
        out["partition"] = ("OP-Fence FLOP-proportional contiguous split of [embeddings, blocks, head]: "
                            + str(partition(cfg.n_layer, world, cfg)))
    return out


def _fp_model_check(pipe, cfg, mb, seq_len, n_micro, ratio, dev, link_times=None, chain=None) -> dict:
    """The FP (fill) phase measured next to the planner's closed forms, from measured inputs:
    C_d = each stage's forward time for one micro-batch, R_d = the dense boundary
    receive time of the link into stage d (R_0 = 0), r_d = the plan's ratio on that link."""
    world = dist.get_world_size()
    tok, tgt = synthetic_batch(cfg, mb * n_micro, seq_len, dev, seed=123)
    c = torch.zeros(world, dtype=torch.float64, device=dev)
    c[pipe.s] = pipe.stage_fp_time(tok, tgt)  # indexed by stage
    dist.all_reduce(c)
    C = c.tolist()
    lt = link_times if link_times is not None else measure_link_times((mb, seq_len, cfg.n_embd), dev, chain=chain)
    R = [0.0] + list(lt)
    if pipe.dev_plan is not None:
        rr = pipe.dev_plan.r.tolist()
        r_dev = [1.0] + [rr[pipe.dev_plan.index[(s, s + 1)]] for s in range(world - 1)]
    else:
        r_dev = [1.0] + [pipe.plan.ratio_for(s, s + 1) for s in range(world - 1)]

    def timed_fp(p) -> float:
        ts = []
        for _ in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p.forward_only(tok, tgt, n_micro)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        tt = torch.tensor([sorted(ts)[1]], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # the DES charges a compressed message select_k(elems, r) * 12 bytes
    # (simulator.py:96-105); with measured R_d that is R_d scaled by the byte ratio
    d_b = mb * seq_len * cfg.n_embd
    M_comp = [0.0] + [x * (12 * select_k(d_b, q) / (4 * d_b)) if q > 1.0 else x for x, q in zip(R[1:], r_dev[1:])]
    t_comp = timed_fp(pipe)
    saved = pipe.plan, pipe.dev_plan
    pipe.plan, pipe.dev_plan = None, None  # the same stages with dense boundaries
    t_dense = timed_fp(pipe)
    pipe.plan, pipe.dev_plan = saved
    return {"C_stage_fp_s": [round(v, 6) for v in C], "R_link_dense_s": [round(v, 7) for v in R],
            "r_link": [round(v, 3) for v in r_dev], "n_b": n_micro,
            "eq3_dense_fp_ms": round(1e3 * eq3_pipeline_time(C, R, n_micro), 3),
            "measured_dense_fp_ms": round(1e3 * t_dense, 3),
            "eq7_compressed_fp_ms": round(1e3 * eq7_pipeline_time(C, R, n_micro, ratio, r_dev), 3),
            "eq7_scaled_bottleneck_fp_ms": round(1e3 * eq7_pipeline_time(C, R, n_micro, ratio, r_dev, True), 3),
            "measured_compressed_fp_ms": round(1e3 * t_comp, 3),
            "des_dense_fp_ms": round(1e3 * des_chain_fp_time(C, R, n_micro), 3),
            "des_compressed_fp_ms": round(1e3 * des_chain_fp_time(C, M_comp, n_micro), 3),
            "note": "planner closed forms (planner.py:90-147) and the reference's discrete-event model "
                    "(simulator.py:108-268, restated for a chain: des_chain_fp_time) from measured C_d / R_d, next "
                    "to the measured fill phase; neither model charges the compress/decompress kernels"}


def synthetic_batch(cfg: GPT2Config, batch: int, seq_len: int, device, seed: int = 0):
    g = torch.Generator(device=device).manual_seed(seed)
    tok = torch.randint(0, cfg.vocab, (batch, seq_len + 1), device=device, generator=g)
    return tok[:, :-1].contiguous(), tok[:, 1:].contiguous()


__all__ = ["GPT2Config", "GPT2_SMALL", "GPT2_MEDIUM", "GPT2_XL", "GPT2_TINY", "partition", "proportional_split", "op_flops", "make_stage",
           "link_plan", "two_cluster_link_times", "measure_link_times", "measured_link_plan", "DevicePlan",
           "eq3_pipeline_time",
           "eq7_pipeline_time", "des_chain_fp_time", "VirtualPipeline", "DistPipeline", "synthetic_batch", "run_pipeline",
           ]
