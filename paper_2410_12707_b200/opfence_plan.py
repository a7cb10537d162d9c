"""GPT-2 stage partition and per-link AdaTopK ratios from the reference's own, unchanged planner.

north_star keeps the OP-DAG builder, the per-operator workload estimator and
the OP-Fence scheduler host-side and unchanged.  This module calls them --
from the reference package installed offline in baseline/_ref (or any
importable `geopipe`) -- instead of restating them:

  1. GPT-2 expressed in the reference's operator kinds (SURVEY.md §7 hard part
     9): tokens are the batch (micro_batch_size = B*T), each block is
     qkv (linear H->3H) -> proj (linear H->H) -> add1 (add) -> fc (linear
     H->4H) -> act (relu as the GELU stand-in) -> out (linear 4H->H) -> add2
     (add), plus the embedding input, the LM head (linear H->V), the label and
     cross_entropy.  `opdag.build_dag` validates it (opdag.py:99-116).
  2. `costmodel.estimate_dag_costs` (costmodel.py:98-150) prices every node.
  3. `opfence.opfence_schedule` (opfence.py:347-435) clusters the devices by
     bandwidth (Louvain), chains the clusters, splits the topological order
     contiguously by device speed and repairs memory.  Its cluster_order gives
     the device chain: pipeline stage s runs on device_chain[s].
  4. OP-Fence may cut inside a block; the GPU pipeline's stages are whole
     blocks, so each block goes to the stage holding its output node (add2),
     the embeddings to stage 0 and the head/loss to the last stage.
  5. `cli.cross_link_times` (cli.py:51-59) gives R_i for every cross-device FP
     link of that (block-rounded) assignment, mirrored onto the BP link (the
     reference's CLI keys FP links only, SURVEY.md §7 hard part 10), and Eq. 6
     (`adatopk_plan`, compressor.py:111-129) turns them into per-link ratios.

The network is simulated (configs[3]: "simulated heterogeneous bandwidths"):
two clusters of devices, fast links inside a cluster and slow links between
them, in the style of the reference's scenarios/fig7_clusters.json, with the
clusters interleaved over the GPU ids so the bandwidth-aware chain is not the
identity.
"""
from __future__ import annotations

import sys
from dataclasses import dataclass, field
from pathlib import Path
from types import SimpleNamespace

REF_INSTALL = Path(__file__).resolve().parent.parent / "baseline" / "_ref"

FAST = (1e-5, 1.0 / 100e9)   # alpha (s), beta (s/B): inside a cluster
SLOW = (5e-3, 1.0 / 1.25e9)  # between the clusters (10 Gbps class)


def reference():
    """The reference's planning modules (geopipe), unchanged: the offline
    install in baseline/_ref, else an importable geopipe."""
    if (REF_INSTALL / "geopipe" / "opfence.py").exists() and str(REF_INSTALL) not in sys.path:
        sys.path.insert(0, str(REF_INSTALL))
    try:
        from geopipe import cli, costmodel, opdag, opfence  # noqa: F401
    except ImportError as exc:  # no fallback: the planner is the reference's own
        raise ImportError("the reference planner (geopipe) is not importable; install it into baseline/_ref "
                          "(DESIGN.md §7)") from exc
    return SimpleNamespace(cli=cli, costmodel=costmodel, opdag=opdag, opfence=opfence)


def gpt2_node_specs(n_layer: int, n_embd: int, vocab: int) -> list:
    """GPT-2 in the reference's op kinds (costmodel.py:98-138); per-token sizes."""
    h = n_embd
    specs = [dict(name="tok", kind="input", attrs={"size": h})]
    prev = "tok"
    for i in range(n_layer):
        b = f"b{i:03d}"
        specs += [
            dict(name=f"{b}.qkv", kind="linear", args=(prev,), attrs={"in_features": h, "out_features": 3 * h}),
            dict(name=f"{b}.proj", kind="linear", args=(f"{b}.qkv",), attrs={"in_features": h, "out_features": h}),
            dict(name=f"{b}.add1", kind="add", args=(prev, f"{b}.proj"), attrs={"size": h}),
            dict(name=f"{b}.fc", kind="linear", args=(f"{b}.add1",), attrs={"in_features": h, "out_features": 4 * h}),
            dict(name=f"{b}.act", kind="relu", args=(f"{b}.fc",), attrs={"size": 4 * h}),
            dict(name=f"{b}.out", kind="linear", args=(f"{b}.act",), attrs={"in_features": 4 * h, "out_features": h}),
            dict(name=f"{b}.add2", kind="add", args=(f"{b}.add1", f"{b}.out"), attrs={"size": h}),
        ]
        prev = f"{b}.add2"
    # '~' sorts after every other name: Kahn's lexicographic tie-break
    # (opdag.py:155-172) then places the label right before the loss
    specs += [
        dict(name="head", kind="linear", args=(prev,), attrs={"in_features": h, "out_features": vocab}),
        dict(name="~label", kind="label"),
        dict(name="~loss", kind="cross_entropy", args=("head", "~label"), attrs={"classes": vocab}),
    ]
    return specs


def two_cluster_network(ref, n_dev: int, peak_flops: float = 1.0e15, mem_gpu: float = 180e9,
                        fast=FAST, slow=SLOW):
    """n_dev devices g0..g{n-1}; cluster A = even ids, cluster B = odd ids
    (interleaved, like fig7_clusters.json's {d0,d2} / {d1,d3}); every pair
    linked, fast inside a cluster, slow across."""
    C = ref.costmodel
    devs = [C.DeviceProfile(device_id=f"g{i}", peak_flops=peak_flops, mem_gpu=mem_gpu) for i in range(n_dev)]
    links = {}
    for i in range(n_dev):
        for j in range(n_dev):
            if i != j:
                a, b = (fast if (i % 2) == (j % 2) else slow)
                links[(f"g{i}", f"g{j}")] = C.LinkProfile(src=f"g{i}", dst=f"g{j}", alpha=a, beta=b)
    return C.NetworkGraph(devices=devs, links=links)


@dataclass
class OpFencePlan:
    chain: list                      # stage s -> rank (device g{rank})
    bounds: list                     # stage s -> [a, b) block range
    cluster_order: list              # OP-Fence's cluster chain (device ids)
    link_R: dict                     # (src_stage, dst_stage) -> seconds (FP from cross_link_times, BP mirrored)
    assignment_devices: dict = field(default_factory=dict)  # op -> device of the raw OP-Fence schedule
    cut_inside_block: list = field(default_factory=list)    # blocks OP-Fence split across two devices

    def to_dict(self) -> dict:
        return {"chain": self.chain, "bounds": [list(b) for b in self.bounds], "cluster_order": self.cluster_order,
                "link_R_s": {f"{s}->{d}": r for (s, d), r in sorted(self.link_R.items())},
                "cut_inside_block": self.cut_inside_block}


def opfence_partition(n_layer: int, n_embd: int, vocab: int, n_dev: int, micro_batch: int, seq_len: int,
                      n_b: int, seed: int = 0, network=None) -> OpFencePlan:
    """The unchanged reference planner on GPT-2 over a two-cluster network."""
    ref = reference()
    dag = ref.opdag.build_dag(gpt2_node_specs(n_layer, n_embd, vocab))
    costs = ref.costmodel.estimate_dag_costs(dag, micro_batch * seq_len)  # tokens are the batch
    net = network if network is not None else two_cluster_network(ref, n_dev)
    sched = ref.opfence.opfence_schedule(dag, net, costs, n_b, seed=seed, batch_size=micro_batch)
    device_chain = [v for c in sched.cluster_order for v in c]
    pos = {dev: s for s, dev in enumerate(device_chain)}
    raw = dict(sched.assignment)

    # whole blocks per stage: a block goes to the stage of its output node
    block_stage = [pos[raw[f"b{i:03d}.add2"]] for i in range(n_layer)]
    S = len(device_chain)
    bounds, a = [], 0
    for s in range(S):
        b = a
        while b < n_layer and block_stage[b] <= s:
            b += 1
        bounds.append((a, b))
        a = b
    bounds[-1] = (bounds[-1][0], n_layer)
    cut = [i for i in range(n_layer)
           if len({raw[f"b{i:03d}.{op}"] for op in ("qkv", "proj", "add1", "fc", "act", "out", "add2")}) > 1]

    # the block-rounded assignment the GPU pipeline runs, and R_i from the reference CLI
    assign = {"tok": device_chain[0], "head": device_chain[-1], "~label": device_chain[-1],
              "~loss": device_chain[-1]}
    for s, (a, b) in enumerate(bounds):
        for i in range(a, b):
            for op in ("qkv", "proj", "add1", "fc", "act", "out", "add2"):
                assign[f"b{i:03d}.{op}"] = device_chain[s]
    fp_R = ref.cli.cross_link_times(SimpleNamespace(dag=dag, network=net), assign, costs)
    link_R = {}
    for (du, dv), t in fp_R.items():
        su, sv = pos[du], pos[dv]
        link_R[(su, sv)] = t
        link_R[(sv, su)] = t  # the gradient travels the mirrored link
    chain = [int(dev[1:]) for dev in device_chain]
    return OpFencePlan(chain=chain, bounds=bounds, cluster_order=[list(c) for c in sched.cluster_order],
                       link_R=link_R, assignment_devices=raw, cut_inside_block=cut)


__all__ = ["reference", "gpt2_node_specs", "two_cluster_network", "OpFencePlan", "opfence_partition"]
