"""configs[3]'s partition from the reference's own, unchanged planner (CPU only).

opfence_plan builds GPT-2 in the reference's op kinds, prices it with
costmodel.estimate_dag_costs, schedules it with opfence.opfence_schedule over a
simulated two-cluster network, and takes R_i from cli.cross_link_times.  These
tests check the stage -> GPU mapping and the per-link plan at 2, 4 and 8
devices.
"""
import pytest

from paper_2410_12707_b200 import opfence_plan as OF
from paper_2410_12707_b200 import pipeline as PL
from paper_2410_12707_b200.compressor import adatopk_plan

XL = PL.GPT2_XL


@pytest.mark.parametrize("n_dev", [2, 4, 8])
def test_opfence_chain_and_block_ranges(n_dev):
    p = OF.opfence_partition(XL.n_layer, XL.n_embd, XL.vocab, n_dev, micro_batch=4, seq_len=1024, n_b=8)
    assert sorted(p.chain) == list(range(n_dev))
    assert [f"g{r}" for r in p.chain] == [v for c in p.cluster_order for v in c]
    # contiguous whole-block ranges tiling the layers; every block where its output node was scheduled
    assert p.bounds[0][0] == 0 and p.bounds[-1][1] == XL.n_layer
    assert all(p.bounds[i][1] == p.bounds[i + 1][0] for i in range(n_dev - 1))
    for s, (a, b) in enumerate(p.bounds):
        for i in range(a, b):
            assert p.assignment_devices[f"b{i:03d}.add2"] == f"g{p.chain[s]}"
    assert p.assignment_devices["tok"] == f"g{p.chain[0]}" and p.assignment_devices["head"] == f"g{p.chain[-1]}"
    # R_i for every consecutive stage pair, both directions, nothing else
    want = {(s, s + 1) for s in range(n_dev - 1)} | {(s + 1, s) for s in range(n_dev - 1)}
    assert set(p.link_R) == want
    assert all(p.link_R[(s, s + 1)] == p.link_R[(s + 1, s)] > 0 for s in range(n_dev - 1))


def test_opfence_clusters_and_eq6_at_8_devices():
    """Eight GPUs in two interleaved clusters: OP-Fence chains each cluster's
    devices together, so exactly one stage boundary crosses the slow link; Eq. 6
    gives it 3r and the fast links proportionally less."""
    p = OF.opfence_partition(XL.n_layer, XL.n_embd, XL.vocab, 8, micro_batch=4, seq_len=1024, n_b=8)
    assert len(p.cluster_order) == 2 and all(len(c) == 4 for c in p.cluster_order)
    par = [r % 2 for r in p.chain]
    assert par[:4] == [par[0]] * 4 and par[4:] == [1 - par[0]] * 4  # one cluster, then the other
    slow = [s for s in range(7) if p.chain[s] % 2 != p.chain[s + 1] % 2]
    assert slow == [3]
    plan = adatopk_plan(None, dict(p.link_R), 100.0)
    assert plan.ratio_for(3, 4) == 300.0 and plan.ratio_for(4, 3) == 300.0
    assert all(1.0 <= plan.ratio_for(s, s + 1) < 300.0 for s in range(7) if s != 3)
    # the reference CLI's alpha + beta*M per cross-device FP edge: the block boundary crosses two edges
    # (add2 -> next qkv and add2 -> next add1), each 4*1024*1600*4 bytes
    M = 4 * 1024 * 1600 * 4
    assert p.link_R[(3, 4)] == pytest.approx(2 * (OF.SLOW[0] + OF.SLOW[1] * M), rel=1e-12)
    assert p.link_R[(0, 1)] == pytest.approx(2 * (OF.FAST[0] + OF.FAST[1] * M), rel=1e-12)


def test_opfence_uses_the_reference_modules():
    ref = OF.reference()
    assert ref.opfence.opfence_schedule.__module__ == "geopipe.opfence"
    assert ref.cli.cross_link_times.__module__ == "geopipe.cli"
    dag = ref.opdag.build_dag(OF.gpt2_node_specs(2, 64, 100))
    order = ref.opdag.topological_order(dag)
    assert order[0] == "tok" and order[-2:] == ["~label", "~loss"] and order[-3] == "head"
