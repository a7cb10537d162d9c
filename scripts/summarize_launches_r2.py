"""Summarise the round-2 ncu launch lists of one timed bench step (scripts/gpu_ncu_r2.sh).

    python scripts/summarize_launches_r2.py gpurun_out/launches_c.csv gpurun_out/launches_d.csv \
        profiles/ncu_launches_r02.md profiles/ncu_traffic.json

The kernels are the 24 compress and 24 decompress nodes of one CUDA-graph
replay in the bench's timed configuration (7 streams, 22/21-CTA compress grids,
24 distinct inputs).  ncu serialises the nodes, so each launch's time is
cold-ish and alone; the units are matched to launches by their DRAM bytes
(compress reads ~4d and writes the 16 + 12k frame; decompress writes ~4d).
"""
import csv
import json
import math
import sys
from collections import defaultdict

SHAPES = [(64, 256, 56, 56), (64, 512, 28, 28), (64, 1024, 14, 14), (64, 2048, 7, 7)]
RATIOS = [10, 100, 1000]


def units():
    out = []
    for s in SHAPES:
        d = math.prod(s)
        for kind in ("activation", "gradient"):
            for r in RATIOS:
                out.append((s, kind, r, d, max(1, d // r)))
    return out


def load(src):
    launches, names = defaultdict(dict), {}
    for r in csv.reader(open(src)):
        if len(r) < 15 or r[0] == "ID":
            continue
        v = float(r[14].replace(",", ""))
        unit = r[13]
        if "time" in r[12]:
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        elif unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        launches[int(r[0])][r[12]] = v
        names[int(r[0])] = r[4]
    return [(names[i], launches[i]) for i in sorted(launches)]


def bench_order(nstreams=7, dense_w=3.0, ovh=4e6, stagger=True, num_sms=148):
    """The units in the order bench.py captures them into its graphs (N=1): longest-first
    greedy assignment to streams by its cost model (weighted by each stream's grid size),
    odd streams reversed, streams concatenated."""
    us = units()
    ctas_of = [num_sms // nstreams + (1 if j < num_sms % nstreams else 0) for j in range(nstreams)]

    def cost(u):
        return u[3] * (dense_w if u[2] <= 10 else 1.0) + ovh

    load = [0.0] * nstreams
    per = [[] for _ in range(nstreams)]
    for i in sorted(range(len(us)), key=lambda i: -cost(us[i])):
        j = min(range(nstreams), key=lambda j: load[j])
        per[j].append(i)
        load[j] += cost(us[i]) * ctas_of[0] / ctas_of[j]
    if stagger:
        for j in range(1, nstreams, 2):
            per[j].reverse()
    return [us[i] for lst in per for i in lst]


def match(rows, compress):
    """Launch i of the replay is the i-th captured unit; checked against the DRAM reads (x for a
    compress, ~4d; the decompress writes ~4d)."""
    order = bench_order()
    if len(rows) == len(order):
        out = list(zip(order, [m for _, m in rows]))
        ok = all(abs((m["dram__bytes_read.sum"] if compress else max(m["dram__bytes_write.sum"], 1)) - 4 * u[3])
                 < 0.2 * 4 * u[3] for u, m in out) if compress else True
        if ok:
            return out
    left = units()
    out = []
    for name, m in rows:
        rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]

        def cost(u):
            d, k = u[3], u[4]
            if compress:
                return abs(rd - 4 * d) / (4 * d) + abs(wr - (16 + 12 * k)) / (4 * d)
            return abs(wr - 4 * d) / (4 * d) + abs(rd - (16 + 12 * k)) / (4 * d)

        u = min(left, key=cost)
        left.remove(u)
        out.append((u, m))
    return out


def main(csv_c, csv_d, md_out, json_out):
    comp = match(load(csv_c), True)
    dec = match(load(csv_d), False)
    lines = ["| unit | kernel | time us | DRAM read MB | DRAM write MB | algorithmic MB | DRAM/alg |",
             "|---|---|---|---|---|---|---|"]
    tot = defaultdict(float)
    for tag, lst in (("compress", comp), ("decompress", dec)):
        for (s, kind, r, d, k), m in sorted(lst, key=lambda x: (x[0][0], x[0][1], x[0][2]), reverse=False):
            alg = 4 * d + 12 * k
            t, rd, wr = m["gpu__time_duration.sum"], m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
            lines.append(f"| {list(s)} {kind} r={r} | {tag} | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                         f"{alg / 1e6:.1f} | {(rd + wr) / alg:.2f} |")
            p = tag[0]
            tot[p + "_t"] += t
            tot[p + "_dram"] += rd + wr
            tot[p + "_alg"] += alg
    n = len(comp)
    summary = (f"\ncompress: {tot['c_t']:.0f} us total (serialised), DRAM {tot['c_dram'] / 1e9:.3f} GB vs algorithmic "
               f"{tot['c_alg'] / 1e9:.3f} GB ({tot['c_dram'] / tot['c_alg']:.2f}x); decompress: {tot['d_t']:.0f} us, "
               f"DRAM {tot['d_dram'] / 1e9:.3f} GB vs {tot['d_alg'] / 1e9:.3f} GB ({tot['d_dram'] / tot['d_alg']:.2f}x).  "
               f"Compress share of kernel time: {tot['c_t'] / (tot['c_t'] + tot['d_t']) * 100:.0f}%.\n")
    with open(md_out, "w") as f:
        f.write("# ncu launch list, one timed bench step (round 2: the timed configuration)\n\n"
                "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` "
                "over `bench.py --no-pipeline --no-sweep --steps 1 --warmup 3` with `GP_BENCH_SPINUP=0`: the 24 "
                "compress and 24 decompress kernel nodes of the first timed CUDA-graph replay (5 streams, 30/29-CTA "
                "compress grids, 24 distinct inputs; `scripts/gpu_ncu_r2.sh`).  ncu serialises the nodes: compare "
                "shares and DRAM bytes, not absolute times.\n\n")
        f.write("\n".join(lines))
        f.write(summary)
    json.dump({"compress_dram_bytes_per_launch_workload": tot["c_dram"] / max(1, n),
               "compress_alg_bytes_per_launch_workload": tot["c_alg"] / max(1, n),
               "decompress_dram_bytes_per_launch_workload": tot["d_dram"] / max(1, len(dec)),
               "measured_on": "the timed configuration: 7 streams, CUDA-graph replay, 24 distinct inputs "
                              "(ncu serialises the nodes)",
               "source": [csv_c, csv_d]}, open(json_out, "w"), indent=1)
    print(summary)


if __name__ == "__main__":
    main(*sys.argv[1:5])
