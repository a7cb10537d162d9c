"""Summarise an ncu launch list (gpu__time_duration + dram bytes) of one bench step.

    python scripts/summarize_launches.py gpurun_out/launches.csv profiles/ncu_launches_r01.md profiles/ncu_traffic.json
"""
import csv
import json
import math
import sys
from collections import defaultdict

SHAPES = [(64, 256, 56, 56), (64, 512, 28, 28), (64, 1024, 14, 14), (64, 2048, 7, 7)]
RATIOS = [10, 100, 1000]


def units():
    for s in SHAPES:
        d = math.prod(s)
        for kind in ("activation", "gradient"):
            for r in RATIOS:
                yield s, kind, r, d, max(1, d // r)


def main(src, md_out, json_out):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10 and r[0] != "ID"]
    launches = defaultdict(dict)
    names = {}
    for r in rows:
        v = float(r[14].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[13])
        launches[int(r[0])][r[12]] = v * scale if scale is not None and "time" in r[12] else v
        names[int(r[0])] = r[4]
    ids = sorted(launches)
    comp = [i for i in ids if names[i].startswith("void compress_kernel")]
    dec = [i for i in ids if "decompress" in names[i]]
    # bench.py --streams 1 launches the units longest-first by its cost
    # estimate (bench.py: dense_w 2.2 for r <= 10, 4e6 per unit), stable
    us = sorted(units(), key=lambda u: -(u[3] * (2.2 if u[2] <= 10 else 1.0) + 4e6))
    lines = ["| unit | kernel | time us | DRAM read MB | DRAM write MB | algorithmic MB | DRAM/alg |",
             "|---|---|---|---|---|---|---|"]
    tot = {"c_t": 0.0, "c_dram": 0.0, "c_alg": 0.0, "d_t": 0.0, "d_dram": 0.0, "d_alg": 0.0}
    for (s, kind, r, d, k), ci, di in zip(us, comp, dec):
        alg = d * 4 + 12 * k
        for tag, i in (("compress", ci), ("decompress", di)):
            m = launches[i]
            t = m["gpu__time_duration.sum"]  # microseconds
            rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
            lines.append(f"| {list(s)} {kind} r={r} | {tag} | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                         f"{alg / 1e6:.1f} | {(rd + wr) / alg:.2f} |")
            p = "c" if tag == "compress" else "d"
            tot[p + "_t"] += t
            tot[p + "_dram"] += rd + wr
            tot[p + "_alg"] += alg
    summary = (f"\ncompress: {tot['c_t']:.0f} us total, DRAM {tot['c_dram'] / 1e9:.2f} GB vs algorithmic "
               f"{tot['c_alg'] / 1e9:.2f} GB; decompress: {tot['d_t']:.0f} us, DRAM {tot['d_dram'] / 1e9:.2f} GB "
               f"vs {tot['d_alg'] / 1e9:.2f} GB.  Compress share of kernel time: "
               f"{tot['c_t'] / (tot['c_t'] + tot['d_t']) * 100:.0f}%.\n")
    with open(md_out, "w") as f:
        f.write("# ncu launch list, one timed bench step (configs[1] workload)\n\n"
                "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none` (cold-cache, serialised: compare shares, not absolutes).\n\n")
        f.write("\n".join(lines))
        f.write(summary)
    json.dump({"compress_dram_bytes_per_launch_workload": tot["c_dram"] / max(1, len(comp)),
               "compress_alg_bytes_per_launch_workload": tot["c_alg"] / max(1, len(comp)),
               "decompress_dram_bytes_per_launch_workload": tot["d_dram"] / max(1, len(dec)),
               "source": src}, open(json_out, "w"), indent=1)
    print(summary)


if __name__ == "__main__":
    main(*sys.argv[1:4])
