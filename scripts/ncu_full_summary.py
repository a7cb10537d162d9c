"""Key metrics per launch of an `ncu --set full` report: python scripts/ncu_full_summary.py REPORT [--md]"""
import collections
import csv
import io
import subprocess
import sys

WANT = [("GPU Speed Of Light Throughput", "Duration"), ("GPU Speed Of Light Throughput", "DRAM Throughput"),
        ("Compute Workload Analysis", "Issue Slots Busy"), ("Instruction Statistics", "Executed Instructions"),
        ("Memory Workload Analysis", "L2 Hit Rate"), ("Launch Statistics", "Registers Per Thread"),
        ("Occupancy", "Achieved Occupancy")]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    idx = {h: i for i, h in enumerate(rows[0])}
    by, names = collections.defaultdict(dict), {}
    for r in rows[1:]:
        if len(r) < 15:
            continue
        i = int(r[idx["ID"]])
        by[i][(r[idx["Section Name"]], r[idx["Metric Name"]])] = (r[idx["Metric Value"]], r[idx["Metric Unit"]])
        names[i] = f'{r[idx["Kernel Name"]].split("(")[0]} grid {r[idx["Grid Size"]]}'
    print("| launch | kernel | " + " | ".join(w[1] for w in WANT) + " |")
    print("|---|---|" + "---|" * len(WANT))
    for i in sorted(by):
        m = by[i]
        print(f"| {i} | {names[i]} | " + " | ".join(f"{m.get(w, ('?', ''))[0]} {m.get(w, ('?', ''))[1]}".strip()
                                                    for w in WANT) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
