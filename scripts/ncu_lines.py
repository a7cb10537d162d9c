"""Aggregate ncu per-SASS warp-stall samples by CUDA source line.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--top 40]

ncu's CSV source page has no line numbers for SASS rows, so the kernel is
re-disassembled from the built object with `nvdisasm --print-line-info` and
instructions are matched by their index within the function.
"""
import argparse
import csv
import io
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIBDIR = ROOT / "paper_2410_12707_b200" / "_lib"


def ncu_sass(report, kregex):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "-k", f"regex:{kregex}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    kernels, cur = [], None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            kernels.append(cur)
        elif row[0] == "Address":
            cur["hdr"] = {h: i for i, h in enumerate(row)}
        elif cur is not None and "hdr" in cur:
            cur["rows"].append(row)
    return kernels


def line_table(mangled_hint):
    """instruction index -> (file, line) for the function whose name contains mangled_hint."""
    table = {}
    with tempfile.TemporaryDirectory() as td:
        for obj in LIBDIR.glob("*.o"):
            subprocess.run(["cuobjdump", "-xelf", "all", str(obj)], cwd=td, capture_output=True)
        for cub in Path(td).glob("*.cubin"):
            dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout
            fn, idx, loc = None, 0, None
            for ln in dis.splitlines():
                m = re.match(r"\s*\.text\.(\S+):", ln)
                if m:
                    fn, idx, loc = m.group(1), 0, None
                    continue
                m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                if m:
                    loc = (Path(m.group(1)).name, int(m.group(2)))
                    continue
                if fn and re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
                    table.setdefault(fn, {})[idx] = loc
                    idx += 1
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("kernel")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--fn", default=None, help="substring of the mangled function name (disambiguates templates)")
    args = ap.parse_args()
    tables = line_table(args.kernel)
    for k in ncu_sass(args.report, args.kernel):
        hdr = k["hdr"]
        stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        cands = [fn for fn in tables if re.search(args.kernel.lstrip("^"), fn) and (args.fn is None or args.fn in fn)]
        # pick the function whose instruction count matches
        fn = next((f for f in cands if len(tables[f]) == len(k["rows"])), cands[0] if cands else None)
        tab = tables.get(fn, {})
        agg = defaultdict(lambda: defaultdict(float))
        total = 0.0
        for i, r in enumerate(k["rows"]):
            try:
                s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
            except ValueError:
                continue
            total += s
            loc = tab.get(i) or ("?", 0)
            agg[loc]["_all"] += s
            try:
                agg[loc]["_inst"] += float(r[hdr["Instructions Executed"]] or 0)
            except (ValueError, KeyError):
                pass
            for st in stalls:
                try:
                    agg[loc][st[6:]] += float(r[hdr[st]] or 0)
                except ValueError:
                    pass
        print(f"== {k['name'][:100]}  ({fn}, {len(k['rows'])} instr, {total:.0f} samples)")
        tot_st = defaultdict(float)
        for d in agg.values():
            for st, v in d.items():
                if not st.startswith("_"):
                    tot_st[st] += v
        print("   stalls: " + ", ".join(f"{st}={100 * v / max(total, 1):.1f}%"
                                       for st, v in sorted(tot_st.items(), key=lambda kv: -kv[1])[:10]))
        for loc, d in sorted(agg.items(), key=lambda kv: -kv[1]["_all"])[: args.top]:
            top = sorted(((s, v) for s, v in d.items() if not s.startswith("_")), key=lambda kv: -kv[1])[:3]
            print(f"  {loc[0]}:{loc[1]:<5d} {d['_all']:6.0f} ({100 * d['_all'] / max(total, 1):4.1f}%) "
                  f"inst {d['_inst'] / 1e3:8.1f}K  "
                  + ", ".join(f"{s}={v:.0f}" for s, v in top if v))


if __name__ == "__main__":
    sys.exit(main())
