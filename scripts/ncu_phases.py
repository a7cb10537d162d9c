"""Group ncu per-line samples / instructions of the compress kernel by phase (line ranges found by markers)."""
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "paper_2410_12707_b200" / "csrc" / "gp_compress.cu"
MARKERS = [("prologue+watermark", "compress_kernel(const CompressArgs a) {"),
           ("stream", "  auto stream_unit = [&]"), ("find", "  auto find_b1 = [&]"),
           ("pass loop/B1", "  // first pass, and at most one partial rescan"),
           ("split", "    // One pass over the list: per-warp sure"),
           ("fc-resolve", "    // ---- stage 3: one round trip"), ("walk", "    uint32_t jfc = w_boff[w];"),
           ("slow path", "    // ================= slow path"), ("cleanup", "  // ---- leave the workspace clean")]


def main():
    rep, fn = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "TraitsF32"
    text = SRC.read_text()
    starts = []
    for name, m in MARKERS:
        starts.append((text[:text.index(m)].count("\n") + 1, name))
    out = subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_lines.py"), rep, "compress_kernel", "--fn", fn,
                          "--top", "100000"], capture_output=True, text=True).stdout
    agg = defaultdict(lambda: [0, 0.0])
    for line in out.splitlines():
        m = re.match(r"\s+(\S+):(\d+)\s+(\d+)\s+\(.*?\)\s+inst\s+([\d.]+)K", line)
        if not m:
            if line.startswith(("==", "   stalls")):
                print(line)
            continue
        f, ln, s, n = m.group(1), int(m.group(2)), int(m.group(3)), float(m.group(4)) * 1e3
        ph = "helpers/" + f
        if f == "gp_compress.cu":
            ph = "helpers<kernel"
            for st, name in starts:
                if ln >= st:
                    ph = name
        agg[ph][0] += s
        agg[ph][1] += n
    ts = sum(v[0] for v in agg.values())
    ti = sum(v[1] for v in agg.values())
    for k, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:26s} samples {s:6d} ({100 * s / ts:4.1f}%)  inst {n / 1e6:7.2f}M ({100 * n / ti:4.1f}%)")


if __name__ == "__main__":
    main()
