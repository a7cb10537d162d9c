import sys, re, subprocess
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
import ncu_lines as N
from collections import defaultdict
rep = sys.argv[1]
tables = N.line_table("compress_kernel")
for k in N.ncu_sass(rep, "compress_kernel"):
    hdr = k["hdr"]
    fn = next((f for f in tables if "compress_kernel" in f and len(tables[f]) == len(k["rows"])), None)
    tab = tables[fn]
    agg = defaultdict(float); samp = defaultdict(float)
    tot = 0; ts = 0
    for i, r in enumerate(k["rows"]):
        try: n = float(r[hdr["Instructions Executed"]] or 0); s = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError: continue
        loc = tab.get(i) or ("?", 0)
        line = loc[1] if loc[0] == "gp_compress.cu" else -1
        ph = "other/helpers"
        if 395 <= line < 470: ph = "prologue/watermark"
        elif 470 <= line < 700: ph = "stream"
        elif 700 <= line < 780: ph = "stream-tail+flush+find"
        elif 780 <= line < 880: ph = "split"
        elif 880 <= line < 1080: ph = "stage3/FC"
        elif 1080 <= line < 1140: ph = "walk"
        elif 1140 <= line < 1260: ph = "slow/cleanup"
        elif line > 0: ph = "lib-helpers(<395)"
        agg[ph] += n; samp[ph] += s; tot += n; ts += s
    print(k["name"][:60], f"total warp-instr {tot/1e6:.2f}M samples {ts:.0f}")
    for ph in sorted(agg, key=lambda p: -agg[p]):
        print(f"  {ph:28s} {agg[ph]/1e6:6.2f}M ({100*agg[ph]/tot:4.1f}%)  samples {100*samp[ph]/ts:4.1f}%")
