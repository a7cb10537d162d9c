"""Compare per-config compress/decompress times across bench JSON files (development aid)."""
import json
import sys

runs = {}
for f in sys.argv[1:]:
    j = json.loads(open(f).read().strip().splitlines()[-1])
    runs[f.split("bench_")[-1].replace(".json", "")] = j
names = list(runs)
print("value GB/s: " + "  ".join(f"{n}={runs[n]['value']:.0f} ({runs[n]['ms_per_step']:.3f} ms)" for n in names))
keys = list(runs[names[0]]["per_config"])
for key in keys:
    c = "  ".join(f"{runs[n]['per_config'][key]['compress_us']:7.2f}" for n in names)
    d = "  ".join(f"{runs[n]['per_config'][key]['decompress_us']:7.2f}" for n in names)
    print(f"{key:40s} comp {c} | dec {d}")
