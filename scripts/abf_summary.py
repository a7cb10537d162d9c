"""Summarise scripts/gpu_ab_fast.sh runs: value, compress frac and launch mean, decompress, C1 pair per variant."""
import json
import sys

for v in sys.argv[1:]:
    row = []
    for rep in (1, 2):
        try:
            d = json.loads(open(f"gpurun_out/abf_{v}_{rep}.json").read().strip().splitlines()[-1])
            r = d["roofline"]
            c1 = d.get("c1_gpt2_small", {})
            row.append(f"{d['value']:8.1f} frac {r['frac']:.4f} cmp {r['launch_us_mean']:6.2f}us dec {r.get('decompress_achieved')} "
                       f"c1 {c1.get('pair_us')} b8 {c1.get('batch8_8streams', {}).get('frac_of_peak')}")
        except Exception as e:  # noqa: BLE001
            row.append(f"ERR {e}")
    print(f"{v:8s}", " | ".join(row))
