"""Summarise gpurun_out/ab_<variant>_<rep>.json bench lines (scripts/gpu_ab_r2.sh)."""
import json
import sys
from pathlib import Path

out = Path(__file__).resolve().parent.parent / "gpurun_out"
for v in sys.argv[1:]:
    for rep in (1, 2):
        p = out / f"ab_{v}_{rep}.json"
        try:
            d = json.loads(p.read_text().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            print(v, rep, "FAILED", e)
            continue
        pc = d["per_config"]
        big = {k.split("/")[1][0] + k.split("/")[2]: (v_["compress_us"], v_["decompress_us"]) for k, v_ in pc.items()
               if k.startswith("[64, 256")}
        print(f"{v:10s} rep{rep} value {d['value']:8.1f} ms {d['ms_per_step']:.4f} frac {d['roofline']['frac']:.4f} "
              f"dec {d['roofline']['decompress_achieved']:.0f} c1 {d['c1_gpt2_small']['pair_us']} "
              f"b8 {d['c1_gpt2_small']['batch8_8streams']['frac_of_peak']} big {big}")
