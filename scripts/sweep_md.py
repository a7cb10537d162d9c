"""Render a scripts/sweep.py JSON result as the markdown table kept in profiles/ (development aid).

    python scripts/sweep_md.py gpurun_out/sweep.json "round 1" > profiles/sweep_r01.md
"""
import json
import sys


def main():
    res = json.loads(open(sys.argv[1]).read())
    tag = sys.argv[2] if len(sys.argv) > 2 else ""
    print(f"# configs[4] sweep: compress + decompress, 1 MB..1 GB x ratio 1e-1..1e-4 ({tag})\n")
    print("`python scripts/sweep.py` on one B200: CUDA graphs, every launch after a 512 MB L2 read flush, differenced;")
    print(f"GB/s = algorithmic bytes (d*s + 12k) / device time; frac = pair throughput / measured HBM peak "
          f"({res['peak_gbs']:.0f} GB/s).")
    print("Every GPU result checked (k entries, increasing indices, threshold separation, round trip). CPU = NumPy oracle")
    print("port of the reference algorithm (stable argsort), 1 core, compress+decompress of the same input.\n")
    print("| dtype | size | ratio | compress µs | decompress µs | compress GB/s | decompress GB/s | pair frac | CPU GB/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in res["rows"]:
        print(f"| {r['dtype']} | {r['size_mb']} MB | 1e-{len(str(r['ratio'])) - 1} | {r['compress_us']} | "
              f"{r['decompress_us']} | {r['compress_gbs']:.0f} | {r['decompress_gbs']:.0f} | "
              f"{r['pair_frac_of_peak']:.3f} | {r.get('cpu_reference_gbs', '')} |")


if __name__ == "__main__":
    main()
