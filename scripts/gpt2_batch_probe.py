"""GPT-2 boundary shapes, n tensors in flight: compress+decompress throughput vs n and streams (development aid).

    python scripts/gpt2_batch_probe.py

bench.py's gpt2_batch (c1_gpt2_small.batch8_8streams): every tensor compressed
then decompressed on its stream (grids of num_sms/streams CTAs, a workspace per
stream), one CUDA graph, L2 flushed (512 MB read) before each replay, median
of 10.  Prints GB/s (algorithmic d*4+12k per launch) and the
fraction of the measured HBM peak.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2410_12707_b200 import _lib  # noqa: E402
from scripts.sweep import peak_gbs  # noqa: E402


def run(shape, n, ns, flush):
    from bench import gpt2_batch  # the bench's own measurement

    return gpt2_batch(_lib.lib(), torch.device("cuda", 0), shape, n, ns, flush)


def main():
    peak = peak_gbs()
    flush = torch.ones(128 << 20, device="cuda")
    for name, shape in (("C1 8x1024x768", (8, 1024, 768)), ("C3 8x1024x1024", (8, 1024, 1024))):
        for n in (1, 8, 16, 32):
            for ns in (1, 4, 8):
                if ns > n:
                    continue
                t, gbs = run(shape, n, ns, flush)
                print(f"{name:16s} n={n:3d} streams={ns} | {t:8.1f} us  {gbs:7.0f} GB/s  {gbs / peak:5.3f} of peak",
                      flush=True)
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
