"""Generate golden vectors for the AdaTopK hot path FROM THE REFERENCE ITSELF.

Run in the build container, where the reference is importable:

    python tests/golden/make_golden.py            # writes tests/golden/golden.npz

It imports `geopipe.compressor` from /root/reference/pkg/src (read-only) and
records, for every case, the input bits, the ratio and the reference's
`SparsePayload.to_bytes()` frame (compressor.py:39-44).  The GPU box never
reads /root/reference; tests replay the committed .npz.

Cases (SURVEY.md §4 gaps + §7 step 1):
  * the reference's own unit-test vectors (tests/test_compressor.py:34-118)
  * acceptance criterion 4's 10,000 seeded vectors (tests/test_acceptance.py:105-123,
    rng 404), as float64 (reference dtype) and float32
  * special values: NaN, +-inf, +-0, denormals, massive ties
  * ReLU-like inputs (50% exact zeros) where the threshold key is 0
  * N(0,1), Student-t(3), quantized (heavy ties) float32 up to d = 200,000
  * bfloat16 inputs, parity defined as the reference on the exact fp32 upcast
  * Eq. 6 plans: acceptance criterion 5's 200 instances (rng 505) + direct cases
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"


def _ref():
    sys.path.insert(0, str(REF_SRC))
    from geopipe import compressor  # noqa: E402

    return compressor


class Bank:
    """Concatenated cases of one dtype."""

    def __init__(self, bits_dtype):
        self.bits_dtype = bits_dtype
        self.inputs, self.in_id, self.ratios, self.frames, self.names = [], [], [], [], []
        self._seen = {}

    def add(self, name, bits, ratio, frame):
        bits = np.asarray(bits, dtype=self.bits_dtype).reshape(-1)
        h = hashlib.sha256(bits.tobytes()).hexdigest()
        if h not in self._seen:  # each distinct input is stored once
            self._seen[h] = len(self.inputs)
            self.inputs.append(bits)
        self.names.append(name)
        self.in_id.append(self._seen[h])
        self.ratios.append(float(ratio))
        self.frames.append(np.frombuffer(frame, dtype=np.uint8))

    def arrays(self, prefix):
        def offs(chunks):
            return np.cumsum([0] + [len(c) for c in chunks]).astype(np.int64)

        return {
            f"{prefix}_inputs": np.concatenate(self.inputs),
            f"{prefix}_in_off": offs(self.inputs),
            f"{prefix}_in_id": np.array(self.in_id, dtype=np.int64),
            f"{prefix}_ratios": np.array(self.ratios),
            f"{prefix}_frames": np.concatenate(self.frames),
            f"{prefix}_fr_off": offs(self.frames),
            f"{prefix}_names": np.array(self.names),
        }


def main():
    C = _ref()
    f32, f64, bf16 = Bank(np.uint32), Bank(np.uint64), Bank(np.uint16)

    def add32(name, x, ratio):
        x = np.asarray(x, dtype=np.float32)
        f32.add(name, x.view(np.uint32), ratio, C.topk_compress(x, ratio).to_bytes())

    def add64(name, x, ratio):
        x = np.asarray(x, dtype=np.float64)
        f64.add(name, x.view(np.uint64), ratio, C.topk_compress(x, ratio).to_bytes())

    def add16(name, bits, ratio):
        bits = np.asarray(bits, dtype=np.uint16)
        up = (bits.astype(np.uint32) << 16).view(np.float32)
        bf16.add(name, bits, ratio, C.topk_compress(up, ratio).to_bytes())

    # -- the reference's own unit vectors (tests/test_compressor.py)
    add64("two_largest", [0.1, -5.0, 3.0, 0.0], 2)
    add64("ratio_one_identity", [1.0, -2.0, 0.5], 1)
    add64("magnitude_tie_lower_index", [2.0, -2.0, 1.0], 3)
    add64("all_zero", np.zeros(8), 4)
    add64("lossless_on_support", np.random.default_rng(0).standard_normal(50), 5)
    add32("byte_round_trip", [1.5, -2.25, 0.125, 4.0], 2)
    rng = np.random.default_rng(1)
    for d, ratio in [(10, 2), (100, 100), (7, 3.5)]:
        add64(f"payload_matches_wire_{d}_{ratio}", rng.standard_normal(d), ratio)
    add32("two_largest_f32", [0.1, -5.0, 3.0, 0.0], 2)

    # -- acceptance criterion 4 generator (tests/test_acceptance.py:107-112), rng 404
    rng = np.random.default_rng(404)
    small = []
    for _ in range(10_000):
        d = int(rng.integers(1, 13))
        values = np.round(rng.standard_normal(d) * rng.choice([1, 10, 100]), 3)
        ratio = float(rng.uniform(1, 20))
        small.append((values, ratio))
    for i, (v, r) in enumerate(small):
        add64(f"acc4_{i}", v, r)
    for i, (v, r) in enumerate(small[:2000]):
        add32(f"acc4_f32_{i}", v, r)

    # -- special values (fp32)
    rng = np.random.default_rng(7)
    specials = np.array([np.nan, -np.nan, np.inf, -np.inf, 0.0, -0.0, 1e-45, -1e-45, 1.17549435e-38,
                         -1.1754942e-38, 3.4028235e38, -3.4028235e38, 1.0, -1.0, 2.0, -2.0], dtype=np.float32)
    for d in (17, 256, 4099):
        x = rng.standard_normal(d).astype(np.float32)
        pos = rng.choice(d, size=min(d, 64), replace=False)
        x[pos] = rng.choice(specials, size=pos.size)
        for ratio in (1, 1.5, 2, 3, 10, 100, 1000):
            add32(f"specials_d{d}_r{ratio}", x, ratio)
    nan_heavy = np.full(1000, np.nan, dtype=np.float32)
    nan_heavy[::7] = rng.standard_normal(nan_heavy[::7].size).astype(np.float32)
    for ratio in (1.2, 2, 10, 100):
        add32(f"nan_heavy_r{ratio}", nan_heavy, ratio)
    nan_bits = np.full(300, 0x7FC00000, dtype=np.uint32)
    nan_bits[::3] = 0xFFC00001  # negative NaNs with payload
    nan_bits[::5] = 0x7F800001  # signalling NaN pattern
    for ratio in (1, 2, 30):
        add32(f"all_nan_r{ratio}", nan_bits.view(np.float32), ratio)
    denorm = (rng.integers(0, 1 << 23, 5000).astype(np.uint32) | (rng.integers(0, 2, 5000).astype(np.uint32) << 31))
    for ratio in (2, 10, 100):
        add32(f"denormals_r{ratio}", denorm.view(np.float32), ratio)
    ties = np.tile(np.array([1.0, -1.0, 0.5, -0.5, 0.0, -0.0], dtype=np.float32), 1000)
    for ratio in (1.5, 2, 3, 7, 100):
        add32(f"massive_ties_r{ratio}", ties, ratio)
    add32("constant_r10", np.full(4096, -3.25, dtype=np.float32), 10)

    # -- ReLU-like (50% exact zeros): threshold key is 0 when k > nnz
    x = np.maximum(rng.standard_normal(65536), 0).astype(np.float32)
    for ratio in (1.2, 1.5, 2, 10, 100):
        add32(f"relu_r{ratio}", x, ratio)

    # -- distributions at moderate d
    for d in (1, 2, 3, 5, 8, 31, 32, 33, 63, 127, 1000, 4097, 65537, 200_000):
        x = rng.standard_normal(d).astype(np.float32)
        for ratio in ((10, 100, 1000, 10000) if d >= 100_000 else (1, 1.01, 2, 10, 100)):
            add32(f"normal_d{d}_r{ratio}", x, ratio)
    t3 = rng.standard_t(3, 100_000).astype(np.float32)
    for ratio in (10, 100, 1000):
        add32(f"student_t3_r{ratio}", t3, ratio)
    q = (np.round(rng.standard_normal(120_000) * 4) / 4).astype(np.float32)
    for ratio in (10, 100, 1000):
        add32(f"quantized_ties_r{ratio}", q, ratio)
    ramp = np.arange(50_000, dtype=np.float32)  # sorted input: adversarial for sampling
    for ratio in (3, 100):
        add32(f"sorted_ramp_r{ratio}", ramp, ratio)
        add32(f"sorted_ramp_rev_r{ratio}", ramp[::-1].copy(), ratio)
    spike = np.zeros(70_000, dtype=np.float32)
    spike[12345:12345 + 500] = rng.standard_normal(500).astype(np.float32) * 1e3
    for ratio in (100, 1000):
        add32(f"spike_r{ratio}", spike, ratio)

    # -- float64 moderate
    for d in (1000, 65537):
        x = rng.standard_normal(d)
        for ratio in (1.5, 10, 100):
            add64(f"normal64_d{d}_r{ratio}", x, ratio)
    add64("quantized64_r10", np.round(rng.standard_normal(20000) * 2) / 2, 10)

    # -- bfloat16 (reference applied to the exact fp32 upcast)
    for d in (9, 1000, 100_003):
        xb = (rng.standard_normal(d).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        for ratio in (1, 2, 10, 100, 1000):
            add16(f"bf16_normal_d{d}_r{ratio}", xb, ratio)
    xb = np.array([0x7FC0, 0xFFC0, 0x7F80, 0xFF80, 0x0000, 0x8000, 0x0001, 0x8001, 0x3F80, 0xBF80] * 50,
                  dtype=np.uint16)
    for ratio in (1.5, 3, 10):
        add16(f"bf16_specials_r{ratio}", xb, ratio)

    # -- Eq. 6 plans: acceptance criterion 5 (tests/test_acceptance.py:126-140), rng 505
    rng = np.random.default_rng(505)
    plan_R = np.full((203, 8), np.nan)
    plan_n = np.zeros(203, dtype=np.int64)
    plan_r = np.zeros(203)
    plan_out = np.full((203, 8), np.nan)
    cases = []
    for _ in range(200):
        n = int(rng.integers(1, 9))
        R = {f"l{i}": float(rng.uniform(1e-6, 1e3)) for i in range(n)}
        r = float(rng.uniform(1, 1e4))
        cases.append((R, r))
    cases.append(({"L1": 10.0, "L2": 5.0, "L3": 1.0}, 100))
    cases.append(({"L1": 10.0, "L2": 0.01}, 100))
    cases.append(({"big": 1e6, "tiny": 1e-9}, 10))
    for i, (R, r) in enumerate(cases):
        plan = C.adatopk_plan(None, R, r)
        vals = list(R.values())
        plan_n[i] = len(vals)
        plan_R[i, :len(vals)] = vals
        plan_r[i] = r
        plan_out[i, :len(vals)] = [plan.per_link[l] for l in R]

    arrays = {}
    arrays.update(f32.arrays("f32"))
    arrays.update(f64.arrays("f64"))
    arrays.update(bf16.arrays("bf16"))
    arrays.update(plan_R=plan_R, plan_n=plan_n, plan_r=plan_r, plan_out=plan_out)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB): f32 {len(f32.names)}, f64 {len(f64.names)}, "
          f"bf16 {len(bf16.names)}, plans {len(cases)}")


if __name__ == "__main__":
    main()
