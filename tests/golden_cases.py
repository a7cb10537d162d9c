"""Loader for tests/golden/golden.npz (frames produced by the reference itself)."""
from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"

_VIEW = {"f32": np.float32, "f64": np.float64, "bf16": None}


@lru_cache(maxsize=1)
def _load():
    with np.load(GOLDEN) as g:
        return {k: g[k] for k in g.files}


def cases(prefix: str):
    """Yield (name, x, ratio, frame) — x is float32/float64, or uint16 bf16 bits."""
    g = _load()
    inp, ioff, iid = g[f"{prefix}_inputs"], g[f"{prefix}_in_off"], g[f"{prefix}_in_id"]
    fr, foff = g[f"{prefix}_frames"], g[f"{prefix}_fr_off"]
    for i, name in enumerate(g[f"{prefix}_names"]):
        j = iid[i]
        bits = inp[ioff[j]:ioff[j + 1]]
        x = bits.view(_VIEW[prefix]) if _VIEW[prefix] is not None else bits
        yield str(name), x, float(g[f"{prefix}_ratios"][i]), fr[foff[i]:foff[i + 1]].tobytes()


def plans():
    """Yield (R list, base_ratio, expected per-link ratios list) from the reference's adatopk_plan."""
    g = _load()
    for i in range(len(g["plan_n"])):
        n = int(g["plan_n"][i])
        yield list(g["plan_R"][i, :n]), float(g["plan_r"][i]), list(g["plan_out"][i, :n])
