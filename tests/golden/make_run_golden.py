"""Golden `geopipe run` loss curves FROM THE STOCK REFERENCE.

Run in the build container, where the reference is importable:

    python tests/golden/make_run_golden.py        # writes tests/golden/run_loss/*.csv

For each scenario bundled with the reference (pkg/src/geopipe/scenarios/*.json)
it runs the reference CLI's `run` command (cli.py:156-175: one numeric training
run per compression mode none / uniform_topk / adatopk through the reference
executor, executor.py:207-297) and stores `loss.csv` verbatim, plus the
SHA-256 of the scenario file it used.  Each scenario runs at its own base ratio
and with "ratio" overridden to 1.5, 3 and 100, as the reference's CLI test does
(tests/test_cli.py:138-142) (scenarios the stock reference itself
cannot run are listed with the exception it raises).  tests/test_reference_executor.py reruns
the same command with the GPU compressor bound into the executor
(paper_2410_12707_b200.host_binding) and requires byte-identical files.
"""
from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "run_loss"
ITERS = 20
RATIOS = (None, 1.5, 3, 100)  # None = the scenario's own ratio (fig3: 10)


def main():
    sys.path.insert(0, str(REF_SRC))
    from geopipe import cli  # noqa: E402

    OUT.mkdir(exist_ok=True)
    meta = {"iters": ITERS, "scenarios": {}, "reference_fails": {}}
    for scen in sorted((REF_SRC / "geopipe" / "scenarios").glob("*.json")):
        for ratio in RATIOS:
            with tempfile.TemporaryDirectory() as td:
                name = run_one(cli, scen, ratio, Path(td), meta)
                if name is None:
                    break
                (OUT / f"{name}.csv").write_bytes((Path(td) / "loss.csv").read_bytes())
                print(name, "ok")
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1) + "\n")


def run_one(cli, scen: Path, ratio, td: Path, meta: dict):
    """`geopipe run` on `scen` (its "ratio" overridden unless None) -> case name, or None if the reference fails."""
    doc = json.loads(scen.read_text())
    if ratio is not None:
        doc["ratio"] = ratio
    f = td / "scenario.json"
    f.write_text(json.dumps(doc))
    name = scen.stem if ratio is None else f"{scen.stem}_r{ratio}"
    try:
        assert cli.main(["run", "--scenario", str(f), "--out", str(td), "--iters", str(ITERS)]) == 0
    except Exception as exc:  # the stock reference cannot run this scenario: nothing to pin
        meta["reference_fails"][scen.stem] = f"{type(exc).__name__}: {exc}"
        print(scen.stem, "reference fails:", repr(exc))
        return None
    meta["scenarios"][name] = {"file": scen.name, "ratio_override": ratio,
                               "sha256": hashlib.sha256(scen.read_bytes()).hexdigest()}
    return name


if __name__ == "__main__":
    main()
