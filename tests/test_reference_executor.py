"""The reference's own executor and CLI, unmodified, with the GPU compressor bound in
("byte-identical loss.csv from `geopipe run`").

`baseline/_ref` is the stock reference installed offline: its
`geopipe run` (cli.py:156-175) trains the scenario's model through the
reference executor, which compresses every cross-device activation and gradient
with `topk_compress` / `topk_decompress` (executor.py:207-297).  The golden
loss.csv files were written by that same command on the stock reference
(tests/golden/make_run_golden.py).  With `host_binding.patch_executor` the
executor calls the sm_100a kernels instead (float64 key path), and every
loss curve -- none / uniform_topk / adatopk at ratios 1.5 .. 100 -- must come
out byte-identical.  Skipped where baseline/_ref is not installed.
"""
import hashlib
import importlib.util
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
GOLD = ROOT / "tests" / "golden" / "run_loss"
META = json.loads((GOLD / "meta.json").read_text())

needs_ref = pytest.mark.skipif(not (REF / "geopipe" / "cli.py").exists(),
                               reason="reference not installed in baseline/_ref")


def _reference():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import geopipe.cli as cli
    import geopipe.errors as errors
    import geopipe.executor as executor

    return cli, executor, errors


def _gen():
    spec = importlib.util.spec_from_file_location("make_run_golden", ROOT / "tests" / "golden" / "make_run_golden.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _run(case: str, tmp_path: Path) -> bytes:
    cli, _, _ = _reference()
    info = META["scenarios"][case]
    scen = REF / "geopipe" / "scenarios" / info["file"]
    assert hashlib.sha256(scen.read_bytes()).hexdigest() == info["sha256"], "baseline/_ref is a different reference"
    meta = {"scenarios": {}, "reference_fails": {}}
    name = _gen().run_one(cli, scen, info["ratio_override"], tmp_path, meta)
    assert name == case, meta["reference_fails"]
    return (tmp_path / "loss.csv").read_bytes()


CASES = sorted(META["scenarios"])


def test_golden_runs_recorded():
    assert META["iters"] >= 10 and {"fig3", "fig3_r1.5", "fig3_r100"} <= set(CASES)
    for c in CASES:
        rows = (GOLD / f"{c}.csv").read_text().splitlines()
        assert rows[0] == "iter,none,uniform_topk,adatopk" and len(rows) == META["iters"] + 1


@needs_ref
@pytest.mark.parametrize("case", CASES)
def test_stock_reference_reproduces_golden(case, tmp_path):
    """The installed reference (CPU compressor) reproduces the committed curves."""
    assert _run(case, tmp_path) == (GOLD / f"{case}.csv").read_bytes()


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_compressor_in_reference_executor_byte_identical(cuda, case, tmp_path):
    from paper_2410_12707_b200 import host_binding
    from paper_2410_12707_b200 import compressor as C

    _, executor, errors = _reference()
    calls = {"compress": 0, "decompress": 0}
    real_c, real_d = C.topk_compress, C.topk_decompress

    def counted_c(*a, **kw):
        calls["compress"] += 1
        return real_c(*a, **kw)

    def counted_d(*a, **kw):
        calls["decompress"] += 1
        return real_d(*a, **kw)

    undo = host_binding.patch_executor(executor, errors)
    C.topk_compress, C.topk_decompress = counted_c, counted_d
    try:
        got = _run(case, tmp_path)
    finally:
        C.topk_compress, C.topk_decompress = real_c, real_d
        undo()
    assert calls["compress"] > 0 and calls["compress"] == calls["decompress"]
    assert got == (GOLD / f"{case}.csv").read_bytes()


@needs_ref
@pytest.mark.gpu
def test_host_binding_raises_reference_exceptions(cuda):
    import numpy as np

    from paper_2410_12707_b200 import host_binding

    _, executor, errors = _reference()
    undo = host_binding.patch_executor(executor, errors)
    try:
        with pytest.raises(errors.InvalidRatio):
            executor.topk_compress(np.ones(4), 0.5)
        with pytest.raises(errors.EmptyVector):
            executor.topk_compress(np.ones(0), 2.0)
        p = executor.topk_compress(np.arange(8.0), 2.0)
        out = executor.topk_decompress(p)
        assert isinstance(out, np.ndarray) and out.dtype == np.float64
        np.testing.assert_array_equal(out, [0, 0, 0, 0, 4, 5, 6, 7])
    finally:
        undo()


def test_host_binding_translates_exceptions_cpu():
    """patch_executor's wrappers re-raise the four compressor exceptions as the
    given errors module's classes (CPU: stub compressor, fake modules)."""
    import types

    from paper_2410_12707_b200 import errors as E
    from paper_2410_12707_b200 import host_binding

    class RefBase(Exception):
        pass

    ref_errors = types.SimpleNamespace(**{n: type(n, (RefBase,), {}) for n in
                                          ("InvalidRatio", "EmptyVector", "IndexOutOfRange", "NoCommunication")})
    raised = {}

    def make(exc):
        def fn(*a, **kw):
            raise exc("boom")
        return fn

    for name in ("InvalidRatio", "EmptyVector", "IndexOutOfRange"):
        wrapped = host_binding._translate(ref_errors)(make(getattr(E, name)))
        with pytest.raises(getattr(ref_errors, name)) as ei:
            wrapped(1)
        raised[name] = ei.value
        assert isinstance(ei.value.__cause__, getattr(E, name))
    with pytest.raises(ValueError):  # anything else passes through untouched
        host_binding._translate(ref_errors)(make(ValueError))()
    ex = types.SimpleNamespace(topk_compress="c", topk_decompress="d")
    undo = host_binding.patch_executor(ex, ref_errors)
    assert callable(ex.topk_compress) and callable(ex.topk_decompress)
    undo()
    assert (ex.topk_compress, ex.topk_decompress) == ("c", "d")
