"""Build recipe for the sm_100a C-ABI library (libadatopk.so).

Plain nvcc, no torch extension machinery: the library exports only the
`extern "C"` symbols declared in include/adatopk.h, takes raw device pointers
and a cudaStream_t, and is loaded with ctypes.  Built in-tree so the .so travels
with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libadatopk.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
          "-I", str(ROOT / "include"), "-I", str(CSRC)]
# fmad is irrelevant to the integer select path; the Eq. 6 bookkeeping has only
# mul/div, but keep contraction off there so the IEEE order is explicit.
PER_FILE = {"gp_capi.cu": ["--fmad=false"]}
SOURCES = ["gp_compress.cu", "gp_cluster.cu", "gp_decompress.cu", "gp_capi.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the AdaTopK library needs the CUDA toolkit to build")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out_dir: Path = OUT_DIR, defines=()) -> Path:
    """Compile the library; `out_dir`/`defines` build development variants (see scripts/build_variant.py)."""
    out_dir.mkdir(parents=True, exist_ok=True)
    lib_path = out_dir / LIB.name
    headers = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "adatopk.h"]
    objs = []
    log = []
    for src in SOURCES:
        s = CSRC / src
        o = out_dir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers]):
            cmd = [nvcc(), *ARCH, *COMMON, *defines, *PER_FILE.get(src, []), "-Xptxas", "-v", "-c", str(s), "-o", str(o)]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log.append(r.stdout + r.stderr)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
    if force or _stale(lib_path, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(lib_path), *map(str, objs), "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    if log:
        (out_dir / "ptxas.log").write_text("\n".join(log))
    if verbose and log:
        print("\n".join(log))
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
