"""Build a development variant of the library with extra -D flags (A/B timing).

    python scripts/build_variant.py NAME -DGP_LIST_KB=40 ...
    GP_LIB=paper_2410_12707_b200/_lib/variants/NAME/libadatopk.so python scripts/graph_timing.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2410_12707_b200 import build as B  # noqa: E402

if __name__ == "__main__":
    name, defines = sys.argv[1], sys.argv[2:]
    print(B.build(force=True, out_dir=B.OUT_DIR / "variants" / name, defines=defines))
