"""Build a variant of the extension into tools/variants/<name>.so (tuning aid).

    python tools/build_variant.py NAME [-DMACRO=V ...] [-Xptxas ...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_12698_b200._build import build_to  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = ROOT / "tools" / "variants"
out.mkdir(exist_ok=True)
so = out / f"{name}.so"
(out / f"{name}.ptxas.txt").write_text(build_to(so, extra))
print(so)
