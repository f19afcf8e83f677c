"""Build a variant of the extension into tools/variants/<name>.so (tuning aid).

    python tools/build_variant.py NAME [-DMACRO=V ...] [-Xptxas ...]
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2308_12698_b200._build import CSRC, INCLUDE, NVCC_FLAGS, _nvcc, sources  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
out = ROOT / "tools" / "variants"
out.mkdir(exist_ok=True)
so = out / f"{name}.so"
cmd = [_nvcc(), *NVCC_FLAGS, *extra, f"-I{INCLUDE}", f"-I{CSRC}", "-o", str(so), *map(str, sources())]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-3000:])
(out / f"{name}.ptxas.txt").write_text(r.stderr)
print(so)
