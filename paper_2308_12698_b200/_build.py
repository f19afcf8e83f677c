"""In-tree build of the sm_100a extension (nvcc, no JIT cache).

``python -m paper_2308_12698_b200._build`` or ``__graft_entry__.build()``
produces ``paper_2308_12698_b200/libswarmstep_b200.so`` next to this file,
so it travels with the repo snapshot to the GPU box.
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
LIB = PKG / "libswarmstep_b200.so"
INCLUDE = ROOT / "include"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    # ptxas' most register-frugal allocation: fewer spills in the 128-register
    # paired kernel, 2-3 % faster at K = 4..10, other kernels unchanged
    # (profiles/tune_r01_v8_reglevel.log)
    "-Xptxas", "--register-usage-level=0",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the sm_100a extension cannot be built")
    return cand


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = sources() + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > mtime for p in deps)


def _compile(src: Path, obj: Path, extra: list[str]) -> subprocess.CompletedProcess:
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    return subprocess.run([_nvcc(), *flags, *extra, f"-I{INCLUDE}", f"-I{CSRC}", "-c", "-o", str(obj), str(src)],
                          capture_output=True, text=True)


def build_to(out: Path, extra: list[str] | None = None) -> str:
    """Compile every translation unit (in parallel, one nvcc per file) and link
    them into the shared library `out`; returns the ptxas report."""
    import tempfile
    from concurrent.futures import ThreadPoolExecutor

    extra = list(extra or [])
    srcs = sources()
    with tempfile.TemporaryDirectory(prefix="ssb_build_") as tmpd:
        objs = [Path(tmpd) / (s.stem + ".o") for s in srcs]
        # the largest translation unit first: it bounds the wall time
        order = sorted(range(len(srcs)), key=lambda i: -srcs[i].stat().st_size)
        with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
            futs = {i: ex.submit(_compile, srcs[i], objs[i], extra) for i in order}
            res = {i: f.result() for i, f in futs.items()}
        for i in range(len(srcs)):
            if res[i].returncode != 0:
                raise RuntimeError(f"nvcc failed on {srcs[i].name} ({res[i].returncode}):\n{res[i].stderr[-4000:]}")
        tmp = out.with_suffix(".so.tmp")
        link = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                               "-o", str(tmp), *map(str, objs)], capture_output=True, text=True)
        if link.returncode != 0:
            raise RuntimeError(f"nvcc link failed ({link.returncode}):\n{link.stderr[-4000:]}")
        os.replace(tmp, out)
    return "".join(res[i].stderr for i in range(len(srcs)))


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    report = build_to(LIB)
    if verbose:
        sys.stderr.write(report)
    (PKG / "ptxas_info.txt").write_text(report)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
