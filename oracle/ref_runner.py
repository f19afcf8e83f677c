"""TEST / BENCH INFRASTRUCTURE ONLY -- the reference's own CPU path, run here.

``install()`` (called by ``__graft_entry__.build()`` in the build container)
pip-installs the unmodified reference package (``/root/reference/pkg``, the
pure-Python + numpy ``swarmstep``) into ``oracle/_ref/`` from a copy under
/tmp (the reference tree is read-only).  ``oracle/_ref/`` is git-ignored but
travels to the GPU box with the repo snapshot, so the GPU tests can drive the
unmodified ``swarmstep.core.World`` and bench.py can time the reference's
``QuadGroup.step`` (core.py:166-202) on the box's own host cores.

``run_quadgroup()`` is BASELINE.md 2's CPU-baseline plan: the n_total-agent
bench swarm (``paper_2308_12698_b200.synthetic``, the same rows the GPU arm
steps) is sharded by contiguous index over P worker processes with numpy
pinned to one thread each; each worker owns one reference ``QuadGroup`` of
its rows; every timed sample starts on a barrier, and a sample's time is the
max over workers.  Only tests/, smoke() and bench.py's CPU legs import this.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg")
_THREAD_VARS = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMEXPR_NUM_THREADS")


def available() -> bool:
    return (REF / "swarmstep" / "core.py").is_file()


def install(force: bool = False) -> bool:
    """pip install the reference package into oracle/_ref (from a /tmp copy).
    Returns whether the reference is importable from oracle/_ref afterwards."""
    if available() and not force:
        return True
    if not (REF_SRC / "pyproject.toml").is_file():
        return available()
    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "pkg"
        shutil.copytree(REF_SRC, src, ignore=shutil.ignore_patterns(
            "frontend", "build", "*.egg-info", "__pycache__", ".pytest_cache"))
        for p in src.rglob("*"):               # the copy inherits read-only modes
            p.chmod(p.stat().st_mode | 0o200)
        src.chmod(src.stat().st_mode | 0o200)
        stage = Path(td) / "target"
        subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index", "--no-build-isolation",
                        "--no-deps", "--find-links", "/opt/wheelhouse", "--target", str(stage), str(src)],
                       check=True, capture_output=True)
        if REF.exists():
            shutil.rmtree(REF)
        shutil.copytree(stage, REF)
    return available()


def import_path() -> str:
    if not available():
        raise RuntimeError("the reference is not installed in oracle/_ref (run __graft_entry__.build())")
    return str(REF)


def _worker(idx, lo, hi, n_total, dt, ticks, samples, warm, barrier, q, root):
    # numpy is pinned to one thread by the parent's environment at spawn time
    sys.path.insert(0, str(REF))
    sys.path.insert(0, root)
    try:
        import numpy as np
        from swarmstep.core import QuadGroup
        from swarmstep.quad import QuadParams
        from swarmstep.state import batch_create

        from paper_2308_12698_b200.synthetic import swarm

        pos, sp = swarm(n_total, lo, hi)
        g = QuadGroup(0, batch_create(0, hi - lo, pos, id_base=lo), QuadParams())
        g.cmd_level[:] = 0                            # POS (core.py:98, _LVL_POS)
        g.cmd_values[:] = sp.T.astype(np.float64)     # the device's float32 setpoints, widened exactly
        g._level_dirty = True
        for _ in range(warm):
            g.step(dt)
        times = []
        for _ in range(samples):
            barrier.wait()
            t0 = time.perf_counter()
            for _ in range(ticks):
                g.step(dt)
            times.append(time.perf_counter() - t0)
        q.put((idx, times, int(np.count_nonzero(~g.batch.alive)), None))
    except BaseException as e:  # noqa: BLE001 -- reported to the parent
        try:
            barrier.abort()
        except Exception:
            pass
        q.put((idx, None, 0, f"{type(e).__name__}: {e}"))


def run_quadgroup(n_total: int, dt: float = 1e-3, ticks: int = 1, samples: int = 3, warm: int = 1,
                  procs: int | None = None, timeout: float = 1800.0, n_rows: int | None = None) -> dict:
    """Time the reference QuadGroup.step on rows [0, n_rows) (default: all) of
    the n_total-agent bench swarm over ``procs`` host processes (default: every
    core of the affinity mask).

    Returns per-sample max-over-workers times and the derived agent-steps/s.
    """
    n_rows = n_total if n_rows is None else min(int(n_rows), n_total)
    import multiprocessing as mp

    from oracle.oracle import cpu_count
    from paper_2308_12698_b200.parallel import shard_range

    P = max(1, min(procs or cpu_count(), n_rows))
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(P), ctx.Queue()
    saved = {k: os.environ.get(k) for k in _THREAD_VARS}
    os.environ.update({k: "1" for k in _THREAD_VARS})
    t_setup = time.perf_counter()
    try:
        ps = []
        for i in range(P):
            lo, hi = shard_range(n_rows, i, P)
            p = ctx.Process(target=_worker, args=(i, lo, hi, n_total, dt, ticks, samples, warm, barrier, q,
                                                  str(HERE.parent)), daemon=True)
            p.start()
            ps.append(p)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    res, err = {}, None
    deadline = time.perf_counter() + timeout
    while len(res) < P:
        idx, times, dead, e = q.get(timeout=max(1.0, deadline - time.perf_counter()))
        if e is not None:
            err = err or e
        res[idx] = (times, dead)
    for p in ps:
        p.join(timeout=60)
    if err is not None:
        raise RuntimeError(f"reference worker failed: {err}")
    wall = time.perf_counter() - t_setup
    per_sample = [max(res[i][0][s] for i in range(P)) for s in range(samples)]
    total = sum(per_sample)
    per_core = sorted((shard_range(n_rows, i, P)[1] - shard_range(n_rows, i, P)[0]) * ticks * samples
                      / sum(res[i][0]) for i in range(P))
    return {
        "value": n_rows * ticks * samples / total,
        "agents": n_rows,
        "sample_s": per_sample,
        "procs": P,
        "ticks_per_sample": ticks,
        "samples": samples,
        "per_core_median": per_core[len(per_core) // 2],
        "faults": sum(res[i][1] for i in range(P)),
        "wall_s": wall,
    }
