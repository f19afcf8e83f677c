"""The hot path driven from plain C through the C ABI (tools/c_host_demo.c:
params_init -> unpack -> bulk setpoints -> fused launches -> pack) gives the
same bits as the same workload through B200QuadGroup."""

import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

DEMO = Path(__file__).resolve().parent.parent / "tools" / "c_host_demo"


@pytest.mark.parametrize("n,k,launches,overlap", [(1000, 10, 10, 0), (300, 1, 7, 0), (200_000, 10, 12, 1)])
def test_c_host_matches_python_group(n, k, launches, overlap, tmp_path):
    if not DEMO.exists():
        pytest.fail("tools/c_host_demo not built (run __graft_entry__.build())")
    dump = tmp_path / "pos.bin"
    out = subprocess.run([str(DEMO), str(n), str(k), str(launches), str(dump), str(overlap)], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    c = json.loads(out.stdout.strip().splitlines()[-1])

    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    from paper_2308_12698_b200.layout import layout_poses
    pos, _ = layout_poses({"kind": "grid", "spacing": 3.0, "origin": (0.0, 0.0, 10.0)}, n)
    g = B200QuadGroup(0, batch_create(0, n, pos))
    sp = np.zeros((n, 7), dtype=np.float32)
    sp[:, 0] = (pos[:, 0] + 0.25).astype(np.float32)
    sp[:, 1] = pos[:, 1].astype(np.float32)
    sp[:, 2] = (pos[:, 2] + 0.5).astype(np.float32)
    sp[:, 6] = np.float32(0.1)
    g.set_setpoints(sp)
    for _ in range(launches):
        g.step_k(1e-3, k)
    p = g.batch.pos
    assert c["abi"] == 3 and c["alive"] == n and c["faults"] == 0
    np.testing.assert_array_equal(np.fromfile(dump, dtype=np.float64).reshape(n, 3), p)
