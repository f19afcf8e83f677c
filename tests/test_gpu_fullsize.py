"""Parity at the bench's full size (10M quadrotors per GPU, bench.py's workload)
through size-independent properties, read on the device without pulling the
whole float64 mirror:

  * K fused ticks == K single ticks, bit for bit, over the whole column block;
  * a 4096-row sample steps like the float64 oracle (per-step rel. error <= 1e-5)
    from the GPU's own pre-step state (rows are independent, quad.py:6-7);
  * dead rows stay bit-frozen and nothing faults."""

import numpy as np
import pytest
import torch

from conftest import cuda_ok
from gpu_util import PER_STEP_TOL, f32, oracle_twin, rel_errors

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

N = 10_000_000


def _group(compensated=True):
    from bench import _Batch
    from paper_2308_12698_b200 import B200QuadGroup
    from paper_2308_12698_b200.synthetic import swarm
    pos, sp = swarm(N)
    g = B200QuadGroup(0, _Batch(N, pos, 0), device="cuda:0", compensated=compensated)
    g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
    return g


def _rows_state(g, rows):
    """float64 state / PID / command columns of `rows`, read from the device."""
    from paper_2308_12698_b200._lib import (COL_CMD, COL_INTEGRAL, COL_OMEGA, COL_POS, COL_POS_LO, COL_PREV,
                                            COL_QUAT, COL_SP, COL_VEL, FLAG_ALIVE, FLAG_HAS_PREV, LEVEL_MASK,
                                            LEVEL_SHIFT)
    from paper_2308_12698_b200._lib import pos_lo_decode
    r = torch.as_tensor(rows, device=g.device)
    raw = g.cols[r >> 7, :, r & 127].cpu().numpy()                   # (len, NCOL) float32
    blk = raw.astype(np.float64)
    fl = g.flags[r].cpu().numpy()

    def c(a, k):
        return blk[:, a:a + k].copy()
    lo = pos_lo_decode(raw[:, COL_POS_LO].view(np.uint32), raw[:, COL_POS:COL_POS + 3])
    return dict(pos=c(COL_POS, 3) + lo, vel=c(COL_VEL, 3), quat=c(COL_QUAT, 4),
                omega=c(COL_OMEGA, 3), alive=(fl & FLAG_ALIVE) != 0, integral=c(COL_INTEGRAL, 3),
                prev_omega=c(COL_PREV, 3), has_prev=(fl & FLAG_HAS_PREV) != 0, omega_sp=c(COL_SP, 3),
                f_c_sp=c(COL_SP + 3, 1)[:, 0], cmd_level=((fl & LEVEL_MASK) >> LEVEL_SHIFT).astype(np.uint8),
                cmd_values=c(COL_CMD, 7))


def test_full_size_fused_equals_single_ticks():
    """10M agents: one K=10 launch == ten one-tick launches, bit for bit, with a
    plain float32 position (with the compensated position the two differ only
    in where the low part is folded -- gpu_util.FUSION_TOL, asserted on the
    parity scenarios; at this size a handful of the random-setpoint rows sit
    on the reference's own free-fall discontinuity, control.py:243-247, where
    any rounding difference switches branch)."""
    a = _group(compensated=False)
    a.mark_dead(list(range(0, N, 1_000_003)))
    a.step_k(1e-3, 10)
    frozen_rows = np.arange(0, N, 1_000_003)
    dead_before = _rows_state(a, frozen_rows)
    b = _group(compensated=False)
    b.mark_dead(list(range(0, N, 1_000_003)))
    b.step_k(1e-3, 10)
    assert torch.equal(a.cols, b.cols) and torch.equal(a.flags, b.flags)
    a.step_k(1e-3, 10)
    for _ in range(10):
        b.step(1e-3)
    assert torch.equal(a.cols, b.cols) and torch.equal(a.flags, b.flags)
    assert a.alive_count() == N - frozen_rows.size
    dead_after = _rows_state(a, frozen_rows)
    for k in ("pos", "vel", "quat", "omega", "integral"):
        np.testing.assert_array_equal(dead_after[k], dead_before[k])
    del a, b
    torch.cuda.empty_cache()


def test_full_size_sampled_rows_vs_oracle():
    g = _group()
    g.step_k(1e-3, 10)
    rows = np.sort(np.random.default_rng(9).choice(N, 4096, replace=False))
    og = oracle_twin(None, _rows_state(g, rows))
    g.step(1e-3)
    og.step(f32(1e-3))
    e = rel_errors(_rows_state(g, rows), og)
    for k, v in e.items():
        assert v <= PER_STEP_TOL, f"{k}: {v:.2e}"
    del g
    torch.cuda.empty_cache()
