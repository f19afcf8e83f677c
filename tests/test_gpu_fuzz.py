"""Randomised parity fuzzing of the fused step against the float64 oracle.

Each seed draws a swarm size (including sizes that leave partial 128-row
tiles and odd pair partners), per-agent levels (POS / RATE / MOTOR, including
saturating and free-fall commands), tilts, rates, deaths, overlays and fault
injections, then checks (a) every step against the oracle twin (per-step
relative error <= 1e-5, identical fault ids) and (b) that the direct, paired
and TMA kernels and K-fused launches agree bit for bit."""

import os

import numpy as np
import pytest

from paper_2308_12698_b200._lib import COL_OVERLAY

from conftest import cuda_ok
from gpu_util import PER_STEP_TOL, f32, gpu_state, oracle_twin, rel_errors
from scenarios import Scenario

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

HOVER = 9.81
# SWARMSTEP_FUZZ_SEEDS=200 for a soak run (profiles/fuzz_soak_r01.txt)
N_SEEDS = int(os.environ.get("SWARMSTEP_FUZZ_SEEDS", "12"))


def _random_swarm(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 63, 64, 65, 127, 129, 200, 383]))
    q = rng.standard_normal((n, 4))
    tilt = rng.uniform(0, 1, n) < 0.5
    q[~tilt] = [1, 0, 0, 0]
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = Scenario(f"fuzz{seed}", n, float(rng.choice([1e-3, 2e-3, 5e-3])), 1,
                  rng.uniform(-120, 120, (n, 3)), rng.uniform(-4, 4, (n, 3)), q, rng.uniform(-3, 3, (n, 3)),
                  record=[])
    return rng, sc


def _commands(rng, g, sc):
    from paper_2308_12698_b200 import AgentCommand, CommandLevel
    n = sc.n
    for i in range(n):
        kind = rng.integers(0, 6)
        if kind == 0:      # POS near the agent
            vals = tuple(sc.pos[i] + rng.uniform(-3, 3, 3)) + tuple(rng.uniform(-2, 2, 3)) + (rng.uniform(-3.1, 3.1),)
            g.apply_command(AgentCommand(i, CommandLevel.POS, vals))
        elif kind == 1:    # POS far away (saturating outer loop)
            vals = tuple(sc.pos[i] + rng.uniform(-200, 200, 3)) + (0.0, 0.0, 0.0, rng.uniform(-3.1, 3.1))
            g.apply_command(AgentCommand(i, CommandLevel.POS, vals))
        elif kind == 2:    # RATE, possibly saturating the mixer
            vals = tuple(rng.uniform(-8, 8, 3)) + (rng.uniform(0, 80),)
            g.apply_command(AgentCommand(i, CommandLevel.RATE, vals))
        elif kind == 3:    # MOTOR speeds, including out of range
            g.apply_command(AgentCommand(i, CommandLevel.MOTOR, tuple(rng.uniform(-5e3, 5e4, 4))))
        elif kind == 4:    # free fall (zero thrust)
            g.apply_command(AgentCommand(i, CommandLevel.RATE, (0.0, 0.0, 0.0, 0.0)))
        # kind 5: keep the default position hold
    dead = rng.choice(n, size=int(rng.integers(0, max(1, n // 10) + 1)), replace=False)
    g.mark_dead([int(d) for d in dead])


@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_fuzz_per_step_against_oracle(seed):
    from gpu_util import make_group
    rng, sc = _random_swarm(seed)
    g = make_group(sc)
    _commands(rng, g, sc)
    worst = {}
    for t in range(12):
        if rng.uniform() < 0.3:
            g.add_velocity_overlay(rng.uniform(-1, 1, (sc.n, 3)))
        og = oracle_twin(g)
        if g._overlay_active:
            og.add_velocity_overlay(g.column_block(COL_OVERLAY, COL_OVERLAY + 3).double().cpu().numpy().astype(np.float32).astype(float))
        og_f = og.step(f32(sc.dt))
        g_f = g.step(sc.dt)
        assert sorted(g_f.tolist()) == sorted(og_f.tolist()), f"tick {t}: fault ids differ"
        e = rel_errors(gpu_state(g), og)
        for k, v in e.items():
            worst[k] = max(worst.get(k, 0.0), v)
    for k, v in worst.items():
        assert v <= PER_STEP_TOL, f"seed {seed}: per-step {k} rel err {v:.2e}"


@pytest.mark.parametrize("compensated", [False, True])
@pytest.mark.parametrize("seed", range(max(6, N_SEEDS // 2)))
def test_fuzz_kernels_and_fusion_bit_identical(seed, compensated):
    """Every kernel variant gives identical bits at the same ticks per launch;
    fusing ticks is bit-identical with a plain float32 position and equal up to
    the compensated low part's fold / storage rounding otherwise (FUSION_TOL)."""
    from gpu_util import assert_fusion_close, make_group
    outs = {}
    for kern, k in (("direct", 1), ("direct", 7), ("pair", 7), ("tma", 7), ("pair", 1)):
        rng, sc = _random_swarm(100 + seed)
        g = make_group(sc, compensated=compensated)
        g.kernel = kern
        _commands(rng, g, sc)
        for _ in range(14 // k):
            g.step_k(sc.dt, k)
        st = gpu_state(g)
        outs[(kern, k)] = {q: st[q].copy() for q in ("pos", "vel", "quat", "omega", "integral", "prev_omega",
                                                     "alive")}
    ref = {1: outs[("direct", 1)], 7: outs[("direct", 7)]}
    for (kern, k), o in outs.items():
        for q in o:
            np.testing.assert_array_equal(ref[k][q], o[q], err_msg=f"{kern} K={k} {q}")
    for q in ref[1]:
        if not compensated or q == "alive":
            np.testing.assert_array_equal(ref[1][q], ref[7][q], err_msg=f"fused {q}")
    if compensated:
        assert_fusion_close(ref[1], ref[7], ("pos", "vel", "quat", "omega", "integral", "prev_omega"))


def _asym_params():
    """A vehicle that is NOT axisymmetric (I_xx != I_yy, different x / y
    gains): the general step kernels, not the axisymmetric instantiation."""
    from paper_2308_12698_b200.params import OuterGains, PidGains, QuadParams
    quad = QuadParams(m=1.2, i_diag=(0.011, 0.0093, 0.021))
    rate = PidGains(kp=(0.27, 0.22, 0.11), ki=(0.05, 0.04, 0.02), kd=(0.0021, 0.0018, 0.001),
                    i_limit=(0.2, 0.15, 0.2))
    outer = OuterGains(kp_pos=(15.0, 17.0, 16.0), kv=(8.0, 7.5, 8.5), k_att=(12.0, 11.0, 3.0))
    return quad, rate, outer


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_non_axisymmetric_vehicle_per_step(seed):
    """Per-step parity (and identical fault ids) for a non-axisymmetric vehicle,
    paired (K = 7) and direct kernels alike."""
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    params = _asym_params()
    rng, sc = _random_swarm(300 + seed)
    g = B200QuadGroup(0, batch_create(0, sc.n, sc.pos, quat=sc.quat, vel=sc.vel, omega=sc.omega), *params)
    _commands(rng, g, sc)
    g.step_k(sc.dt, 7)                     # the paired kernel on the general (non-AXI) instantiation
    worst = {}
    for t in range(6):
        og = oracle_twin(g, params=params)
        og_f = og.step(f32(sc.dt))
        g_f = g.step(sc.dt)
        assert sorted(g_f.tolist()) == sorted(og_f.tolist()), f"tick {t}: fault ids differ"
        for k, v in rel_errors(gpu_state(g), og).items():
            worst[k] = max(worst.get(k, 0.0), v)
    for k, v in worst.items():
        assert v <= PER_STEP_TOL, f"seed {seed}: per-step {k} rel err {v:.2e}"


@pytest.mark.parametrize("seed", range(3))
def test_non_axisymmetric_kernels_bit_identical(seed):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    params = _asym_params()
    outs = []
    for kern in ("direct", "pair", "tma"):
        rng, sc = _random_swarm(400 + seed)
        g = B200QuadGroup(0, batch_create(0, sc.n, sc.pos, quat=sc.quat, vel=sc.vel, omega=sc.omega), *params)
        g.kernel = kern
        _commands(rng, g, sc)
        for _ in range(2):
            g.step_k(sc.dt, 5)
        st = gpu_state(g)
        outs.append({q: st[q].copy() for q in ("pos", "vel", "quat", "omega", "integral", "alive")})
    for o in outs[1:]:
        for q in o:
            np.testing.assert_array_equal(outs[0][q], o[q], err_msg=q)
