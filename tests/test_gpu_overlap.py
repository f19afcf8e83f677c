"""Overlapped step launches (swarmstep_quad_step_overlapped, programmatic
dependent launch with per-tile epochs): a chain of step_async launches that
overlap one another -- interleaved with setpoint uploads, single commands,
kills and host reads -- leaves the device state bit-identical to the same
sequence launched with full stream ordering."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


class _Cmd:
    def __init__(self, agent_id, level, values):
        self.agent_id, self.level, self.values = agent_id, level, values


def _groups(n, seed):
    import torch

    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    from paper_2308_12698_b200.synthetic import swarm
    pos, sp = swarm(n, seed=seed)
    out = []
    for overlap in (True, False):
        g = B200QuadGroup(0, batch_create(0, n, pos))
        g.overlap_launches = overlap
        g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
        out.append(g)
    return out


def _device_state(g):
    import torch
    torch.cuda.synchronize()
    return g.cols.cpu().numpy().copy(), g.flags.cpu().numpy().copy()


@pytest.mark.parametrize("n", [1000, 400_000])
def test_overlapped_chain_bit_identical(n):
    import torch

    from paper_2308_12698_b200.commands import LEVEL_RATE
    rng = np.random.default_rng(n)
    a, b = _groups(n, seed=3)
    rate = rng.uniform(-1, 1, (n // 4, 4)).astype(np.float32)
    rate[:, 0] = 9.81 * 0.5 + rng.uniform(0, 4, n // 4)
    for g in (a, b):
        g.set_setpoints(torch.from_numpy(rate).cuda(), level=LEVEL_RATE, row0=n // 2)
    plan = [(1, None), (10, None), (10, "cmd"), (3, None), (10, "kill"), (1, None), (10, "rate"), (10, None),
            (2, "read"), (10, None), (10, None)]
    for k, between in plan:
        for g in (a, b):
            g.step_async(1e-3, k)
            if between == "cmd":
                g.apply_command(_Cmd(7, "pos", (1.0, 2.0, 3.0, 0.1, 0.0, 0.0, 0.0)))
                g.apply_command(_Cmd(n - 1, "rate", (0.2, -0.1, 0.05, 6.0)))
            elif between == "kill":
                g.mark_dead([3, n // 2 + 1])
            elif between == "rate":
                g.set_setpoints(torch.from_numpy(rate[::-1].copy()).cuda(), level=LEVEL_RATE, row0=n // 2)
            elif between == "read":
                g.batch.pos
    fa, fb = a.collect_faults(), b.collect_faults()
    assert [x.tolist() for x in fa] == [x.tolist() for x in fb]
    assert a._pdl_epoch == sum(k >= 4 for k, _ in plan) and b._pdl_epoch == 0
    ca, fla = _device_state(a)
    cb, flb = _device_state(b)
    np.testing.assert_array_equal(fla, flb)
    assert ca.tobytes() == cb.tobytes()


def test_overlapped_long_chain_matches_ordered():
    """100 back-to-back overlapped K = 4 launches over 1M agents (7813 tiles,
    several waves per launch, so consecutive launches do overlap)."""
    a, b = _groups(1_000_000, seed=8)
    for _ in range(100):
        a.step_async(1e-3, 4)
        b.step_async(1e-3, 4)
    a.collect_faults(), b.collect_faults()
    ca, fla = _device_state(a)
    cb, flb = _device_state(b)
    np.testing.assert_array_equal(fla, flb)
    assert ca.tobytes() == cb.tobytes()


def test_overlapped_circle_feed_chain():
    """Fused circle-feed launches share the group's overlap chain with plain
    step launches: the mixed sequence is bit-identical to ordered launches."""
    from paper_2308_12698_b200.feed import CircleFeed
    a, b = _groups(300_000, seed=4)
    fa, fb = CircleFeed(a, 1e-3), CircleFeed(b, 1e-3)
    for feed, g in ((fa, a), (fb, b)):
        for _ in range(3):
            feed.step_fused(10)
        g.step_async(1e-3, 10)
        feed.step_fused(5)
        g.step_async(1e-3, 1)
        feed.step_fused(10)
        feed.step_fused(2)
        feed.step_fused(10)
        g.collect_faults()
    assert a._pdl_epoch == 7 and b._pdl_epoch == 0
    ca, fla = _device_state(a)
    cb, flb = _device_state(b)
    np.testing.assert_array_equal(fla, flb)
    assert ca.tobytes() == cb.tobytes()


def test_overlapped_chain_with_faults():
    """Rows that fault inside overlapped launches (non-finite setpoints, the
    per-row re-execution path) report the same ticks and leave the same bits
    as with ordered launches."""
    import torch

    from paper_2308_12698_b200.commands import LEVEL_POS
    n = 200_000
    a, b = _groups(n, seed=6)
    rng = np.random.default_rng(6)
    bad_rows = np.sort(rng.choice(n, 40, replace=False))
    for i, g in enumerate((a, b)):
        g.step_async(1e-3, 10)
        for j, r in enumerate(bad_rows[:20]):
            vals = torch.full((1, 7), float("nan") if j % 2 else float("inf"), device="cuda")
            g.set_setpoints(vals, level=LEVEL_POS, row0=int(r))
        g.step_async(1e-3, 10)
        g.step_async(1e-3, 10)
        for r in bad_rows[20:]:
            g.set_setpoints(torch.full((1, 7), 1e30, device="cuda"), level=LEVEL_POS, row0=int(r))
        for _ in range(4):
            g.step_async(1e-3, 10)
    fa, fb = a.collect_faults(), b.collect_faults()
    assert [x.tolist() for x in fa] == [x.tolist() for x in fb]
    assert sum(x.size for x in fa) >= 20
    ca, fla = _device_state(a)
    cb, flb = _device_state(b)
    np.testing.assert_array_equal(fla, flb)
    assert ca.tobytes() == cb.tobytes()


def test_overlapped_chain_around_graph_replays():
    """CUDA-graph tick loops (plain launches) between overlapped launches: the
    chain resumes on the epoch it left, bit-identical to ordered launches."""
    from paper_2308_12698_b200.feed import CircleFeed, TickGraph
    a, b = _groups(300_000, seed=9)
    for g in (a, b):
        feed = CircleFeed(g, 1e-3)
        g.step_async(1e-3, 10)
        tg = TickGraph(g, 1e-3, 5, feed=feed)
        tg.replay()
        g.step_async(1e-3, 10)
        feed.step_fused(10)
        tg.replay()
        tg.replay()
        g.step_async(1e-3, 8)
        g.collect_faults()
    assert a._pdl_epoch == 4 and b._pdl_epoch == 0
    ca, fla = _device_state(a)
    cb, flb = _device_state(b)
    np.testing.assert_array_equal(fla, flb)
    assert ca.tobytes() == cb.tobytes()
