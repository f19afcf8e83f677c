"""GPU checks of the neighbour-coupled swarm controller (config 5): the device
spatial-hash separation overlay against the float64 all-pairs oracle, at small
size and at the config-5 size (100k agents, sampled rows)."""

import numpy as np
import pytest

from paper_2308_12698_b200._lib import COL_OVERLAY

from conftest import cuda_ok
from gpu_util import make_group
from oracle import oracle as orc
from scenarios import Scenario

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _swarm(n, box, seed=0):
    rng = np.random.default_rng(seed)
    q = np.tile([1.0, 0, 0, 0], (n, 1))
    return Scenario("swarm", n, 1e-3, 1, rng.uniform(0, box, (n, 3)) + [0, 0, 5], np.zeros((n, 3)), q,
                    np.zeros((n, 3)), record=[])


def _overlay(g):
    return g.column_block(COL_OVERLAY, COL_OVERLAY + 3).double().cpu().numpy()


def _positions(g):
    return g.batch.pos.copy(), g.batch.alive.copy()


@pytest.mark.parametrize("n,box", [(3000, 15.0), (257, 4.0)])
def test_overlay_matches_all_pairs_oracle(n, box):
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    g = make_group(_swarm(n, box))
    g.mark_dead([1, 7, n - 1])
    ns = NeighborSeparation(g, make_shard(n), r_sense=2.0, k_sep=1.5)
    ns.apply()
    got = _overlay(g)
    pos, alive = _positions(g)
    want = orc.neighbor_overlay(pos, alive, 2.0, 1.5)
    scale = np.max(np.abs(want))
    assert scale > 0.1
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-5 * scale)
    assert np.all(got[~alive] == 0.0)


def test_overlay_deterministic_and_one_tick():
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    sc = _swarm(2000, 12.0, seed=3)
    outs = []
    for _ in range(2):
        g = make_group(sc)
        ns = NeighborSeparation(g, make_shard(sc.n), r_sense=2.0, k_sep=1.0)
        ns.apply()
        ov = _overlay(g)
        assert np.abs(ov).sum() > 0
        outs.append(ov.tobytes())
        ns.group.step(1e-3)
        assert np.all(_overlay(g) == 0.0)          # cleared after the tick (core.py:199-201)
    assert outs[0] == outs[1]


def test_coupled_steps_push_neighbours_apart():
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    sc = _swarm(500, 3.0, seed=4)
    g = make_group(sc)
    ns = NeighborSeparation(g, make_shard(sc.n), r_sense=2.0, k_sep=2.0)

    def mean_nn(pos):
        d = np.linalg.norm(pos[:, None] - pos[None], axis=2) + np.eye(len(pos)) * 1e9
        return d.min(axis=1).mean()

    d0 = mean_nn(g.batch.pos)
    for _ in range(300):
        ns.step(2e-3)
    assert mean_nn(g.batch.pos) > d0
    assert g.batch.alive.all()


def test_config5_size_sampled_rows():
    """100k agents (config 5), r_sense 2 m: sampled rows vs the all-pairs oracle."""
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    n = 100_000
    sc = _swarm(n, 60.0, seed=5)
    g = make_group(sc)
    ns = NeighborSeparation(g, make_shard(n), r_sense=2.0, k_sep=1.0)
    ns.apply()
    got = _overlay(g)
    pos, alive = _positions(g)
    rows = np.random.default_rng(6).choice(n, 1024, replace=False)
    want = orc.neighbor_overlay(pos, alive, 2.0, 1.0, rows=rows)
    scale = np.max(np.abs(want))
    np.testing.assert_allclose(got[rows], want, rtol=1e-4, atol=1e-5 * scale)


def test_graph_captured_coupling_matches_eager():
    """Exchange + overlay + step captured in a CUDA graph == the eager loop, bitwise."""
    from paper_2308_12698_b200.feed import TickGraph
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    sc = _swarm(1500, 9.0, seed=8)
    ga, gb = make_group(sc), make_group(sc)
    na = NeighborSeparation(ga, make_shard(sc.n), r_sense=2.0, k_sep=1.0)
    nb = NeighborSeparation(gb, make_shard(sc.n), r_sense=2.0, k_sep=1.0)
    graph = TickGraph(ga, 1e-3, 20, coupling=na)
    for _ in range(3):
        graph.replay()
    ga.collect_faults()
    for _ in range(60):
        nb.step(1e-3)
    for k in ("pos", "vel", "quat", "omega"):
        np.testing.assert_array_equal(getattr(ga.batch, k), getattr(gb.batch, k), err_msg=k)
    assert np.all(_overlay(ga) == 0.0)


def test_swarm_stats_match_host_reduction():
    """Device swarm-wide reductions (alive count of World.alive_counts,
    core.py:370; centroid; speeds; alive bounding box) == numpy over the
    float64 mirror, deterministic run to run, dead rows excluded."""
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    rng = np.random.default_rng(11)
    for n in (1, 300, 200_003):
        pos = rng.uniform(-50, 50, (n, 3))
        g = B200QuadGroup(0, batch_create(0, n, pos, vel=rng.uniform(-2, 2, (n, 3))))
        g.mark_dead(list(range(0, n, 7)))
        g.step_k(1e-3, 3)
        st = g.swarm_stats()
        b = g.batch
        al = b.alive
        assert st["alive"] == int(al.sum())
        if al.any():
            np.testing.assert_allclose(st["centroid"], b.pos[al].mean(axis=0), rtol=1e-12, atol=1e-9)
            np.testing.assert_allclose(st["bbox_min"], b.pos[al].astype(np.float32).min(axis=0), rtol=0, atol=0)
            np.testing.assert_allclose(st["bbox_max"], b.pos[al].astype(np.float32).max(axis=0), rtol=0, atol=0)
            sp2 = np.sum(b.vel[al] ** 2, axis=1)
            np.testing.assert_allclose(st["mean_speed_sq"], sp2.mean(), rtol=1e-6)
            np.testing.assert_allclose(st["max_speed"], np.sqrt(sp2.max()), rtol=1e-6)
        else:
            assert np.all(np.isinf(st["bbox_min"]))
        st2 = g.swarm_stats()
        assert st2["centroid"].tobytes() == st["centroid"].tobytes()


@pytest.fixture
def one_rank_group():
    """A 1-rank torch.distributed group (the P2P exchange needs one for its
    symmetric-memory rendezvous); world 1 runs the fused pack + peer-store +
    signal + wait path with this GPU as the only peer."""
    import socket

    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        yield dist.group.WORLD
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        yield dist.group.WORLD
    finally:
        dist.destroy_process_group()


def test_p2p_exchange_equals_nccl_path(one_rank_group):
    """The fused P2P exchange (csrc/exchange.cu) gathers exactly the positions
    the pack + all-gather path does, epoch after epoch (both slots of its
    double buffer), eager and inside a CUDA graph: identical trajectories."""
    import torch
    from paper_2308_12698_b200.feed import TickGraph
    from paper_2308_12698_b200.parallel import NeighborSeparation, make_shard
    sc = _swarm(3000, 14.0, seed=5)
    ga, gb = make_group(sc), make_group(sc)
    ga.mark_dead([3, 99])
    gb.mark_dead([3, 99])
    na = NeighborSeparation(ga, make_shard(sc.n), r_sense=2.0, k_sep=1.0, exchange="nccl")
    nb = NeighborSeparation(gb, make_shard(sc.n), r_sense=2.0, k_sep=1.0, exchange="p2p")
    for t in range(5):
        na.apply()
        nb.apply()
        assert na.gathered_positions().cpu().numpy().tobytes() == nb.gathered_positions().cpu().numpy().tobytes()
        assert _overlay(ga).tobytes() == _overlay(gb).tobytes()
        ga.step(1e-3)
        gb.step(1e-3)
    assert int(nb._epoch.item()) == 5
    ta, tb = TickGraph(ga, 1e-3, 7, coupling=na), TickGraph(gb, 1e-3, 7, coupling=nb)
    for _ in range(3):                      # odd tick count: the slot parity alternates across replays
        ta.replay()
        tb.replay()
    torch.cuda.synchronize()
    sa, sb = ga.batch, gb.batch
    assert sa.pos.tobytes() == sb.pos.tobytes() and sa.vel.tobytes() == sb.vel.tobytes()
    assert int(nb._epoch.item()) == 5 + 7 * 3   # capture records only; 3 replays of 7 ticks
