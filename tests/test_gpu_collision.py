"""GPU collision / neighbour detection (f3) against the reference's detect()
golden output (tests/golden/collision.npz, collision.py:110-176) and the
all-pairs float64 oracle, exactly."""

import numpy as np
import pytest

from conftest import cuda_ok
from golden_io import GOLDEN
from oracle import oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]


def _group(type_id, pos, alive, id_base):
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    n = pos.shape[0]
    g = B200QuadGroup(type_id, batch_create(type_id, n, pos, id_base=id_base))
    dead = (np.nonzero(~alive)[0] + id_base).tolist()
    if dead:
        g.mark_dead(dead)
    return g


def _world(z, w):
    pre = f"w{w}_"
    p0, p1, a0, a1 = z[pre + "p0"], z[pre + "p1"], z[pre + "a0"], z[pre + "a1"]
    r0, r1, r_sense, cell = (float(x) for x in z[pre + "cfg"])
    keys, lens, flat = z[pre + "nb_keys"], z[pre + "nb_len"], z[pre + "nb_ids"]
    nb, o = {}, 0
    for k, ln in zip(keys, lens):
        nb[int(k)] = tuple(int(x) for x in flat[o:o + ln])
        o += ln
    coll = tuple(tuple(int(x) for x in r) for r in z[pre + "coll"])
    return p0, p1, a0, a1, (r0, r1, r_sense, cell), coll, nb


def test_matches_reference_detect_golden():
    from paper_2308_12698_b200.collision import CollisionConfig, GpuDetector
    z = dict(np.load(GOLDEN / "collision.npz"))
    n_pairs = 0
    for w in range(int(z["worlds"])):
        p0, p1, a0, a1, (r0, r1, r_sense, cell), coll, nb = _world(z, w)
        groups = [_group(0, p0, a0, 0)]
        if p1.shape[0]:
            groups.append(_group(1, p1, a1, p0.shape[0]))
        cfg = CollisionConfig(r_collide={0: r0, 1: r1}, r_sense=r_sense, cell=cell)
        rep = GpuDetector(cfg, groups[0].device).detect(groups, tick=w)
        assert rep.collisions == coll, w
        assert rep.neighbor_sets == nb, w
        n_pairs += len(coll)
    assert n_pairs > 0


@pytest.mark.parametrize("n,box,seed", [(4000, 20.0, 1), (20000, 40.0, 2)])
def test_matches_all_pairs_oracle_after_steps(n, box, seed):
    """Unquantised positions after a few ticks (hi + lo): exact against the oracle
    evaluated on the group's own float64 mirror."""
    from paper_2308_12698_b200.collision import CollisionConfig, detect
    rng = np.random.default_rng(seed)
    g = _group(0, rng.uniform(0, box, (n, 3)) + [0, 0, 5], rng.random(n) > 0.05, 0)
    for _ in range(5):
        g.step(2e-3)
    cfg = CollisionConfig(r_collide={0: 0.15}, r_sense=1.0, cell=0.5)
    rep = detect([g], cfg, tick=5)
    b = g.batch
    rows = np.arange(n)
    if n > 5000:   # the O(N^2) oracle on a sub-box keeps the test fast
        inside = np.all((b.pos >= [10, 10, 15]) & (b.pos < [20, 20, 25]), axis=1)
        rows = np.nonzero(inside)[0]
    pairs, nbrs = orc.collide_all_pairs(b.agent_ids[rows], b.pos[rows], np.full(rows.size, 0.15),
                                        b.alive[rows], 1.0)
    if rows.size == n:
        assert list(rep.collisions) == pairs
        assert rep.neighbor_sets == nbrs
    else:
        # agents well inside the sub-box have all their neighbours in it
        core = np.all((b.pos[rows] >= [11, 11, 16]) & (b.pos[rows] < [19, 19, 24]), axis=1) & b.alive[rows]
        for i in b.agent_ids[rows][core]:
            assert rep.neighbor_sets[int(i)] == nbrs[int(i)]
        assert {p for p in rep.collisions if p[0] in set(b.agent_ids[rows].tolist())
                and p[1] in set(b.agent_ids[rows].tolist())} == set(pairs)


def test_degenerate_worlds():
    from paper_2308_12698_b200.collision import CollisionConfig, detect
    cfg = CollisionConfig(r_collide={0: 0.5}, r_sense=1.0, cell=1.0)
    g = _group(0, np.array([[0.0, 0.0, 5.0]]), np.array([True]), 7)
    rep = detect([g], cfg, tick=0)
    assert rep.collisions == () and rep.neighbor_sets == {7: ()}
    # exact contact is not a collision (test_collision.py:77-83)
    g = _group(0, np.array([[0.0, 0.0, 5.0], [1.0, 0.0, 5.0]]), np.array([True, True]), 0)
    rep = detect([g], cfg, tick=0)
    assert rep.collisions == () and rep.neighbor_sets == {0: (), 1: ()}
    g = _group(0, np.array([[0.0, 0.0, 5.0], [0.5, 0.0, 5.0], [0.25, 0.0, 5.0]]), np.array([True, False, True]), 0)
    rep = detect([g], cfg, tick=0)
    assert rep.collisions == ((0, 2),) and rep.neighbor_sets == {0: (2,), 2: (0,)}


def _snapshot(z, w, tick):
    from paper_2308_12698_b200.state import BatchSnapshot, WorldSnapshot
    p0, p1, a0, a1, cfgv, coll, nb = _world(z, w)
    bs = [BatchSnapshot(tick=tick, type_id=0, agent_ids=np.arange(p0.shape[0], dtype=np.uint64), pos=p0,
                        vel=np.zeros_like(p0), quat=np.tile([1.0, 0, 0, 0], (p0.shape[0], 1)),
                        omega=np.zeros_like(p0), alive=a0)]
    if p1.shape[0]:
        n0 = p0.shape[0]
        bs.append(BatchSnapshot(tick=tick, type_id=1, agent_ids=np.arange(n0, n0 + p1.shape[0], dtype=np.uint64),
                                pos=p1, vel=np.zeros_like(p1), quat=np.tile([1.0, 0, 0, 0], (p1.shape[0], 1)),
                                omega=np.zeros_like(p1), alive=a1))
    return WorldSnapshot(tick=tick, batches=tuple(bs)), cfgv, coll, nb


def test_snapshot_detector_matches_reference_detect_golden():
    """GpuDetector.detect_snapshot: the reference's detect(snapshot, config)
    signature (the out-of-loop detector's input, any groups) on the GPU."""
    from paper_2308_12698_b200.collision import CollisionConfig, GpuDetector
    z = dict(np.load(GOLDEN / "collision.npz"))
    for w in range(int(z["worlds"])):
        snap, (r0, r1, r_sense, cell), coll, nb = _snapshot(z, w, tick=w)
        cfg = CollisionConfig(r_collide={0: r0, 1: r1}, r_sense=r_sense, cell=cell)
        rep = GpuDetector(cfg, "cuda:0").detect_snapshot(snap, dropped=3)
        assert rep.tick == w and rep.dropped == 3
        assert rep.collisions == coll, w
        assert rep.neighbor_sets == nb, w


def test_snapshot_detector_validation_and_run_detector_semantics():
    """collision.py:66-80 validation and run_detector's jump-to-newest /
    dropped counting / sentinel echo (collision.py:179-215, test_collision.py:
    140-175)."""
    import dataclasses
    import queue

    from paper_2308_12698_b200.collision import CollisionConfig, GpuDetector, run_detector
    from paper_2308_12698_b200.errors import ValidationError
    from paper_2308_12698_b200.state import WorldSnapshot
    z = dict(np.load(GOLDEN / "collision.npz"))
    snap, (r0, r1, r_sense, cell), coll, nb = _snapshot(z, 0, tick=4)
    cfg = CollisionConfig(r_collide={0: r0, 1: r1}, r_sense=r_sense, cell=cell)
    det = GpuDetector(cfg, "cuda:0")
    bad = WorldSnapshot(tick=5, batches=snap.batches)
    with pytest.raises(ValidationError):
        det.detect_snapshot(bad)                                  # sections disagree on tick
    with pytest.raises(ValidationError):
        GpuDetector(CollisionConfig(r_collide={0: r0}, r_sense=r_sense, cell=cell), "cuda:0").detect_snapshot(
            WorldSnapshot(tick=4, batches=tuple(dataclasses.replace(b, type_id=7) for b in snap.batches[:1])))
    in_q, out_q = queue.Queue(), queue.Queue()
    snaps = [WorldSnapshot(tick=t, batches=tuple(dataclasses.replace(b, tick=t) for b in snap.batches))
             for t in range(3)]
    for s in snaps:
        in_q.put(s)
    in_q.put(None)
    run_detector(in_q, out_q, cfg, "cuda:0")
    reports = []
    while (r := out_q.get_nowait()) is not None:
        reports.append(r)
    assert [r.tick for r in reports] == [0, 2] and [r.dropped for r in reports] == [0, 1]
    assert all(r.collisions == coll for r in reports)
