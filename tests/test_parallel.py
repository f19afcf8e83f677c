"""Host-side multi-rank logic on CPU (gloo, world_size 2): shard ranges, id
routing, fault-id gathering, and the position all-gather layout the GPU
neighbour controller relies on (padding + self offset), checked against the
all-pairs float64 oracle of the whole swarm."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_2308_12698_b200.parallel import ShardedSwarm, make_shard, shard_range, shard_sizes


def test_shard_ranges_cover_and_balance():
    for n in (0, 1, 7, 100, 10_000_001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sz = shard_sizes(n, w)
            assert max(sz) - min(sz) <= 1 and sum(sz) == n
    s = make_shard(10, 1, 3)
    assert (s.lo, s.hi, s.pad, s.self_offset, s.n_gathered) == (4, 7, 4, 4, 12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _FakeGroup:
    """Rank-local stand-in for B200QuadGroup (CPU): numpy positions + fault injection."""

    def __init__(self, lo, hi, fault_ids=()):
        self.lo, self.hi = lo, hi
        self.alive = np.ones(hi - lo, dtype=bool)
        self.faults = [f for f in fault_ids if lo <= f < hi]
        self.applied = []

    def apply_command(self, cmd):
        self.applied.append(int(cmd.agent_id))
        return bool(self.alive[int(cmd.agent_id) - self.lo])

    def mark_dead(self, ids):
        out = []
        for a in ids:
            if self.alive[a - self.lo]:
                self.alive[a - self.lo] = False
                out.append(a)
        return out

    def step(self, dt):
        f, self.faults = self.faults, []
        return np.array(f, dtype=np.uint64)


def _worker(rank, world, port, n_total, pos, alive, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = make_shard(n_total, rank, world)
        g = _FakeGroup(shard.lo, shard.hi, fault_ids=(3, n_total - 2))
        sw = ShardedSwarm(g, shard)
        cmd = type("C", (), {})
        results = [sw.apply_command(type("C", (), dict(agent_id=a, level="pos", values=(0,) * 7))())
                   for a in range(n_total)]
        local = sw.step(1e-3).tolist()             # no collective: this rank's ids only
        assert all(shard.lo <= f < shard.hi for f in local)
        assert sw.step(1e-3).size == 0
        coll = sw.collect()                        # one exchange for both ticks
        assert [t for t, _ in coll] == [0]
        faults = coll[0][1].tolist()
        assert sw.collect() == []
        # position all-gather exactly as NeighborSeparation lays it out
        local = torch.full((shard.pad, 4), float("nan"))
        mine = np.arange(shard.lo, shard.hi)
        keep = alive[mine]
        local[:shard.n_local][torch.from_numpy(keep), :3] = torch.from_numpy(pos[mine][keep]).float()
        gathered = torch.empty((shard.n_gathered, 4))
        dist.all_gather_into_tensor(gathered, local)
        gp = gathered.numpy().astype(float)
        galive = ~np.isnan(gp[:, 0])
        rows = shard.self_offset + np.arange(shard.n_local)
        ov = orc.neighbor_overlay(np.nan_to_num(gp[:, :3], nan=1e9), galive, 2.0, 1.0, rows=rows)
        result_q.put((rank, results, faults, ov, shard.lo, shard.hi))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_position_exchange():
    world, n_total = 2, 301
    rng = np.random.default_rng(5)
    pos = rng.uniform(0, 12, (n_total, 3))
    alive = rng.random(n_total) > 0.1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, pos, alive, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    # routing: each id answered by exactly its owner
    for a in range(n_total):
        answers = [res[1][a] for res in out]
        assert sum(x is not None for x in answers) == 1
    # fault ids of the whole swarm reach every rank
    assert out[0][2] == out[1][2] == [3, n_total - 2]
    # overlay from the sharded exchange == overlay of the whole swarm
    want = orc.neighbor_overlay(pos, alive, 2.0, 1.0)
    got = np.zeros((n_total, 3))
    for rank, _, _, ov, lo, hi in out:
        got[lo:hi] = ov
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6)
    assert np.abs(want).sum() > 0
