"""GPU collision / neighbour detection at scale.

  python tools/collision_bench.py [agents] [reps]

Agents uniformly at ~1 per 8 m^3 (the cfg5 density), r_collide 0.15 m,
r_sense 2 m, cell 2 m.  Prints one JSON line: wall time of GpuDetector.detect returning the
collisions (neighbour sets left on the device until read -- the in-loop
collision-death use, core.py:495-498), and with the reference's per-agent
neighbor_sets dict materialised, and the out-of-loop form (detect_snapshot on a host
WorldSnapshot, upload included).
With --reference (build container only) it times the reference's own
collision.detect (numpy) on the same positions instead.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def positions(n, seed=3):
    side = (8.0 * n) ** (1 / 3)
    return np.random.default_rng(seed).uniform(0, side, (n, 3)) + [0, 0, 10]


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n = int(args[0]) if args else 100_000
    reps = int(args[1]) if len(args) > 1 else 5
    pos = positions(n)
    if "--reference" in sys.argv:
        sys.path.insert(0, "/root/reference/pkg/src")
        from swarmstep.collision import CollisionConfig, detect
        from swarmstep.state import WorldSnapshot, batch_create, batch_snapshot
        snap = WorldSnapshot(tick=0, batches=(batch_snapshot(batch_create(0, n, pos), 0),))
        cfg = CollisionConfig(r_collide={0: 0.15}, r_sense=2.0, cell=2.0)
        detect(snap, cfg)
        t0 = time.perf_counter()
        for _ in range(reps):
            rep = detect(snap, cfg)
        el = (time.perf_counter() - t0) / reps
        print(json.dumps({"impl": "reference numpy collision.detect (1 core, build container)", "agents": n,
                          "wall_ms": el * 1e3, "collisions": len(rep.collisions)}))
        return
    import torch
    from paper_2308_12698_b200 import B200QuadGroup, batch_create
    from paper_2308_12698_b200.collision import CollisionConfig, GpuDetector
    g = B200QuadGroup(0, batch_create(0, n, pos))
    cfg = CollisionConfig(r_collide={0: 0.15}, r_sense=2.0, cell=2.0)
    det = GpuDetector(cfg, g.device)
    rep = det.detect([g], 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        rep = det.detect([g], 0)          # collisions; neighbour sets stay on the device (lazy)
    detect_ms = (time.perf_counter() - t0) / reps * 1e3
    t0 = time.perf_counter()
    for _ in range(reps):
        rep = det.detect([g], 0)
        n_neigh = sum(len(v) for v in rep.neighbor_sets.values())   # materialise the reference's dict
    full_ms = (time.perf_counter() - t0) / reps * 1e3
    # out-of-loop form: detect(snapshot, config) on a host WorldSnapshot (float64 upload included)
    from paper_2308_12698_b200.state import WorldSnapshot, batch_snapshot
    snap = WorldSnapshot(tick=0, batches=(batch_snapshot(g.batch, 0),))
    rep_s = det.detect_snapshot(snap)
    t0 = time.perf_counter()
    for _ in range(reps):
        rep_s = det.detect_snapshot(snap)
    snap_ms = (time.perf_counter() - t0) / reps * 1e3
    assert rep_s.collisions == rep.collisions
    print(json.dumps({"impl": "b200", "agents": n, "detect_ms": detect_ms, "detect_with_neighbor_sets_ms": full_ms,
                      "detect_snapshot_ms": snap_ms, "collisions": len(rep.collisions), "neighbor_entries": n_neigh}))


if __name__ == "__main__":
    main()
