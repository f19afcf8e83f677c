"""The B200 groups inside the reference's OWN, unmodified loop code.

``oracle/_ref`` holds the reference package itself (pip-installed by
``__graft_entry__.build()`` from /root/reference/pkg; it travels to the GPU
box with the snapshot).  These tests import ``swarmstep`` from there and run:

* ``swarmstep.core.World([B200QuadGroup, B200UnicycleGroup], dt, ...)`` with
  in-loop collision detection over the recorded script, checked against the
  reference World's own recording (tests/golden/world.npz): identical event
  log, state within float32 trajectory tolerance;
* the reference bench's world construction (``swarmstep.bench._bench_world``
  -> ``build_world``, core.py:508-541) and ``run_bench`` (bench.py:117-149)
  with ``swarmstep.core.QuadGroup`` bound to ``B200QuadGroup`` -- the one-line
  drop-in INTEGRATION.md describes -- against the same world built with the
  reference's own QuadGroup.
"""

import json
import sys

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs CUDA")]

# same bounds as the World replay (tests/test_gpu_world_golden.py)
TOL = dict(pos=2e-6, vel=2e-5, quat=5e-6, omega=1e-4)


@pytest.fixture(scope="module")
def swarmstep():
    from oracle import ref_runner
    if not ref_runner.available():
        pytest.skip("oracle/_ref (the reference package) is not installed: run __graft_entry__.build()")
    path = ref_runner.import_path()
    if path not in sys.path:
        sys.path.insert(0, path)
    import swarmstep as ss
    import swarmstep.bench  # noqa: F401
    import swarmstep.collision  # noqa: F401
    import swarmstep.core  # noqa: F401
    import swarmstep.state  # noqa: F401
    import swarmstep.wire  # noqa: F401
    assert str(ss.__file__).startswith(path)
    return ss


def test_unmodified_world_with_b200_groups_matches_reference_recording(swarmstep):
    from golden_io import GOLDEN

    from paper_2308_12698_b200 import B200QuadGroup, B200UnicycleGroup
    core, wire, state = swarmstep.core, swarmstep.wire, swarmstep.state
    z = dict(np.load(GOLDEN / "world.npz"))
    script = json.loads(str(z["script"]))
    want_events = json.loads(str(z["events"]))
    qpos, upos = z["qpos"], z["upos"]
    n_q, n_u, dt, ticks = qpos.shape[0], upos.shape[0], float(z["dt"]), int(z["ticks"])
    quads = B200QuadGroup(0, state.batch_create(0, n_q, qpos))
    unis = B200UnicycleGroup(1, state.batch_create(1, n_u, upos, id_base=n_q))
    cfg = swarmstep.collision.CollisionConfig(r_collide={0: 0.2, 1: 0.3}, r_sense=1.2, cell=1.2)
    world = core.World([quads, unis], dt=dt, collision_config=cfg, collision_in_loop=True)
    worst = dict.fromkeys(TOL, 0.0)
    try:
        for t in range(ticks):
            for item in script.get(str(t), []):
                if item[0] == "cmd":
                    world.submit_commands([wire.AgentCommand(item[1], wire.CommandLevel(item[2]), tuple(item[3]))])
                else:
                    world.submit_viewer_input(wire.ViewerInputMsg(mode=wire.InfluenceMode(item[1]),
                                                                  world_point=tuple(item[2]), radius=item[3],
                                                                  strength=item[4]))
            world.tick()
            if (t + 1) % 20 == 0:
                for g in world.groups:
                    b = g.batch
                    np.testing.assert_array_equal(b.alive, z[f"t{t}_g{g.type_id}_alive"], err_msg=f"tick {t}")
                    for k, tol in TOL.items():
                        err = float(np.max(np.abs(getattr(b, k) - z[f"t{t}_g{g.type_id}_{k}"])))
                        worst[k] = max(worst[k], err)
                        assert err <= tol, f"tick {t} type {g.type_id} {k}: {err:.2e} > {tol:.0e}"
    finally:
        world.close()
    print("unmodified World max |err|:", worst)
    events = [[e.tick, e.kind.value, [int(a) for a in e.agent_ids]] for e in world.event_log]
    assert events == want_events
    assert any(e[1] == "collision_death" for e in want_events)
    assert world.clock.tick == ticks


def test_reference_bench_world_with_b200_quadgroup(swarmstep, monkeypatch):
    """The reference bench's own world construction and loop, with the B200
    group bound in place of QuadGroup, tracks the same world built with the
    reference QuadGroup (RATE hover through World.submit_commands)."""
    from paper_2308_12698_b200 import B200QuadGroup
    core, bench = swarmstep.core, swarmstep.bench
    n, dt, ticks = 1000, 1e-3, 200
    ref_world = bench._bench_world(n, dt, False)
    monkeypatch.setattr(core, "QuadGroup", B200QuadGroup)
    b200_world = bench._bench_world(n, dt, False)
    assert isinstance(b200_world.groups[0], B200QuadGroup)
    assert not isinstance(ref_world.groups[0], B200QuadGroup)
    # kick the hover with a small rate command on a few agents, through the World
    cmds = [swarmstep.wire.AgentCommand(a, swarmstep.wire.CommandLevel.RATE, (0.2, -0.1, 0.05, 9.9))
            for a in range(0, n, 7)]
    for w in (ref_world, b200_world):
        w.submit_commands(cmds)
        for _ in range(ticks):
            w.tick()
    rb, gb = ref_world.groups[0].batch, b200_world.groups[0].batch
    for k, tol in TOL.items():
        err = float(np.max(np.abs(getattr(gb, k) - getattr(rb, k))))
        assert err <= tol, (k, err)
    assert ref_world.state_table_bytes() != b""       # the World's own readers work on the B200 group
    assert len(b200_world.state_table_bytes()) == len(ref_world.state_table_bytes())
    assert b200_world.alive_counts() == ref_world.alive_counts() == {0: n}
    ref_world.close()
    b200_world.close()

    # run_bench itself (warm-up, timed rounds, repeats), unmodified
    res = bench.run_bench(bench.BenchSpec(agent_counts=(256, 4096), warmup_rounds=5, timed_rounds=20, repeats=1))
    assert [r.n_agents for r in res.rows] == [256, 4096] and not res.skipped
    assert all(r.mean_ms > 0 for r in res.rows)
