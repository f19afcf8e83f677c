"""Parity evidence on a B200: per-step relative error and horizon divergence of
the CUDA float32 path against the float64 oracle / the reference's golden
trajectories.  Writes one JSON report (default gpurun_out/parity.json).

  * golden scenarios (reference float64 runs): max |abs divergence| per quantity
    at every recorded tick;
  * cfg1 full horizon: 1,000 quads, RATE hover with perturbed rates, dt 1 ms,
    10 s = 10,000 ticks, CUDA vs oracle, with and without compensated position;
  * cfg3-shaped closed loop: 1,000 quads POS random setpoints, 10 s horizon;
  * per-step relative error along those trajectories (identical pre-step state).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

from golden_io import load_scenario  # noqa: E402
from gpu_util import f32, gpu_state, make_group, oracle_twin, rel_errors  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from scenarios import ALL, Scenario, run_script  # noqa: E402

Q = ("pos", "vel", "quat", "omega", "integral")


def golden_divergence():
    out = {}
    for name in ("hover_rate", "pos_random", "mixed", "fault_nan"):
        sc, rec, cmd_ok, faults, _ = load_scenario(name)
        g = make_group(sc)
        got, ok, gf = run_script(g, sc, state_of=gpu_state)
        per_tick = {}
        for t in sorted(rec):
            a = rec[t]["alive"]
            per_tick[t] = {q: float(np.max(np.abs(got[t][q][a] - rec[t][q][a]))) for q in Q if a.any()}
        out[name] = {"per_tick_abs": per_tick, "cmd_ok_equal": bool(np.array_equal(ok, cmd_ok)),
                     "faults_equal": {t: f for t, f in gf.items() if f} == faults}
    return out


def horizon(sc: Scenario, compensated: bool, every: int = 500, per_step_every: int = 1000):
    g = make_group(sc, compensated=compensated)
    og = orc.OracleGroup(0, type("B", (), dict(agent_ids=np.arange(sc.n, dtype=np.uint64),
                                               pos=gpu_state(g)["pos"], vel=gpu_state(g)["vel"],
                                               quat=gpu_state(g)["quat"], omega=gpu_state(g)["omega"],
                                               alive=np.ones(sc.n, bool)))())
    for c in sc.cmds:
        cmd = type("C", (), dict(agent_id=c[1], level=["pos", "rate", "motor"][c[2]],
                                 values=tuple(np.float32(c[3]).astype(float))))
        g.apply_command(cmd)
        og.apply_command(cmd)
    curve, per_step = [], {q: 0.0 for q in Q}
    t0 = time.perf_counter()
    for t in range(sc.ticks):
        if per_step_every and t % per_step_every == 0 and t > 0:
            tw = oracle_twin(g)
            tw.step(f32(sc.dt))
        g.step(sc.dt)
        og.step(f32(sc.dt), nthreads=orc.cpu_count())
        if per_step_every and t % per_step_every == 0 and t > 0:
            e = rel_errors(gpu_state(g), tw)
            per_step = {q: max(per_step[q], e[q]) for q in Q}
        if (t + 1) % every == 0:
            st = gpu_state(g)
            curve.append({"tick": t + 1, **{q: float(np.max(np.abs(st[q] - getattr(og, q)))) for q in Q}})
    return {"n": sc.n, "ticks": sc.ticks, "dt": sc.dt, "compensated": compensated, "abs_divergence": curve,
            "per_step_rel_max": per_step, "wall_s": time.perf_counter() - t0}


def main():
    out_path = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "parity.json")
    rep = {"golden": golden_divergence()}
    cfg1 = ALL["hover_rate"](n=1000, ticks=10_000)
    rep["cfg1_horizon_compensated"] = horizon(cfg1, True)
    rep["cfg1_horizon_plain"] = horizon(cfg1, False)
    cfg3 = ALL["pos_random"](n=1000, ticks=10_000)
    rep["cfg3_horizon_compensated"] = horizon(cfg3, True)
    out_path.parent.mkdir(parents=True, exist_ok=True)
    out_path.write_text(json.dumps(rep, indent=1))
    for k in ("cfg1_horizon_compensated", "cfg1_horizon_plain", "cfg3_horizon_compensated"):
        print(k, rep[k]["abs_divergence"][-1], rep[k]["per_step_rel_max"])
    for k, v in rep["golden"].items():
        last = max(v["per_tick_abs"], key=int)
        print(k, last, v["per_tick_abs"][last])


if __name__ == "__main__":
    main()
