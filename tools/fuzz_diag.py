"""Diagnose a per-step parity outlier of tests/test_gpu_fuzz.py (tuning aid):
python tools/fuzz_diag.py SEED -- replays the test's swarm and prints, for the
worst tick, the rows with the largest per-quantity errors and their state."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from gpu_util import FLOORS, f32, gpu_state, make_group, oracle_twin  # noqa: E402
from test_gpu_fuzz import _commands, _random_swarm  # noqa: E402
from paper_2308_12698_b200._lib import COL_OVERLAY  # noqa: E402

seed = int(sys.argv[1])
rng, sc = _random_swarm(seed)
g = make_group(sc)
_commands(rng, g, sc)
for t in range(12):
    if rng.uniform() < 0.3:
        g.add_velocity_overlay(rng.uniform(-1, 1, (sc.n, 3)))
    pre = gpu_state(g)
    og = oracle_twin(g)
    if g._overlay_active:
        og.add_velocity_overlay(g.column_block(COL_OVERLAY, COL_OVERLAY + 3).double().cpu().numpy().astype(np.float32).astype(float))
    og.step(f32(sc.dt))
    g.step(sc.dt)
    st = gpu_state(g)
    alive = og.alive.astype(bool)
    for q, want in (("pos", og.pos), ("vel", og.vel), ("quat", og.quat), ("omega", og.omega), ("integral", og.integral)):
        w, h = want[alive], st[q][alive]
        scale = np.maximum(np.max(np.abs(w), axis=1, keepdims=True), FLOORS[q])
        e = np.max(np.abs(h - w) / scale, axis=1)
        if e.size and e.max() > 5e-6:
            i = np.flatnonzero(alive)[int(np.argmax(e))]
            print(f"tick {t} {q}: rel {e.max():.2e} row {i} level {pre['cmd_level'][i]} cmd {pre['cmd_values'][i]}")
            print(f"   pre omega {pre['omega'][i]} integ {pre['integral'][i]} prev {pre['prev_omega'][i]} has_prev {pre['has_prev'][i]}")
            print(f"   pre pos {pre['pos'][i]} vel {pre['vel'][i]} quat {pre['quat'][i]}")
            print(f"   gpu {st[q][i]}  oracle {want[i]}  omega_sp gpu {st['omega_sp'][i]} oracle {og.omega_sp[i]}  f_c_sp gpu {st['f_c_sp'][i]} oracle {og.f_c_sp[i]}")
            np.savez(ROOT / "gpurun_out" / f"fuzz_diag_{seed}_{t}_{q}.npz", **{k: np.asarray(v)[i] for k, v in pre.items()},
                     dt=sc.dt, omega_sp_gpu=st['omega_sp'][i], f_c_sp_gpu=st['f_c_sp'][i],
                     omega_sp_or=og.omega_sp[i], f_c_sp_or=og.f_c_sp[i])
