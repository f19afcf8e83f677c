"""Helpers to load the committed golden fixtures (tests/golden/*.npz)."""

from pathlib import Path

import numpy as np

from scenarios import Scenario

GOLDEN = Path(__file__).resolve().parent / "golden"
STATE_KEYS = ("pos", "vel", "quat", "omega", "alive", "integral", "prev_omega", "has_prev",
              "omega_sp", "f_c_sp", "cmd_level", "cmd_values")


def load_functions():
    return dict(np.load(GOLDEN / "functions.npz"))


def load_scenario(name):
    z = dict(np.load(GOLDEN / f"scenario_{name}.npz"))
    sc = Scenario.from_arrays(z)
    rec = {}
    for i, t in enumerate(z["rec_ticks"]):
        rec[int(t)] = {k: z[f"rec_{k}"][i] for k in STATE_KEYS if f"rec_{k}" in z}
    faults = {}
    for t, a in zip(z["fault_tick"], z["fault_id"]):
        faults.setdefault(int(t), []).append(int(a))
    return sc, rec, z["cmd_ok"], faults, int(z["raise_tick"])
