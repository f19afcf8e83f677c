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


def load_viewer():
    """tests/golden/viewer.npz: (pos, alive, quat, [case dicts]) for the
    viewer influence messages (World._apply_viewer_input, core.py:445-453)."""
    z = dict(np.load(GOLDEN / "viewer.npz"))
    cases = []
    for i in range(int(z["cases"])):
        mode, radius, strength = (str(x) for x in z[f"v{i}_msg"])
        c = dict(mode=mode, radius=float(radius), strength=float(strength), point=z[f"v{i}_point"],
                 off=z[f"v{i}_off"], any=bool(z[f"v{i}_any"]))
        if f"v{i}_cmd_level" in z:
            c["cmd_level"], c["cmd_values"] = z[f"v{i}_cmd_level"], z[f"v{i}_cmd_values"]
        cases.append(c)
    return z["pos"], z["alive"], z["quat"], cases


def load(name):
    """A plain golden fixture tests/golden/<name>.npz as a dict."""
    return dict(np.load(GOLDEN / f"{name}.npz"))
