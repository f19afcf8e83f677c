"""Step-kernel time vs swarm size (tuning aid, not product code).

    python tools/nsweep.py [lib.so ...]

For each library (default: the in-tree build) and each N in SIZES: the bench
workload (paper_2308_12698_b200.synthetic), K = 10 and K = 1 launches timed
with CUDA events on the group's stream (20 launches after 5 warm-up), in a
fresh subprocess per library.  Prints one JSON line per (library, N).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SIZES = [int(x) for x in os.environ.get("NSWEEP_SIZES", "100000,300000,1000000,1250000,2500000,5000000,10000000").split(",")]
KS = [int(x) for x in os.environ.get("NSWEEP_KS", "10,1").split(",")]

CHILD = r'''
import json, sys, torch
sys.path.insert(0, "%(root)s")
from bench import _Batch
from paper_2308_12698_b200.synthetic import swarm
from paper_2308_12698_b200 import B200QuadGroup
for n in %(sizes)r:
    pos, sp = swarm(n)
    g = B200QuadGroup(0, _Batch(n, pos, 0), device="cuda:0")
    g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
    out = {"n": n}
    for k in %(ks)r:
        for _ in range(5): g.step_async(1e-3, k)
        g.collect_faults(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 20
        e0.record(g.stream)
        for _ in range(steps): g.step_async(1e-3, k)
        e1.record(g.stream); torch.cuda.synchronize(); g.collect_faults()
        ms = e0.elapsed_time(e1) / steps
        out[f"K{k}_us"] = ms * 1e3
        out[f"K{k}_rate"] = n * k / ms * 1e3
        if k == 10:
            out["K10_frac_nominal"] = n * k * 705 / (ms * 1e-3) / 74.45e12
        if k == 1:
            out["K1_frac182"] = 182 * n / (ms * 1e-3) / 6552.3e9
    print("RESULT " + json.dumps(out), flush=True)
    del g
    torch.cuda.empty_cache()
'''


def run(so):
    env = dict(os.environ)
    if so:
        env["SWARMSTEP_B200_LIB_OVERRIDE"] = str(so)
    p = subprocess.run([sys.executable, "-c", CHILD % dict(root=ROOT, sizes=SIZES, ks=KS)], env=env,
                       capture_output=True, text=True)
    lines = [json.loads(ln[7:]) for ln in p.stdout.splitlines() if ln.startswith("RESULT ")]
    if not lines:
        print(json.dumps({"lib": str(so), "error": p.stderr[-1500:]}), flush=True)
    for d in lines:
        print(json.dumps({"lib": str(so or "in-tree"), **d}), flush=True)


def main():
    libs = sys.argv[1:] or [None]
    for so in libs:
        run(so)


if __name__ == "__main__":
    main()
