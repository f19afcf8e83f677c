"""Kernel-variant sweep on a B200 (tuning aid, not part of the product).

Builds variants of libswarmstep_b200.so with different -D macros into /tmp,
then times the fused step (K=10 and K=1) for each in a fresh subprocess.
Usage: python tools/tune.py [agents]
"""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

VARIANTS = {
    "default": [],
    "p6": ["-DSSB_PAIR_MINB=6"],
    "p7": ["-DSSB_PAIR_MINB=7"],
    "p9": ["-DSSB_PAIR_MINB=9"],
}

CHILD = r'''
import json, sys, torch, numpy as np
sys.path.insert(0, "%(root)s")
from bench import _Batch
from paper_2308_12698_b200.synthetic import swarm as workload
from paper_2308_12698_b200 import B200QuadGroup
n = %(n)d
pos, sp = workload(n)
g = B200QuadGroup(0, _Batch(n, pos, 0), device="cuda:0")
g.set_setpoints(torch.from_numpy(sp).cuda(), columns=True)
out = {}
import os
g.kernel = os.environ.get("TUNE_KERNEL", "auto")
for k in (10, 4, 2, 1):
    for _ in range(5): g.step_async(1e-3, k)
    g.collect_faults(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 20
    e0.record(g.stream)
    for _ in range(steps): g.step_async(1e-3, k)
    e1.record(g.stream); torch.cuda.synchronize(); g.collect_faults()
    ms = e0.elapsed_time(e1) / steps
    out[f"K{k}_ms"] = ms
    out[f"K{k}_agent_steps_per_s"] = n * k / ms * 1e3
out["K1_GBps_182B"] = 182 * n / out["K1_ms"] / 1e6
out["kernel"] = g.kernel
print("RESULT " + json.dumps(out))
'''


def run_prebuilt(so, kern, n):
    env = dict(os.environ, SWARMSTEP_B200_LIB_OVERRIDE=str(so), TUNE_KERNEL=kern)
    p = subprocess.run([sys.executable, "-c", CHILD % dict(root=ROOT, n=n)], env=env, capture_output=True, text=True)
    line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    return json.loads(line[0][7:]) if line else {"error": p.stderr[-800:]}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
    if len(sys.argv) > 2:   # compare prebuilt libraries: tune.py N a.so b.so ...
        for so in sys.argv[2:]:
            for kern in ("direct", "pair"):
                print(so, kern, json.dumps(run_prebuilt(so, kern, n)), flush=True)
        return
    from paper_2308_12698_b200._build import NVCC_FLAGS, _nvcc, sources, INCLUDE, CSRC
    res = {}
    runs = [(name, defs, kern) for name, defs in VARIANTS.items() for kern in ("direct", "pair")]
    for name, defs, kern in runs:
        so = f"/tmp/ssb_{name}.so"
        cmd = [_nvcc(), *NVCC_FLAGS, *defs, f"-I{INCLUDE}", f"-I{CSRC}", "-o", so, *map(str, sources())]
        b = subprocess.run(cmd, capture_output=True, text=True)
        regs = [l for l in b.stderr.splitlines() if "registers" in l]
        env = dict(os.environ, SWARMSTEP_B200_LIB_OVERRIDE=so, TUNE_KERNEL=kern)
        p = subprocess.run([sys.executable, "-c", CHILD % dict(root=ROOT, n=n)], env=env, capture_output=True, text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
        key = f"{name}/{kern}"
        res[key] = json.loads(line[0][7:]) if line else {"error": p.stderr[-800:]}
        print(key, json.dumps(res[key]), flush=True)
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "tune.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
