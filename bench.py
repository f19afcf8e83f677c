#!/usr/bin/env python
"""Headline benchmark: quadrotor agent-steps/s of the fused dynamics+control step.

Workload (BASELINE.json metric "quadrotor agent-steps/sec (dynamics+control) at
N=1M/10M", configs 3/4): per GPU ``--agents`` quadrotors (default 10M) on the
reference bench's grid layout (bench.py:87-93 of the reference: spacing 3 m,
origin (0,0,10)), identity attitude, at rest, POSITION level with random
setpoints p_sp = p0 + U(-1,1)^3, v_sp = 0, yaw U(-pi,pi),
dt = 1 ms, K = 10 fused ticks per launch.  One bench "step" = one launch =
K ticks for every agent, so value = N_total * K * steps / time.

Agents shard by index across ranks (one process per GPU, torchrun); there is
no collective on this path, so per-GPU work is fixed ("scaling": "weak").

``--impl reference`` times the reference's CPU path instead: the float64 C
restatement in oracle/ (the reference itself is Python that does not travel
to the GPU box) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "quadrotor agent-steps/sec (dynamics+control) at N=1M/10M, 1/2/4/8 B200"
UNIT = "agent-steps/s"
# algorithmic bytes per agent per launch, position level, compensated position
# (DESIGN.md "Roofline"): read 13 state + 3 pos-lo + 6 PID + 7 command floats +
# 1 flag byte = 117 B; write 13 + 3 + 6 + 4 stale-setpoint floats = 104 B.
ALG_BYTES_PER_AGENT_LAUNCH = 221
# algorithmic flops per agent-tick at position level (FMA = 2)
ALG_FLOPS_PER_AGENT_TICK = 705
PORT_NOTE = ("the port runs ~5x faster than the reference's own numpy QuadGroup.step on one core "
             "(4.7-5.5x, same results to 2e-15 m; profiles/cpu_ref_vs_port_r01.json): a conservative baseline")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--agents", type=int, default=10_000_000, help="agents per GPU")
    ap.add_argument("--substeps", type=int, default=10, help="fused ticks per launch (K)")
    ap.add_argument("--dt", type=float, default=1e-3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="cpu_baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k1", action="store_true", help="skip the K=1 HBM-roofline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--motor-tau", type=float, default=0.0,
                    help="opt-in first-order rotor lag time constant (s); 0 = the reference's instantaneous mixer")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
def workload(n: int, seed: int, id_base: int = 0):
    """Initial state + POS setpoints (float64 host arrays) for n agents."""
    from paper_2308_12698_b200.layout import layout_poses
    pos, _ = layout_poses({"kind": "grid", "spacing": 3.0, "origin": (0.0, 0.0, 10.0)}, n)
    rng = np.random.default_rng(seed)
    sp = np.empty((7, n), dtype=np.float32)
    sp[0:3] = (pos + rng.uniform(-1.0, 1.0, (n, 3))).T
    sp[3:6] = 0.0
    sp[6] = rng.uniform(-np.pi, np.pi, n)
    return pos, sp


class _Batch:
    def __init__(self, n, pos, id_base):
        self.type_id = 0
        self.agent_ids = np.arange(id_base, id_base + n, dtype=np.uint64)
        self.pos = pos
        self.vel = np.zeros((n, 3))
        self.quat = np.zeros((n, 4))
        self.quat[:, 0] = 1.0
        self.omega = np.zeros((n, 3))
        self.alive = np.ones(n, dtype=bool)


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        return self

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- CPU legs
def cpu_leg(n_sample: int, k: int, dt: float, budget_s: float, min_reps: int = 1, motor_tau: float = 0.0):
    """Time the float64 oracle (reference algorithm) on all host cores."""
    from oracle import oracle as orc
    threads = orc.cpu_count()
    pos, sp = workload(n_sample, seed=0)
    g = orc.OracleGroup(0, _Batch(n_sample, pos, 0), motor_tau=motor_tau)
    g.cmd_values[:] = sp.T.astype(np.float64)
    g.step(dt, nthreads=threads)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        for _ in range(k):
            g.step(dt, nthreads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if reps >= min_reps and el >= budget_s:
            break
    return n_sample * k * reps / el, threads, reps, el


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    n_sample = 262_144
    threads = None
    vals = []
    for i in range(args.warmup + args.steps):
        v, threads, reps, el = cpu_leg(n_sample, args.substeps, args.dt, 0.0, min_reps=1, motor_tau=args.motor_tau)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals))
    sample = (f"{n_sample} agents x {args.substeps} ticks per step (POS level, random setpoints, "
              f"float64 C oracle, {threads} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": n_sample * args.substeps / value * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg3/cfg4 recipe, sampled: {sample}", "agents_sampled": n_sample,
                   "substeps": args.substeps, "dt": args.dt, "level": "pos"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "note": PORT_NOTE},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def run_b200(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2308_12698_b200 import B200QuadGroup

    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, k, dt = args.agents, args.substeps, args.dt
    nccl = _backend() == "nccl"

    def barrier():
        if world > 1:
            if nccl:
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    t_setup = time.perf_counter()
    pos, sp = workload(n, seed=rank, id_base=rank * n)
    g = B200QuadGroup(0, _Batch(n, pos, rank * n), device=dev, motor_tau=args.motor_tau)
    sp_dev = torch.from_numpy(sp).to(dev)
    g.set_setpoints(sp_dev, columns=True)
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t_setup

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if nccl else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, stream):
        barrier()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1))

    # ---- device-resident leg (value): K fused ticks per launch
    for _ in range(args.warmup):
        g.step_async(dt, k)
    faults = g.collect_faults()
    # clocks are sampled (200 ms period) from a soak of the same launches
    # right before the timed region through its end, so that even a short
    # timed region is covered by samples taken under this load
    clocks = ClockSampler(local).start()
    t_soak = time.perf_counter()
    while time.perf_counter() - t_soak < 1.0:
        for _ in range(8):
            g.step_async(dt, k)
        g.collect_faults()
    ms = timed(lambda: g.step_async(dt, k), args.steps, g.stream)
    clk = clocks.stop()
    faults = sum(f.size for f in g.collect_faults())
    ms_per_step = ms / args.steps
    value = world * n * k * args.steps / (ms * 1e-3)
    launch_s = ms_per_step * 1e-3
    achieved_tf = n * k * ALG_FLOPS_PER_AGENT_TICK / launch_s / 1e12
    sm_mhz = clk.get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_nominal_tf = sms * 128 * 2 * sm_mhz * 1e6 / 1e12
    fp32_meas = _fp32_peak()
    if fp32_meas:
        fp32_peak_tf = fp32_meas["tflops"]
        peak_source = (f"measured: FP32 microbenchmark tools/fp32_peak.cu (best of FFMA register / immediate / "
                       f"packed FFMA2: {fp32_meas['form']}) on this GPU; nominal {fp32_nominal_tf:.1f} TFLOP/s = "
                       f"{sms} SMs x 128 lanes x 2 x {sm_mhz:.0f} MHz")
    else:
        fp32_peak_tf = fp32_nominal_tf
        peak_source = (f"derived: {sms} SMs x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz "
                       "(MEASURED_PEAKS.json has no FP32 SIMT figure)")

    # ---- K=1 leg: the same kernel in its HBM-bound regime
    k1 = None
    if not args.no_k1:
        for _ in range(3):
            g.step_async(dt, 1)
        g.collect_faults()
        ms1 = timed(lambda: g.step_async(dt, 1), args.steps, g.stream)
        g.collect_faults()
        t1 = ms1 / args.steps * 1e-3
        peaks = _peaks()
        k1 = {"bound": "hbm", "achieved": ALG_BYTES_PER_AGENT_LAUNCH * n / t1 / 1e9,
              "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": ALG_BYTES_PER_AGENT_LAUNCH * n / t1 / 1e9 / peaks["hbm_gbs"],
              "traffic": _traffic("k1", n), "ms_per_launch": t1 * 1e3,
              "agent_steps_per_s": world * n / t1, "peak_source": peaks["source"]}

    # ---- end-to-end leg through the public API with host buffers:
    # every step uploads a fresh whole-swarm POS setpoint block from pinned host
    # memory (28 B/agent), runs K ticks, and reads the fault result back.
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(sp).pin_memory(), torch.from_numpy(sp[:, ::-1].copy()).pin_memory()]

        # software pipeline: step i's launch is queued before step i+1's
        # setpoints are uploaded (copy engine, side stream), so the PCIe copy
        # overlaps the compute of step i; step i's faults are then read back.
        def e2e_run(steps):
            g.set_setpoints(host[0], columns=True)
            for i in range(steps):
                g.step_async(dt, k)
                if i + 1 < steps:
                    g.set_setpoints(host[(i + 1) & 1], columns=True)
                g.collect_faults()

        e2e_run(args.warmup)
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e2e_run(args.steps)
        torch.cuda.synchronize(dev)
        el = max_over_ranks(time.perf_counter() - t0)
        barrier()
        e2e = {"value": world * n * k * args.steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(7 * 4 * n), "d2h_bytes_per_step": 16,
               "ms_per_step": el / args.steps * 1e3,
               "path": "B200QuadGroup.set_setpoints(pinned host) + step_async(dt, K) + collect_faults()"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_s = 262_144
        v, threads, reps, el = cpu_leg(n_s, k, dt, args.cpu_seconds, motor_tau=args.motor_tau)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "note": PORT_NOTE,
               "sample": f"{n_s} agents x {k} ticks x {reps} reps ({el:.1f} s), same recipe, float64 C oracle "
                         f"(restatement of the reference QuadGroup.step), {threads} threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{n:,} quadrotors per GPU, POS level, random setpoints, "
                                   f"K={k} fused ticks per launch (cfg3 recipe at cfg4 size)",
                       "agents_per_gpu": n, "agents_total": n * world, "substeps": k, "dt": dt,
                       "level": "pos", "compensated_position": True, "motor_tau": args.motor_tau,
                       "l2": f"inputs larger than L2 ({n * 221 / 1e9:.2f} GB touched per launch vs 0.126 GB L2)",
                       "parallelism": f"agent-index shards x{world}, no collective"},
            "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": fp32_peak_tf, "unit": "TFLOP/s",
                         "frac": achieved_tf / fp32_peak_tf, "traffic": _traffic("k10", n),
                         "flops_per_agent_tick": ALG_FLOPS_PER_AGENT_TICK, "peak_source": peak_source,
                         "fp32_peak_measurements": fp32_meas},
            "roofline_k1": k1,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": args.steps,
            "faults": faults,
            "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)


def _fp32_peak():
    """FP32 SIMT peak measured on this GPU (tools/fp32_peak.cu), or None."""
    import ctypes
    so = ROOT / "tools" / "libfp32peak.so"
    if not so.exists():
        return None
    lib = ctypes.CDLL(str(so))
    lib.fp32_peak_tflops.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    res = {}
    for imm, key in ((0, "reg"), (1, "imm"), (2, "ffma2"), (3, "ffma2_3reg")):
        tf, ms = ctypes.c_double(), ctypes.c_double()
        if lib.fp32_peak_tflops(imm, ctypes.byref(tf), ctypes.byref(ms)) == 0:
            res[key] = tf.value
    peaks = {k: v for k, v in res.items() if k != "ffma2_3reg"}
    if not peaks:
        return None
    form = max(peaks, key=peaks.get)
    names = {"reg": "register-operand FFMA", "imm": "immediate-operand FFMA", "ffma2": "packed FFMA2"}
    # ffma2_3reg (three vector-register operands: register-file read bound) is
    # context for the roofline, not a peak: the best form is the denominator
    return {"tflops": peaks[form], "form": names[form], **res}


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "MEASURED_PEAKS.json (measured copy)"}
    return {"hbm_gbs": 6650.0, "source": "fallback 6.65 TB/s (B200_PROFILING.md)"}


def _traffic(key: str, n: int):
    """dram bytes per launch from the committed ncu capture, scaled per agent."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(key)
    if not d:
        return None
    return d["dram_bytes_per_agent"] * n


def _backend() -> str:
    # nccl (one rank per GPU, the driver's launch).  SWARMSTEP_BENCH_BACKEND=gloo
    # is a plumbing check only: N ranks may then share one GPU (LOCAL_RANK mod
    # device count) to exercise the multi-rank code path on a 1-GPU box; its
    # numbers are not measurements.
    return os.environ.get("SWARMSTEP_BENCH_BACKEND", "nccl")


def _local_device() -> int:
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return local % max(1, torch.cuda.device_count()) if _backend() == "gloo" else local


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(_local_device())
        dist.init_process_group(_backend())
    try:
        run_b200(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
