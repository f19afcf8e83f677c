#!/usr/bin/env python
"""Headline benchmark: quadrotor agent-steps/s of the fused dynamics+control step.

Workload (BASELINE.json metric "quadrotor agent-steps/sec (dynamics+control) at
N=1M/10M, 1/2/4/8 B200", configs 3/4): ``--agents`` quadrotors in total
(default 10,000,000) on the reference bench's grid layout (bench.py:87-93 of
the reference: spacing 3 m, origin (0,0,10)), identity attitude, at rest,
POSITION level with random setpoints p_sp = p0 + U(-1,1)^3, v_sp = 0,
yaw U(-pi,pi) (paper_2308_12698_b200/synthetic.py),
dt = 1 ms, K = 10 fused ticks per launch.  One bench "step" = one launch =
K ticks for every agent, so value = N_total * K * steps / time.

Multi-GPU (cfg4): the N_total agents are split by contiguous index across
the ranks (one process per GPU, torchrun), each rank stepping its own rows
with no data-path collective, so total work is fixed ("scaling": "strong");
``--agents-per-gpu`` selects weak scaling instead.

``--impl reference`` times the reference's own CPU path instead: the
unmodified ``swarmstep.core.QuadGroup.step`` (core.py:166-202, installed in
oracle/_ref by build()) on the same N_total-agent swarm, sharded over every
host core (oracle/ref_runner.py), rank 0 only.
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
# Algorithmic bytes per agent per launch at position level:
# read 13 state + 6 PID + 7 setpoint floats + 1 flag byte = 105 B, write
# 13 state + 6 PID floats + 1 flag byte = 77 B.
ALG_BYTES_PER_AGENT_LAUNCH = 182
# ... plus what this implementation also moves: the compensated
# position's packed low-part word (4 B read + 4 B written) and the stale
# inner-loop setpoints written for a later MOTOR command (16 B) -- overhead,
# not algorithm
BYTES_WITH_OVERHEAD = 206
# algorithmic flops per agent-tick at position level (FMA = 2)
ALG_FLOPS_PER_AGENT_TICK = 705


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--agents", type=int, default=10_000_000,
                    help="agents in total, split across the GPUs (strong scaling)")
    ap.add_argument("--agents-per-gpu", type=int, default=None,
                    help="weak scaling: this many agents on every GPU instead of --agents in total")
    ap.add_argument("--substeps", type=int, default=10, help="fused ticks per launch (K)")
    ap.add_argument("--dt", type=float, default=1e-3)
    ap.add_argument("--cpu-samples", type=int, default=4,
                    help="cpu_baseline: timed reference ticks of the whole swarm (after one warm tick)")
    ap.add_argument("--cpu-seconds", type=float, default=4.0, help="cpu_baseline: C-port sample budget")
    ap.add_argument("--ref-ticks", type=int, default=1,
                    help="--impl reference: ticks of the whole swarm per timed step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k1", action="store_true", help="skip the K=1 HBM-roofline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--motor-tau", type=float, default=0.0,
                    help="opt-in first-order rotor lag time constant (s); 0 = the reference's instantaneous mixer")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
def layout(args, world: int) -> tuple[int, str]:
    """(total agents, scaling) of the run."""
    if args.agents_per_gpu is not None:
        return args.agents_per_gpu * world, "weak"
    return args.agents, "strong"


def rank_rows(args, rank: int, world: int) -> tuple[int, int]:
    from paper_2308_12698_b200.parallel import shard_range
    if args.agents_per_gpu is not None:
        return rank * args.agents_per_gpu, (rank + 1) * args.agents_per_gpu
    return shard_range(args.agents, rank, world)


def config(args, world: int) -> dict:
    n_total, scaling = layout(args, world)
    per = ("per GPU" if scaling == "weak" else f"in total, split by agent index over {world} GPU(s)")
    return {"workload": f"{n_total:,} quadrotors {per}, POS level, random setpoints, K={args.substeps} fused ticks "
                        f"per launch (cfg3 recipe; cfg4 = 10M over 2/4/8 GPUs)",
            "agents_total": n_total, "agents_per_gpu": -(-n_total // world), "substeps": args.substeps,
            "dt": args.dt, "level": "pos", "compensated_position": True, "motor_tau": args.motor_tau,
            "l2": f"inputs larger than L2 ({-(-n_total // world) * BYTES_WITH_OVERHEAD / 1e9:.2f} GB touched per "
                  f"launch per GPU vs 0.126 GB L2)" if -(-n_total // world) * BYTES_WITH_OVERHEAD > 126e6 else
                  "per-GPU state smaller than L2: launches may hit L2 (not an HBM measurement)",
            "parallelism": f"agent-index shards x{world}, no collective",
            "launch_overlap": ("back-to-back K >= 4 launches overlap tile by tile (programmatic dependent launch, "
                               "per-tile epochs; bit-identical to ordered launches)"
                               if os.environ.get("SWARMSTEP_B200_NO_OVERLAP", "") != "1" else "off")}


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
def port_leg(n_total: int, k: int, dt: float, budget_s: float, motor_tau: float = 0.0) -> dict:
    """The float64 C restatement of QuadGroup.step (oracle/quad_oracle.c) on all
    host threads, on the first rows of the same swarm, for ~budget_s seconds."""
    from oracle import oracle as orc

    from paper_2308_12698_b200.synthetic import swarm
    threads = orc.cpu_count()
    n_s = min(262_144, n_total)
    pos, sp = swarm(n_total, 0, n_s)
    g = orc.OracleGroup(0, _Batch(n_s, pos, 0), motor_tau=motor_tau)
    g.cmd_values[:] = sp.T.astype(np.float64)
    g.step(dt, nthreads=threads)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        for _ in range(k):
            g.step(dt, nthreads=threads)
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return {"value": n_s * k * reps / el, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"rows [0, {n_s}) of the same swarm x {k} ticks x {reps} reps ({el:.1f} s), float64 C "
                      f"restatement of QuadGroup.step (oracle/quad_oracle.c), {threads} threads"}


def _ref_rows(n_total: int) -> int:
    """How many of the swarm's rows the reference workers can hold (~1.8 KB of
    numpy state + workspaces per agent, measured) in half the free memory."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        return n_total
    return max(1, min(n_total, int(avail * 0.5 / 2000)))


def reference_leg(n_total: int, dt: float, ticks: int, samples: int, warm: int) -> dict | None:
    """The unmodified reference QuadGroup.step (oracle/_ref) on the swarm's rows,
    sharded over every host core; None when the reference is not installed."""
    from oracle import ref_runner
    if not ref_runner.available():
        return None
    n_ref = _ref_rows(n_total)
    r = ref_runner.run_quadgroup(n_total, dt, ticks=ticks, samples=samples, warm=warm, n_rows=n_ref)
    rows = f"all {n_total:,} agents" if n_ref == n_total else f"rows [0, {n_ref:,}) of the {n_total:,} agents"
    return {"value": r["value"], "unit": UNIT, "cores": r["procs"], "kind": "reference",
            "sample": f"the unmodified reference swarmstep QuadGroup.step (core.py:166-202, oracle/_ref) on {rows} "
                      f"of this swarm, sharded by index over {r['procs']} processes (numpy 1 thread each), "
                      f"{samples} x {ticks} tick(s) timed after {warm} warm tick(s); sample time = max over "
                      f"processes; {r['wall_s']:.1f} s",
            "agents": n_ref, "ms_per_sample": [t * 1e3 for t in r["sample_s"]],
            "per_core_median": r["per_core_median"], "faults": r["faults"]}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    world = max(1, args.gpus)
    n_total, scaling = layout(args, world)
    port = port_leg(n_total, args.substeps, args.dt, args.cpu_seconds, args.motor_tau)
    ref = None if args.motor_tau > 0 else reference_leg(n_total, args.dt, args.ref_ticks, args.steps,
                                                        args.warmup * args.ref_ticks)
    cfg = config(args, world)
    if ref is not None:
        value, cb = ref["value"], dict(ref)
        ms = statistics.mean(ref["ms_per_sample"])
        cfg["ticks_per_step"] = args.ref_ticks
        cfg["note"] = (f"one timed step = {args.ref_ticks} tick(s) of the whole swarm (the reference has no "
                       f"fused launch); same agents, setpoints and metric as the B200 arm")
    else:
        # motor lag (absent in the reference) or no oracle/_ref: the C port
        value, cb = port["value"], dict(port)
        ms = (min(262_144, n_total) * args.substeps) / value * 1e3
        cfg["note"] = "reference not runnable for this config: float64 C port of QuadGroup.step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": cb, "port": port if ref is not None else None,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def run_b200(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2308_12698_b200 import B200QuadGroup
    from paper_2308_12698_b200.synthetic import swarm

    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n_total, scaling = layout(args, world)
    lo, hi = rank_rows(args, rank, world)
    n, k, dt = hi - lo, args.substeps, args.dt
    nccl = _backend() == "nccl"

    def barrier():
        if world > 1:
            if nccl:
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()

    t_setup = time.perf_counter()
    pos, sp = swarm(n_total, lo, hi)
    g = B200QuadGroup(0, _Batch(n, pos, lo), device=dev, motor_tau=args.motor_tau)
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
        return e0.elapsed_time(e1)

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
    ms_rank = timed(lambda: g.step_async(dt, k), args.steps, g.stream)
    clk = clocks.stop()
    ms = max_over_ranks(ms_rank)
    faults = sum(f.size for f in g.collect_faults())
    ms_per_step = ms / args.steps
    value = n_total * k * args.steps / (ms * 1e-3)
    # roofline of this rank's kernel (rank 0 prints): its own launches and rows
    launch_s = ms_rank / args.steps * 1e-3
    achieved_tf = n * k * ALG_FLOPS_PER_AGENT_TICK / launch_s / 1e12
    sm_mhz = clk.get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_nominal_tf = sms * 128 * 2 * sm_mhz * 1e6 / 1e12
    fp32_meas = _fp32_peak()
    nominal_src = f"{sms} SMs x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz"
    if fp32_meas:
        fp32_peak_tf = fp32_meas["tflops"]
        peak_source = (f"builder-measured: FP32 microbenchmark tools/fp32_peak.cu on this GPU (best of FFMA "
                       f"register / immediate / packed FFMA2: {fp32_meas['form']}); MEASURED_PEAKS.json has no "
                       f"FP32 SIMT figure; nominal {fp32_nominal_tf:.1f} TFLOP/s = {nominal_src} (frac_nominal)")
    else:
        fp32_peak_tf = fp32_nominal_tf
        peak_source = f"nominal: {nominal_src} (MEASURED_PEAKS.json has no FP32 SIMT figure)"

    # ---- K=1 leg: the same step in its HBM-bound regime
    k1 = None
    if not args.no_k1:
        for _ in range(3):
            g.step_async(dt, 1)
        g.collect_faults()
        ms1 = timed(lambda: g.step_async(dt, 1), args.steps, g.stream)
        g.collect_faults()
        t1 = ms1 / args.steps * 1e-3
        peaks = _peaks()
        gbs = ALG_BYTES_PER_AGENT_LAUNCH * n / t1 / 1e9
        gbs_ovh = BYTES_WITH_OVERHEAD * n / t1 / 1e9
        k1 = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
              "frac": gbs / peaks["hbm_gbs"], "traffic": _traffic("k1", n),
              "bytes_per_agent": ALG_BYTES_PER_AGENT_LAUNCH,
              "bytes_basis": "SURVEY.md 8(d): 182 B per agent per launch (state, PID, setpoints, flags)",
              "with_overhead": {"bytes_per_agent": BYTES_WITH_OVERHEAD, "achieved": gbs_ovh,
                                "frac": gbs_ovh / peaks["hbm_gbs"],
                                "note": "182 B + packed position low-part word (8 B) + stale MOTOR setpoints (16 B) as moved"},
              "ms_per_launch": t1 * 1e3, "agent_steps_per_s": n / t1, "peak_source": peaks["source"]}

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
        e2e = {"value": n_total * k * args.steps / el, "unit": UNIT,
               "h2d_bytes_per_step": int(7 * 4 * n_total), "d2h_bytes_per_step": 16 * world,
               "ms_per_step": el / args.steps * 1e3,
               "path": "B200QuadGroup.set_setpoints(pinned host) + step_async(dt, K) + collect_faults() per rank"}
        # informative: the same public-API loop with the setpoints generated on
        # the device (the circle strategy fused into the step,
        # CircleFeed.step_fused) -- no per-step setpoint upload, so this is NOT
        # the e2e figure above (a different setpoint stream, inputs on device)
        if args.motor_tau == 0.0:
            from paper_2308_12698_b200.feed import CircleFeed
            feed = CircleFeed(g, dt)

            def feed_run(steps):
                for _ in range(steps):
                    feed.step_fused(k)
                    g.collect_faults()

            feed_run(args.warmup)
            barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            feed_run(args.steps)
            torch.cuda.synchronize(dev)
            el = max_over_ranks(time.perf_counter() - t0)
            barrier()
            e2e["device_feed"] = {"value": n_total * k * args.steps / el, "ms_per_step": el / args.steps * 1e3,
                                  "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 16 * world,
                                  "path": "CircleFeed.step_fused(K) + collect_faults() per rank (setpoints "
                                          "generated on the device; informative, not the e2e figure)"}

    # ---- the reference's CPU path beside the GPU number (rank 0, after the
    # timed regions; every N): the unmodified reference QuadGroup.step on this
    # swarm over all host cores, plus the float64 C port
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        port = port_leg(n_total, k, dt, args.cpu_seconds, args.motor_tau)
        ref = None if args.motor_tau > 0 else reference_leg(n_total, dt, 1, args.cpu_samples, 1)
        cpu = dict(ref, port=port) if ref is not None else port

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config(args, world),
            "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": fp32_peak_tf, "unit": "TFLOP/s",
                         "frac": achieved_tf / fp32_peak_tf, "frac_nominal": achieved_tf / fp32_nominal_tf,
                         "peak_nominal": fp32_nominal_tf, "traffic": _traffic("k10", n),
                         "flops_per_agent_tick": ALG_FLOPS_PER_AGENT_TICK, "agents_per_launch": n,
                         "peak_source": peak_source, "fp32_peak_measurements": fp32_meas},
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
