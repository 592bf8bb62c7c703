#!/usr/bin/env python
"""bench.py -- amplitude-gate updates/s of the B200 gate engine.

Workload (BASELINE.json configs[1] = "config 2"): random circuit on 24 qubits,
complex128, depth 40 (Haar U2 on every qubit + brickwork CNOTs), initial
|0..0>, 1420 gates.  One step = qsim_init_basis + qsim_run_circuit(all 1420
gates) + qsim_expectations (<Q_i> of every qubit, read back to
the host): every hot-path row of SURVEY.md §8(a) that this circuit uses.
metric = N_O * 2^n / t  (N_O = user gates per step).

N > 1 (torchrun, one rank per GPU, NCCL): weak scaling, n = 24 + log2(N)
qubits of the same circuit family sharded over the N GPUs.

--impl reference runs the CPU oracle (oracle/) on a bounded sample of the
same workload on the host cores (there is no reference implementation).
"""
from __future__ import annotations

import argparse
import csv
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "amplitude-gate updates/s"
UNIT = "AGU/s"
DEPTH = 40
TIMING_EVERY = 4  # roofline events on every 4th step of the timed region
CPU_LAYERS, CPU_REPS = DEPTH, 2  # cpu_baseline sample: two whole steps of the workload (~12 s on 16 cores)
BASE_QUBITS = 24


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(d.get("sm_max_mhz", 1965.0))
    return 6650.0, "fallback (B200_PROFILING.md)", 1965.0


# FP64 ALU peak: 148 SMs x 64 FP64 FMA lanes/clk x 2 flop x max SM clock.
# tools/fp64_peak.cu measured 34.1 TFLOP/s sustained on this pool's B200 (0.92 of it).
FP64_FMA_PER_CLK_PER_SM = 64
N_SM = 148


class Clocks:
    """SM clock and clock-event reasons sampled DURING the timed region: an NVML
    thread every 2 ms (nvidia_ml_py), falling back to `nvidia-smi -lms`."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.stop_flag = False
        self.thread = self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def _nvml_loop(self, nv, h):
        while not self.stop_flag:
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, const in self.REASONS:
                    if r & getattr(nv, const):
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "10"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(1.0)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self.stop_flag = True
            self.thread.join(timeout=5)
            if not self.samples:
                return None
            return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml 2 ms"}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for r in csv.reader(open(self.path)):
            if len(r) >= 9:
                rows.append([x.strip() for x in r])
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


def pass_roofline(n: int, world: int, gates, fp64_tflops: float, hbm_gbs: float):
    """Per-launch roofline of the planned passes (host planner, same plan as
    the engine): each pass needs max(FP64 FMA-slot work / FP64 peak, 32 B/amp /
    HBM peak).  Returns (sum over passes of that bound in ms, FMA-slots per amp)."""
    from paper_quant_ph_0608239_b200 import plan_json
    G = (world - 1).bit_length()
    amps = float(1 << (n - G))
    d = json.loads(plan_json(n, world, gates))
    cost = {0: 8.0, 1: 4.0, 3: 4.0, 5: 4.0, 7: 16.0}
    t = slots = 0.0
    for st in d["plan"]["steps"]:
        if st["type"] != "pass":
            continue
        f = 0.0
        for op in st["ops"]:
            bits = sum(bin(op[k]).count("1") for k in ("mreg", "mlane", "mwarp", "mout"))
            f += cost.get(op["code"], 0.0) / (1 << bits)
        slots += f
        t += max(2.0 * f * amps / (fp64_tflops * 1e12), 32.0 * amps / (hbm_gbs * 1e9))
    return 1e3 * t, slots


def cpu_sample(layers: int, reps: int = 1):
    """The oracle on the first `layers` layers of the same 24-qubit circuit,
    `reps` times (state re-initialised), with <Q_i> each time."""
    import oracle
    from workloads import circuits as C
    gates = C.random_brickwork(BASE_QUBITS, layers, seed=2)
    o = oracle.Oracle(BASE_QUBITS)
    t = 0.0
    for _ in range(reps):
        o.init_basis(0)
        t0 = time.perf_counter()
        o.run(gates)
        o.expectations()
        t += time.perf_counter() - t0
    return reps * len(gates) * (1 << BASE_QUBITS) / t, t, len(gates), oracle.Oracle.threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    layers = 10  # a quarter of the circuit per step (~1.3 s on 16 cores): the run stays within minutes
    for _ in range(args.warmup):
        cpu_sample(layers)
    vals, tot = [], 0.0
    for _ in range(args.steps):
        v, t, ng, cores = cpu_sample(layers)
        vals.append(v)
        tot += t
    value = args.steps * ng * (1 << BASE_QUBITS) / tot
    sample = f"first {layers} of {DEPTH} layers ({ng} gates) of the config-2 circuit at {BASE_QUBITS} qubits, + <Q_i>"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "config2_random_brickwork", "n_qubits": BASE_QUBITS, "depth": DEPTH},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_quant_ph_0608239_b200 import QSim, pack_gates
    from paper_quant_ph_0608239_b200 import _native as N
    from workloads import circuits as C

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G = (world - 1).bit_length()
    n = BASE_QUBITS + G
    gates = C.random_brickwork(n, DEPTH, seed=2)
    n_o = len(gates)
    packed = pack_gates(gates)
    sim = QSim.distributed(n) if world > 1 else QSim(n)
    sim.set_option("timing", 1)  # CUDA events around pass launches (roofline)
    stream = sim.stream

    # <Q_i> of every step goes to pinned host memory with an async copy, so the
    # host enqueues step k+1 while step k runs (the synchronous readout idles
    # the device for the host's per-step work; reported as e2e.value_sync_readout)
    ex_buf = torch.empty(n, dtype=torch.float64, pin_memory=True)

    def step():
        sim.init_basis(0)
        sim.run_circuit(gates, packed=packed)
        sim.expectations_async(ex_buf)

    def step_sync():
        sim.init_basis(0)
        sim.run_circuit(gates, packed=packed)
        return sim.expectations()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        step()
    sim.sync()
    ex = ex_buf.numpy().copy()
    # sanity: <Q_i> in [0,1], equal to the synchronous readout, and norm 1 before timing
    assert np.array_equal(ex, step_sync())
    assert abs(sim.norm() - 1) < 1e-10 and all(0 <= x <= 1 for x in ex)

    # ---- device-timed region (events on the engine's stream)
    clocks = Clocks(local)
    barrier()
    sim.reset_stats()
    clocks.start()
    # per-kernel events (roofline) on every TIMING_EVERY-th step of the region:
    # an event pair around each pass costs ~1.6% of a step when on every step
    n_timed = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        on = k % TIMING_EVERY == 0
        n_timed += on
        sim.set_option("timing", int(on))
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    ms = e0.elapsed_time(e1)
    st = sim.stats()
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = args.steps * n_o * float(1 << n) / (ms / 1e3)

    # ---- end-to-end through the public C-ABI with host buffers: the host
    # gate array (qsim_gate[]) is validated, planned (plan cache off) and
    # uploaded every step and <Q_i> comes back to host memory; wall clock,
    # max over ranks.
    sim.set_option("timing", 0)  # the library default: no per-kernel events
    sim.set_option("plan_cache", 0)
    step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    barrier()
    wall = time.perf_counter() - t0
    # the same with a synchronous readout every step (host and device alternate)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_sync()
    barrier()
    tw = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
    e2e_sync = args.steps * n_o * float(1 << n) / float(tw.item())
    sim.set_option("plan_cache", 1)
    tw = torch.tensor([wall], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
    wall = float(tw.item())
    e2e = args.steps * n_o * float(1 << n) / wall
    # the same with the library's default plan cache (a repeated circuit is
    # validated and uploaded every step but planned once)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    barrier()
    tw = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
    e2e_cached = args.steps * n_o * float(1 << n) / float(tw.item())
    import ctypes
    h2d = n_o * ctypes.sizeof(N.qsim_gate)

    hbm_peak, peak_src, sm_max = peaks()
    pass_ms = st["pass_ms"]
    fp64_peak = 2.0 * FP64_FMA_PER_CLK_PER_SM * N_SM * sm_max * 1e6 / 1e12  # TFLOP/s
    fp64_ach = (2.0 * st["pass_fp64_slots"] / (pass_ms / 1e3) / 1e12) if pass_ms > 0 else None
    hbm_ach = (st["pass_amp_bytes"] / (pass_ms / 1e3) / 1e9) if pass_ms > 0 else None
    t_min_ms, _ = pass_roofline(n, world, gates, fp64_peak, hbm_peak)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "pass_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2_random_brickwork" if world == 1 else "config2_family_weak",
                       "n_qubits": n, "depth": DEPTH, "gates_per_step": n_o, "shard_qubits": n - G,
                       "parallelism": f"sharded{world}" if world > 1 else "single",
                       "l2": "state %d MiB per GPU > 126 MB L2 (no flush needed)" % ((16 << (n - G)) >> 20)},
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * n,
                    "plan_cache": "off: every step validates, plans and uploads the gate list",
                    "readout": "<Q_i> copied to pinned host memory every step (async); host syncs at the end",
                    "value_sync_readout": e2e_sync,
                    "value_plan_cached": e2e_cached},
            "gpu_launches": int(st["kernel_launches"]),
            "roofline": {"bound": "alu", "achieved": fp64_ach, "peak": fp64_peak, "unit": "TFLOP/s",
                         "frac": (fp64_ach / fp64_peak) if fp64_ach else None, "traffic": traffic,
                         "kernel": "qsim_pass (NVRTC pass-specialised k_pass)",
                         "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x %.0f MHz" % sm_max,
                         "launches": int(st["passes"] * n_timed / args.steps), "kernel_ms": pass_ms,
                         "timed_steps": f"{n_timed} of {args.steps} (every {TIMING_EVERY}th)",
                         "kernel_share_of_step": pass_ms / (ms * n_timed / args.steps) if ms > 0 else None,
                         # per-launch bound max(FP64, HBM) summed over the passes of a step
                         "per_pass_bound": {"t_min_ms_per_step": t_min_ms,
                                            "frac": (t_min_ms * n_timed / pass_ms) if pass_ms > 0 else None},
                         "hbm": {"achieved": hbm_ach, "peak": hbm_peak, "unit": "GB/s",
                                 "frac": (hbm_ach / hbm_peak) if hbm_ach else None, "peak_source": peak_src,
                                 "bytes_per_launch": 32 << (n - G)}},
            "clocks": ck,
            "detail": {"passes_per_step": st["passes"] / args.steps, "plan_ms_per_step": st["plan_ms"] / args.steps,
                       "jit_passes_per_step": st["jit_launches"] / args.steps,
                       "plan_cache_hits": int(st["plan_cache_hits"]),
                       "exchanges_per_step": st["exchanges"] / args.steps,
                       "reduce_ms_per_step": st["reduce_ms"] / args.steps},
        }
        if world == 1 and not args.no_cpu_baseline:
            v, tcpu, ng, cores = cpu_sample(CPU_LAYERS, CPU_REPS)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                    "sample": f"{CPU_REPS} steps of the first {CPU_LAYERS} of {DEPTH} layers ({ng} gates) of the same circuit, "
                                              f"{tcpu:.1f} s"}
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
