#!/usr/bin/env python
"""Benchmark of the QVA hot path (BASELINE.json metric: amplitude-layers/s and achieved HBM
GB/s, fp64 complex, at 1/2/4/8 B200).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4|cfg5|cfg5w|cfg2|cfg3|cfg1]
                  [--impl ours|reference]
  N > 1: python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
             --master-port P bench.py --gpus N ...

A step = one full evaluation of the objective f(theta) = <psi(theta)|Q|psi(theta)>
(all p layers of phase + mixer, then <Q>) on seeded synthetic inputs (qva_inputs).
Default workload: N=1 -> cfg4 (QAOA MaxCut n=30, p=3); N>1 -> cfg5 family with 2^30
amplitudes per GPU (n = 30 + log2 N, p=2, sharded over the GPUs with the global<->local
qubit all-to-all), i.e. weak scaling.  Every state is 16 GiB per GPU, larger than L2, so no
L2 flush is needed between steps.

`value`  : device-timed (CUDA events on the launch stream, barrier + synchronize on both sides,
           max over ranks) whole-job amp-layers/s with q already resident in HBM.
`e2e`    : same metric through the public API with HOST buffers: each step uploads q from
           pinned host memory (qva_set_qualities), evolves from a host theta and reads <Q> back.
`roofline`: dominant kernel (the X-mixer tile pass): algorithmic bytes per launch / mean launch
           time (CUDA events around each launch on the plan's stream) vs measured HBM copy peak.
`cpu_baseline` / --impl reference: the CPU oracle (oracle/) on a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from qva_inputs import make_config  # noqa: E402

METRIC = "amplitude-layers/sec and achieved HBM GB/s (fp64 complex) at 1/2/4/8 B200"
UNIT = "amp-layers/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic(kernel: str):
    """dram read+write bytes per launch from the committed ncu --set full capture, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        if os.environ.get("QVA_BENCH_NO_SMI"):  # diagnostics only: no clock sampling
            self.proc = None
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                for k, nm in enumerate(names):
                    if r[3 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def total_bytes_step_gpu(plan, Q, steps):
    """implemented bytes of every kernel class per step (this GPU)"""
    return sum(plan.kernel_stats(c)["bytes"] for c in Q.KERNEL_CLASSES) / steps


def local_n_of(plan):
    return plan.get_partition()[0]


def host_info():
    """nproc, CPU model and MemTotal of the box the oracle is timed on."""
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal"):
                    info["mem_total_gib"] = round(int(line.split()[1]) / 1048576.0, 1)
                    break
    except Exception:
        pass
    return info


# SURVEY 8(d) algorithmic floor of the X-mixer path: two HBM round trips (2 x 32 B) per
# amplitude-layer, q generated inside the passes (NEXT-1) so no q bytes
FLOOR_X_BYTES = 64.0
# NVLink per direction per GPU: measured peer copy on this pool (B200_PROFILING.md); nominal 900
NVL_GBS, NVL_NOMINAL_GBS = 770.0, 900.0


def workload_for(args, world):
    if args.workload:
        name = args.workload
    else:
        name = "cfg4" if world == 1 else "cfg5w"
    if name == "cfg5w":
        n = 30 + int(round(math.log2(world)))
        wl = make_config("cfg5", n_override=n)
        desc = f"cfg5 family weak scaling: QAOA weighted MaxCut n={n} (2^30 amps/GPU), 4-regular, p={wl.p}"
    elif name == "cfg5":
        wl = make_config("cfg5")
        desc = f"cfg5: QAOA weighted MaxCut n={wl.n_qubits}, 4-regular, p={wl.p}, sharded"
    elif name == "cfg4":
        wl = make_config("cfg4")
        desc = f"cfg4: QAOA MaxCut n={wl.n_qubits} (16 GiB state), random 3-regular, unit weights, p={wl.p}"
    elif name == "cfg2":
        wl = make_config("cfg2")
        desc = "cfg2: QAOA weighted MaxCut n=20, G(20,0.5), p=5, batch of 21 FD parameter sets"
    elif name == "cfg3":
        wl = make_config("cfg3")
        desc = "cfg3: QWOA N=10!, q~N(0,1), complete-graph Laplacian circulant mixer via FFT, p=4"
    elif name == "qwoa12":
        wl = make_config("cfg3", n_override=479001600)
        desc = "NEXT-4: QWOA N=12! (479,001,600 states, 7.7 GB), q~N(0,1), K_N Laplacian circulant, three-level FFT, p=4"
    elif name == "cfg1":
        wl = make_config("cfg1")
        desc = "cfg1: QAOA MaxCut n=10, 3-regular, p=2"
    elif name == "cfg3cf":
        wl = make_config("cfg3")
        desc = ("cfg3 with the K_N closed-form mixer (opt-in reference path, SURVEY K10): QWOA N=10!, "
                "q~N(0,1), lambda=(0,N,...,N), p=4")
    elif name == "qaoaz28":
        wl = make_config("cfg4", n_override=28, p_override=2)
        wl.mixer = "parity"
        desc = ("NEXT-2: QAOAz, parity (XY) mixer over qubits 0..27 (B_odd, B_even), n=28, max-cut q of the "
                "cfg4 recipe generated on the device, p=2, from a Hamming-weight-14 basis state")
    else:
        raise SystemExit(f"unknown workload {name}")
    return name, wl, desc


# ---------------------------------------------------------------------------------------------
# CPU oracle arm (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------------
ONE_THREAD = {}  # filled by oracle_sample for the X-mixer recipes: the oracle on one OpenMP thread


def oracle_sample(name, wl, budget_s=20.0):
    """Time the CPU oracle, as it stands, on a bounded sample of the same workload.
    Returns (amp-layers/s, seconds, cores, sample description)."""
    import oracle as O
    cores = O.num_threads()

    def run(swl):
        q = O.maxcut_q(swl.n_qubits, swl.edges_u, swl.edges_v, swl.weights)
        t0 = time.perf_counter()
        psi = O.evolve_x(swl.n_qubits, q, swl.theta)
        f = O.expectation(psi, q)
        return time.perf_counter() - t0, f

    if wl.mixer == "x" and name in ("cfg4", "cfg5", "cfg5w"):
        fam = "cfg4" if name == "cfg4" else "cfg5"
        step = 2 if fam == "cfg4" else 1          # 3-regular graphs need an even vertex count
        n0 = 20
        t0, _ = run(make_config(fam, n_override=n0))
        n = n0
        while n + step <= wl.n_qubits and t0 * 2 ** (n + step - n0) * (n + step) / n0 <= budget_s:
            n += step
        swl = make_config(fam, n_override=n)
        dt, f = run(swl)
        desc = (f"oracle full p={swl.p} evolution + <Q> of the {fam} recipe at n={n} (2^{n} amplitudes; "
                f"the full workload has 2^{wl.n_qubits}), {cores} OpenMP threads, f={f:.6f}")
        # the same oracle on one thread (both core counts), on a smaller sample
        n1 = max(n0, n - 4 if fam == "cfg4" else n - 4)
        O.set_num_threads(1)
        try:
            s1 = make_config(fam, n_override=n1)
            dt1, _ = run(s1)
        finally:
            O.set_num_threads(cores)
        ONE_THREAD.update({"value": (1 << n1) * s1.p / dt1, "cores": 1, "sample": f"n={n1}, 1 thread",
                           "seconds": dt1})
        return (1 << n) * swl.p / dt, dt, cores, desc
    if wl.mixer == "x":
        B = len(wl.batch_thetas) if wl.batch_thetas is not None else 1
        q = O.maxcut_q(wl.n_qubits, wl.edges_u, wl.edges_v, wl.weights)
        t0 = time.perf_counter()
        nb = 0
        thetas = wl.batch_thetas if wl.batch_thetas is not None else [wl.theta]
        for th in thetas:
            O.expectation(O.evolve_x(wl.n_qubits, q, th), q)
            nb += 1
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        desc = f"oracle evolution + <Q> of {nb} of the {B} parameter sets of {name} (n={wl.n_qubits}), {cores} threads"
        return wl.dim * wl.p * nb / dt, dt, cores, desc
    if wl.mixer == "parity":  # QAOAz: the oracle's pair-term loops on a smaller slice of the recipe
        n = min(wl.n_qubits, 22)
        swl = make_config("cfg4", n_override=n, p_override=wl.p)
        q = O.maxcut_q(n, swl.edges_u, swl.edges_v)
        psi0 = np.zeros(1 << n, np.complex128)
        psi0[(1 << (n // 2)) - 1] = 1.0
        t0 = time.perf_counter()
        psi = O.evolve_parity(n, q, list(range(n)), swl.theta, psi0)
        O.expectation(psi, q)
        dt = time.perf_counter() - t0
        return (1 << n) * wl.p / dt, dt, cores, f"oracle QAOAz evolution + <Q> at n={n} (the workload has n={wl.n_qubits}), {cores} threads"
    # circulant: closed-form oracle on the full cfg3 size
    t0 = time.perf_counter()
    psi = O.evolve_complete(wl.q, wl.theta, wl.lam0, wl.lam_rest)
    O.expectation(psi, wl.q)
    dt = time.perf_counter() - t0
    return wl.dim * wl.p / dt, dt, cores, f"oracle closed-form QWOA evolution at N={wl.dim}, p={wl.p}, {cores} threads"


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    name, wl, desc = workload_for(args, world)
    budget = max(3.0, 150.0 / max(1, args.steps + args.warmup))
    vals, times = [], []
    info = None
    for i in range(args.warmup + args.steps):
        v, dt, cores, sdesc = oracle_sample(name, wl, budget_s=budget)
        if i >= args.warmup:
            vals.append(v)
            times.append(dt)
        info = (cores, sdesc)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info[0], "kind": "oracle", "sample": info[1],
                         "host": host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--virtual-shards", type=int, default=1,
                    help="run the sharded schedule with G virtual shards on one GPU (format check of the "
                         "sharded roofline fields before a multi-GPU node exists)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2110_03963_b200 as Q

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    name, wl, desc = workload_for(args, world)
    # a dedicated (non-default) stream: the plan launches on it and the CUDA events below are
    # recorded on it, so they bracket exactly the plan's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    nccl_id = Q.nccl_id_broadcast() if world > 1 else None

    batch = wl.batch_thetas if name == "cfg2" else None
    vshards = max(1, args.virtual_shards) if world == 1 else 1
    plan = Q.Plan(wl.dim, wl.mixer, n_qubits=wl.n_qubits, rank=rank, world=world, nccl_id=nccl_id,
                  device=local_rank, stream=stream.cuda_stream, max_batch=len(batch) if batch is not None else 1,
                  virtual_shards=vshards, peer_store_exchange=vshards > 1, complete_closed_form=name == "cfg3cf")
    G = world * vshards
    if wl.mixer in ("x", "parity"):
        plan.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
        if wl.mixer == "parity":
            psi0 = np.zeros(local_n_of(plan), np.complex128)
            psi0[(1 << (wl.n_qubits // 2)) - 1] = 1.0
            plan.set_initial_state(psi0)
    else:
        plan.set_qualities(wl.q)
        plan.set_circulant_eigenvalues_const(wl.lam0, wl.lam_rest)
    local_n, offset = plan.get_partition()
    theta = wl.theta
    B = len(batch) if batch is not None else 1

    def step():
        if batch is not None:
            return plan.evolve_batch(batch)
        plan.evolve(theta)
        return plan.expectation()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # CUDA events around every launch, on the plan's stream, in the timed region; switched on before
    # the warm-up so that the evaluation's replayed CUDA graph already carries them (event nodes)
    plan.set_profiling(True)
    for _ in range(args.warmup):
        step()
    barrier()

    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    plan.reset_kernel_stats()
    l0 = plan.launch_count()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        f = step()
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = plan.launch_count() - l0
    clk = clocks.stop()
    plan.set_profiling(False)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    amp_layers = float(wl.dim) * wl.p * B  # whole job, per step
    value = amp_layers / (ms_step * 1e-3)

    # dominant kernel
    if wl.mixer in ("x", "parity"):
        cls = "tile" if wl.n_qubits > 12 else "small"
    else:
        cls = "other" if name == "cfg3cf" else "fft_col"
    st = plan.kernel_stats(cls)
    kernel_share = None
    total_kernel_ms = sum(plan.kernel_stats(c)["ms"] for c in Q.KERNEL_CLASSES)
    if total_kernel_ms > 0:
        kernel_share = st["ms"] / total_kernel_ms
    peak, peak_src = _peaks()
    roof = None
    per_gpu = vshards if world == 1 else 1  # shards whose work one GPU does
    if st["launches"] > 0 and st["ms"] > 0:
        impl_bytes = st["bytes"] / st["launches"]
        per_launch_s = st["ms"] * 1e-3 / st["launches"]
        if cls == "tile" and wl.mixer == "x" and local_n >= (1 << 24):
            # algorithmic bytes per launch = the SURVEY 8(d) floor (64 B per amplitude-layer) x the
            # amplitude-layers one launch processes (this GPU's amp-layers of the timed steps over its
            # tile-pass launches)
            amp_layers_per_launch = amp_layers / G * per_gpu * args.steps / st["launches"]
            per_launch_bytes = FLOOR_X_BYTES * amp_layers_per_launch
            basis = (f"SURVEY 8(d) floor {FLOOR_X_BYTES:.0f} B/amp-layer x {amp_layers_per_launch:.6g} amp-layers "
                     "per launch")
        else:
            per_launch_bytes = impl_bytes
            basis = ("bytes of the implemented schedule (state round trip + q/spectrum reads) per launch"
                     + (" (the SURVEY 8(d) 64 B floor is stated for n >= 24; below it fewer passes per layer "
                        "suffice)" if cls == "tile" else ""))
        achieved = per_launch_bytes / per_launch_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": _ncu_traffic(cls), "kernel": f"{cls} pass", "algorithmic_bytes_per_launch": per_launch_bytes,
                "algorithmic_basis": basis, "implemented_bytes_per_launch": impl_bytes,
                "frac_implemented": impl_bytes / per_launch_s / 1e9 / peak,
                "mean_launch_ms": st["ms"] / st["launches"], "launches": st["launches"],
                "share_of_kernel_time": kernel_share, "peak_source": peak_src}
        if cls == "tile" and wl.mixer == "x" and local_n >= (1 << 24):
            # the whole step against the floor (every kernel and gap of the step included)
            roof["frac_step_vs_floor"] = FLOOR_X_BYTES * amp_layers / G * per_gpu / (ms_step * 1e-3) / 1e9 / peak
    # sharded runs: combined HBM / NVLink roofline per layer:
    # T_roof = max(T_HBM, T_NVL), frac = T_roof / T_layer
    sharded = None
    if G > 1:
        xfer = plan.query("xfer_bytes") / args.steps  # bytes one shard sends to the others, per step
        layers = wl.p * B
        t_nvl = xfer / (NVL_GBS * 1e9)
        if wl.mixer == "x":
            hbm_bytes = FLOOR_X_BYTES * float(wl.dim) * wl.p * B / G * per_gpu
        else:
            hbm_bytes = total_bytes_step_gpu(plan, Q, args.steps)
        t_hbm = hbm_bytes / (peak * 1e9)
        t_roof = max(t_hbm, t_nvl)
        sharded = {"shards": G, "virtual": world == 1, "nvlink_bytes_per_gpu_step": xfer,
                   "nvlink_bytes_per_gpu_layer": xfer / layers, "t_nvl_ms_per_layer": 1e3 * t_nvl / layers,
                   "t_hbm_ms_per_layer": 1e3 * t_hbm / layers, "t_layer_ms": ms_step / layers,
                   "bound": "nvlink" if t_nvl > t_hbm else "hbm", "frac": 1e3 * t_roof / ms_step,
                   "nvlink_gbs": NVL_GBS, "nvlink_nominal_gbs": NVL_NOMINAL_GBS,
                   "nvlink_source": "measured peer copy per direction per GPU (B200_PROFILING.md)",
                   "hbm_basis": ("SURVEY 8(d) floor 64 B/amp-layer" if wl.mixer == "x" else
                                 "implemented bytes of every kernel"),
                   "note": ("virtual shards on one GPU: the NVLink bytes are the traffic each shard would send "
                            "on a real node; t_hbm covers all shards of the one GPU") if world == 1 else None}
    # whole-step model bytes (all kernels' algorithmic bytes) / step time
    total_bytes = sum(plan.kernel_stats(c)["bytes"] for c in Q.KERNEL_CLASSES)
    achieved_step_gbs = total_bytes / args.steps / (ms_step * 1e-3) / 1e9 / max(1, 1)
    if roof is not None:
        # every kernel's implemented bytes of a step over the step time: unaffected by launches that
        # overlap on several streams (the three-level FFT's grouped inner passes, whose per-launch
        # event times include the concurrent group's share of the SMs)
        roof["frac_step_implemented"] = achieved_step_gbs / peak

    # ---- e2e through the public API with host buffers.  The step's inputs are the problem
    # (MaxCut graph: edge list + weights) and theta, copied from pinned host memory; q is derived
    # on the device by qva_set_qualities_maxcut, as the paper's observable functions generate the
    # qualities in parallel on each rank (Table 2).  A second variant uploads the
    # full fp64 q vector from pinned host memory (a user holding arbitrary qualities).
    e2e = None
    if not args.no_e2e and wl.mixer == "x" and batch is None:
        th_host = torch.from_numpy(np.ascontiguousarray(theta, np.float64)).pin_memory().numpy()
        eu = torch.from_numpy(np.ascontiguousarray(wl.edges_u, np.int32)).pin_memory().numpy()
        evv = torch.from_numpy(np.ascontiguousarray(wl.edges_v, np.int32)).pin_memory().numpy()
        ew = (torch.from_numpy(np.ascontiguousarray(wl.weights, np.float64)).pin_memory().numpy()
              if wl.weights is not None else None)
        ksteps = max(2, min(args.steps, 5))

        def timed(body):
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            for _ in range(ksteps):
                fe = body()
            e1.record(stream)
            barrier()
            wall = time.perf_counter() - t0
            ems = e0.elapsed_time(e1)
            if dist is not None:
                t = torch.tensor([ems], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ems = float(t.item())
            assert abs(fe - f) <= 1e-9 * max(1.0, abs(f)), (fe, f)
            return ems / ksteps, wall * 1e3 / ksteps

        def graph_step():
            plan.set_qualities_maxcut(eu, evv, ew)
            plan.evolve(th_host)
            return plan.expectation()

        ems, wms = timed(graph_step)
        h2d = int(eu.nbytes + evv.nbytes + (ew.nbytes if ew is not None else 0) + th_host.nbytes)
        e2e = {"value": amp_layers / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8,
               "ms_per_step": ems, "wall_ms_per_step": wms, "steps": ksteps,
               "what": "qva_set_qualities_maxcut(pinned host graph) + qva_evolve(pinned host theta) + "
                       "qva_expectation -> host, every step"}
        q_host = torch.empty(local_n, dtype=torch.float64, pin_memory=True)
        qn = q_host.numpy()
        plan.get_qualities(offset, local_n, out=qn)

        def q_step():
            plan.set_qualities(qn, offset)
            plan.evolve(th_host)
            return plan.expectation()

        q_step()  # untimed warm-up: the graph -> stored q switch allocates q and its code buffers once
        ems2, wms2 = timed(q_step)
        e2e["host_q_variant"] = {"value": amp_layers / (ems2 * 1e-3), "unit": UNIT,
                                 "h2d_bytes_per_step": int(local_n * 8 + th_host.nbytes), "d2h_bytes_per_step": 8,
                                 "ms_per_step": ems2, "wall_ms_per_step": wms2,
                                 "what": "qva_set_qualities(pinned host fp64 q) + qva_evolve + qva_expectation"}
        del q_host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, cores, sdesc = oracle_sample(name, wl, budget_s=20.0)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sdesc, "seconds": dt,
               "host": host_info()}
        if ONE_THREAD:
            cpu["single_thread"] = dict(ONE_THREAD, unit=UNIT)

    # working set of the timed step vs this device's L2 (cudaDevAttrL2CacheSize)
    l2_bytes = torch.cuda.get_device_properties(local_rank).L2_cache_size
    ws = local_n * B * 16
    l2_label = (f"inputs larger than L2: {ws / 2**30:.2f} GiB of state per GPU vs {l2_bytes / 2**20:.0f} MiB L2, no flush"
                if ws > 2 * l2_bytes else
                f"working set {ws / 2**20:.0f} MiB of state vs {l2_bytes / 2**20:.0f} MiB L2: L2-resident or near it, "
                "no flush (the workload's own size)")
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "dim": wl.dim, "p": wl.p, "batch": B,
                       "amplitudes_per_gpu": local_n,
                       "l2": l2_label,
                       "parallelism": (f"state sharded over {world} GPUs" if world > 1 else
                                       (f"1 GPU, {vshards} virtual shards" if vshards > 1 else "1 GPU"))},
            "achieved_hbm_gbs_step": achieved_step_gbs,
            "objective": f if batch is None else float(np.asarray(f)[0]),
            "roofline": roof, "sharded_roofline": sharded, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    plan.destroy()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
