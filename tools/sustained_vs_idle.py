"""Per-pass device times of a cfg4 evaluation run (a) right after an idle period and (b) inside a
sustained sequence of evaluations, with the SM clock and power sampled by NVML during each: tells
whether the sustained-bench slowdown of the compute-heavier passes is a clock (power-cap) effect.
Usage: QVA_TRACE=1 python tools/sustained_vs_idle.py   (per-pass times come from the [qva] trace)"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
import paper_2110_03963_b200 as Q
from qva_inputs import make_config

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.005)


def window(t0, t1):
    s = [x for x in samples if t0 <= x[0] <= t1]
    if not s:
        return "no samples"
    clk = sorted(x[1] for x in s); pw = sorted(x[2] for x in s)
    return f"sm clock median {clk[len(clk) // 2]} MHz (min {clk[0]}), power median {pw[len(pw) // 2]:.0f} W (max {pw[-1]:.0f})"


wl = make_config("cfg4")
th = threading.Thread(target=sampler, daemon=True); th.start()
with Q.Plan(wl.dim, "x", n_qubits=wl.n_qubits) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    for _ in range(3):
        P.evolve(wl.theta)
    P.set_profiling(True)
    for label, pre_sleep, reps in (("after 3 s idle", 3.0, 1), ("sustained (10th of 10)", 0.0, 10),
                                   ("after 3 s idle", 3.0, 1)):
        time.sleep(pre_sleep)
        for r in range(reps):
            sys.stderr.write(f"--- {label} rep {r}\n"); sys.stderr.flush()
            t0 = time.time()
            P.reset_kernel_stats()
            P.evolve(wl.theta)
            t1 = time.time()
        st = P.kernel_stats("tile")
        print(f"{label}: tile passes {st['ms']:.3f} ms / {st['launches']} launches; {window(t0, t1)}", flush=True)
stop.set()
