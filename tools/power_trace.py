"""Sweep-launch time against the SM clock and board power under sustained load.

    python tools/power_trace.py [--workload 4] [--seconds 12] [--sweeps 40]

Runs the bench's workload (BASELINE.json config, bench.py's omega) as a
sequence of pg_transient_continue calls of ONE time step with a fixed number of
sweeps each (tol = 0: every call is sweeps/2 full two-sweep launches of
k_rb_sweep2 plus the step's RHS), each bracketed by CUDA events, from an idle
GPU, while nvidia-smi samples the SM clock and the board power every 20 ms.
Prints per-call device time as us per launch, the implied algorithmic
bandwidth (56 B per node per launch) and its fraction of the
measured HBM peak, binned by the SM clock seen during the call, plus the
first and last seconds of the run: the evidence for DESIGN.md §7's reading
that the board's power limit, not HBM, sets the bench's fraction on the large
grids.  Diagnostic only (no bench number).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import gridgen  # noqa: E402


class Sampler:
    """nvidia-smi SM clock and board power every 20 ms, host-timestamped."""

    def __init__(self):
        self.samples = []
        self.proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                                      "--format=csv,noheader,nounits", "-lms", "20"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        for ln in self.proc.stdout:
            try:
                s, p = (float(x) for x in ln.split(","))
            except ValueError:
                continue
            self.samples.append((time.time(), s, p))

    def stop(self):
        self.proc.terminate()


def report(rows, peak, seconds, label):
    """rows: (t_start, SM MHz, power W, us, GB/s)"""
    print(f"{'SM MHz bin':>12} {'calls':>6} {'power W':>8} {label:>10} {'GB/s':>7} {'frac':>6}")
    bins = {}
    for _, mhz, pw, us, gbs in rows:
        bins.setdefault(int(mhz // 50) * 50, []).append((pw, us, gbs))
    for b in sorted(bins):
        v = bins[b]
        gbs = statistics.median(x[2] for x in v)
        print(f"{b:>7}-{b + 49:<4} {len(v):>6} {statistics.median(x[0] for x in v):>8.0f} "
              f"{statistics.median(x[1] for x in v):>10.1f} {gbs:>7.0f} {gbs / peak:>6.3f}")
    if not rows:
        return
    t_first = rows[0][0]
    for lo, hi in ((0.0, 1.0), (seconds - 2.0, seconds)):
        v = [r for r in rows if lo <= r[0] - t_first < hi]
        if v:
            gbs = statistics.median(r[4] for r in v)
            print(f"seconds {lo:4.1f}-{hi:4.1f}: SM {statistics.median(r[1] for r in v):.0f} MHz, "
                  f"{statistics.median(r[2] for r in v):.0f} W, {statistics.median(r[3] for r in v):.1f} "
                  f"{label}, {gbs:.0f} GB/s = {gbs / peak:.3f} of {peak:.0f}")
    mhz = np.array([r[1] for r in rows])
    gb = np.array([r[4] for r in rows])
    if mhz.std() > 0 and gb.std() > 0:
        print(f"correlation(SM clock, GB/s) = {np.corrcoef(mhz, gb)[0, 1]:.3f}")


def rows_of(calls, samples, nbytes):
    rows = []
    for t0, t1, us in calls:
        s = [x for x in samples if t0 - 0.01 <= x[0] <= t1 + 0.01]
        if s:
            rows.append((t0, statistics.median(x[1] for x in s), statistics.median(x[2] for x in s), us,
                         nbytes / (us * 1e-6) / 1e9))
    return rows


def copy_trace(a):
    import torch
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.4)
    n = 1 << 30
    x = torch.empty(n, dtype=torch.float64, device="cuda").fill_(1.0)
    y = torch.empty_like(x)
    sm = Sampler()
    time.sleep(1.0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    calls = []
    t_end = time.time() + a.seconds
    while time.time() < t_end:
        t0 = time.time()
        ev0.record()
        for _ in range(4):
            y.copy_(x)
        ev1.record()
        ev1.synchronize()
        calls.append((t0, time.time(), ev0.elapsed_time(ev1) * 1e3 / 4))
    time.sleep(0.3)
    sm.stop()
    print(f"device copy of {n} fp64 elements ({2 * 8 * n / 1e9:.1f} GB read + write per copy), {len(calls)} calls "
          f"of 4 copies, {len(sm.samples)} clock samples; idle power {sm.samples[0][2]:.0f} W")
    report(rows_of(calls, sm.samples, 16.0 * n), peak, a.seconds, "us/copy")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=4)
    ap.add_argument("--seconds", type=float, default=12.0)
    ap.add_argument("--sweeps", type=int, default=40)
    ap.add_argument("--copy", action="store_true",
                    help="instead: a sustained device copy (torch b.copy_(a) of 1 Gi fp64 elements, "
                         "the MEASURED_PEAKS.json kind of kernel) under the same sampling")
    ap.add_argument("--duty", type=float, default=0.0,
                    help="idle seconds after every call (bursts: the board power stays low, so the "
                         "SM clock stays high); with --duty, calls alternate between --sweeps and "
                         "3 x --sweeps and the launch time is the difference (no per-call overhead)")
    ap.add_argument("--opt", action="append", default=[], help="library option key=value (pg_set_option)")
    a = ap.parse_args()
    if a.copy:
        return copy_trace(a)
    import torch
    import bench
    import paper_1409_7166_b200 as P
    from paper_1409_7166_b200 import build
    build.build()
    g = gridgen.config_grid(a.workload)
    omega = bench.OMEGA.get(a.workload, bench.FALLBACK_OMEGA)
    G = P.Grid.from_mesh_grid(g, device=True)
    for kv in a.opt:
        k, v = kv.split("=", 1)
        G.set_option(k, int(v))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6550.4)
    nbytes = 56.0 * g.n
    launches = a.sweeps // 2

    sm = Sampler()
    time.sleep(1.0)                     # idle baseline

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    calls = []                          # (t_start, t_end, us per launch)
    G.transient(g.h, 1, tol=0.0, omega=omega, max_sweeps=a.sweeps, raise_on_noconv=False)
    t_end = time.time() + a.seconds
    step = 1
    def call(sweeps):
        nonlocal step
        if step >= g.steps:
            G.transient(g.h, 1, tol=0.0, omega=omega, max_sweeps=sweeps, raise_on_noconv=False)
            step = 1
        t0 = time.time()
        ev0.record()
        G.transient(g.h, 1, tol=0.0, omega=omega, max_sweeps=sweeps, cont=True, raise_on_noconv=False)
        ev1.record()
        ev1.synchronize()
        step += 1
        return t0, time.time(), ev0.elapsed_time(ev1) * 1e3

    while time.time() < t_end:
        if a.duty > 0:
            t0, _, us1 = call(a.sweeps)
            _, t1, us3 = call(3 * a.sweeps)
            calls.append((t0, t1, (us3 - us1) / (2 * launches)))
            time.sleep(a.duty)
        else:
            t0, t1, us = call(a.sweeps)
            calls.append((t0, t1, us / launches))
    time.sleep(0.3)
    sm.stop()
    G.close()
    print(f"config{a.workload}: {g.n} nodes, {launches} launches of 2 sweeps per call, {len(calls)} calls, "
          f"{len(sm.samples)} clock samples; idle power {sm.samples[0][2]:.0f} W")
    report(rows_of(calls, sm.samples, nbytes), peak, a.seconds, "us/launch")


if __name__ == "__main__":
    main()
