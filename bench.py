"""Benchmark: topology-based power-grid transient (arxiv 1409.7166) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload C] [--tsteps T] [--omega w] [--method rbsor|jacobi]
                    [--scaling strong|weak] [--transport auto|nccl|p2p] [--opt key=value ...]

Workload: BASELINE.json config C (default 4: the 8 x 4096 x 4096 RC mesh,
134M nodes, h = 5 ps, 200 steps -- the largest single-GPU configuration,
DESIGN.md §11).  One bench "step" = one window of T consecutive
backward-Euler time steps of that transient (default T = 8 for config 4, the
whole transient for the smaller configs): per time step the fused RHS
kernel, red-black SOR sweeps (F = 2 per launch) to tol = 1e-10 V, and (RLC)
the inductor update, through pg_transient / pg_transient_continue.  Windows
continue the transient (pg_transient_continue) and restart it from x(0) when
it is complete, so W + K windows of T = 8 cover the 200 steps of config 4
exactly once for the driver's --warmup 5 --steps 20.  N > 1 (torchrun, one
rank per GPU): the mesh is split into row slabs, one per GPU, advanced by
pg_group_transient with an exchange after every sweep launch (NCCL halo
send/recv + norm allreduce, or the peer-memory exchange fused into the
sweep); strong scaling by default (the config split), weak stacks N copies.
Inputs are seeded synthetic grids with the BASELINE.json distributions
(DESIGN.md §6), resident in HBM before the timed region (the per-pass working
set, 56 B per node, exceeds the 126 MB L2 on configs 1-4: no flush needed).

Metric: node-sweeps per second (GNode-sweeps/s), whole job; ms per time step
in `detail`.  `roofline` is for the dominant kernel (k_rb_sweep2, the
two-sweep pipeline; k_csr_sweep on CSR grids; k_rb_cluster on meshes small
enough for one cluster): algorithmic bytes per launch (56 B per node: V read +
write, gx, gy, gz, b, 1/d, once per launch of F sweeps) / its CUDA-event
duration inside the timed region (an event pair per time step around the
sweep launches on the grid's stream; graphs and PDL stay on).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "node-updates/sec (GNode-sweeps/s) and ms per time step; fraction of HBM roofline"
UNIT = "GNode-sweeps/s"
BYTES_PER_NODE_PASS = 56  # V r/w 16 + gx, gy, gz 24 + b 8 + invd 8 (one streaming pass, F sweeps)
DEFAULT_WORKLOAD = 4
# omega of each config (R15): Young's optimum omega_b from
# pg_estimate_omega (Rayleigh-quotient estimate of the Jacobi spectral radius:
# config 1 1.96616, 2 1.95824, 3 1.95105, 4 1.97417) and, following Young's
# advice to overestimate omega_b rather than underestimate it, the argmin of the
# mean sweeps per time step over a grid of omega >= omega_b on the config's first
# time steps (tools/omega_scan.py, profiles/r2_omega_scan.log); the same literals
# parametrise the full-size parity goldens (tools/make_golden_fullsize.py)
OMEGA = {
    1: 1.969,
    2: 1.962,
    3: 1.957,
    4: 1.975,
}
FALLBACK_OMEGA = 1.9
DEFAULT_WINDOW = {4: 8}   # time steps per bench step (others: the whole transient)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", type=int, default=DEFAULT_WORKLOAD, help="BASELINE.json config index")
    ap.add_argument("--tsteps", type=int, default=None, help="time steps per bench step (window)")
    ap.add_argument("--omega", type=float, default=None)
    ap.add_argument("--estimate-omega", action="store_true",
                    help="estimate Young's omega on the grid at run time instead of the recorded value")
    ap.add_argument("--tune-omega", action="store_true",
                    help="tune omega on the grid at run time (pg_tune_omega: omega_b and 7 candidates "
                         "4e-4 apart, first 8 time steps) instead of the recorded value")
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--method", default="rbsor", choices=["rbsor", "jacobi"])
    ap.add_argument("--slabs", type=int, default=1,
                    help="N = 1 only: split the mesh into this many row slabs advanced by the "
                         "single-process group (pg_group_local): the multi-GPU protocol's "
                         "exchange cost measured on one GPU")
    ap.add_argument("--transport", default=None, choices=["auto", "nccl", "copy", "p2p"],
                    help="slab exchange: auto (N > 1 default: p2p, checked once against nccl on the "
                         "first window, nccl if they differ), nccl, copy (--slabs default), or p2p: "
                         "fused into the sweep kernel over peer memory (CUDA IPC for N > 1)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N > 1: strong = the config split over the GPUs (default), weak = config rows x N")
    ap.add_argument("--opt", action="append", default=[],
                    help="library option key=value (pg_set_option), e.g. fuse=2, lag=3")
    ap.add_argument("--ref-seconds", type=float, default=None,
                    help="--impl reference: oracle seconds per bench step (default: ~90 s in total)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
                power.append(float(parts[2]))
            except ValueError:
                continue
            smax = m
            sm.append(s)
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(power) if power else None}


# ------------------------------------------------------------ workloads
def make_grid(cfg: int, world: int = 1, scaling: str = "strong"):
    """BASELINE config `cfg`; for N > 1 ranks under weak scaling the mesh is N
    copies of the config's row count stacked (same per-GPU work), under strong
    scaling the config itself is split."""
    import gridgen
    if world > 1 and scaling == "weak":
        L, NY, NX = gridgen.CONFIGS[cfg]["dims"]
        return gridgen.config_grid(cfg, dims=(L, NY * world, NX))
    return gridgen.config_grid(cfg)


def window_of(cfg: int, g, tsteps):
    return int(tsteps or DEFAULT_WINDOW.get(cfg, g.steps))


def omega_of(args, cfg):
    if args.omega:
        return args.omega, "--omega"
    if args.method == "jacobi":
        return FALLBACK_OMEGA, "fixed (Jacobi weight)"
    if args.tune_omega:
        return None, "tuned at run time (pg_tune_omega: omega_b + k 4e-4, k < 8, first 8 time steps)"
    if cfg in OMEGA and not args.estimate_omega:
        return OMEGA[cfg], ("recorded: argmin of sweeps per time step over omega >= Young's omega_b "
                            "(pg_estimate_omega, Rayleigh quotient of 8000 Jacobi sweeps) on this grid "
                            "(DESIGN.md R15)")
    return None, "Young's omega_b (pg_estimate_omega, 8000 Jacobi sweeps, at run time)"


def config_dict(cfg, g, T, tol, omega, omega_src, method, opts, world, scaling, transport, slabs):
    """The workload description both arms print (identical for the same args)."""
    if world > 1:
        par = (f"slab{world}: rows split over {world} GPUs ({scaling} scaling), "
               + {"p2p": "ghost rows and norm exchanged by the sweep kernel over peer memory (CUDA IPC)",
                  "auto": ("ghost rows and norm exchanged by the sweep kernel over peer memory (CUDA IPC), "
                           "checked bit for bit against the NCCL transport on the first window "
                           "(NCCL if they differ; detail.transport says which ran)")}.get(
                   transport, "NCCL ghost-row exchange + norm allreduce per sweep launch"))
    elif slabs > 1:
        par = (f"1 GPU, {slabs} row slabs exchanged in one process ("
               + ("pg_group_local_p2p: peer-memory exchange in the sweep kernel" if transport == "p2p"
                  else "pg_group_local: copies") + ")")
    else:
        par = "1 GPU"
    return {"workload": f"config{cfg}" + (f" x{world} rows (weak scaling)" if world > 1 and scaling == "weak"
                                          else ""),
            "nodes": g.n, "mesh": [g.layers, g.ny, g.nx] if hasattr(g, "gx") else None,
            "grid": "CSR (irregular)" if not hasattr(g, "gx") else ("RLC mesh" if g.is_rlc else "RC mesh"),
            "h_s": g.h, "time_steps_total": g.steps, "time_steps_per_bench_step": T,
            "bench_step": ("window of T consecutive time steps continuing the transient "
                           "(pg_transient_continue), restarted from x(0) after its last step"),
            "tol_V": tol, "omega": omega, "omega_source": omega_src, "method": method, "options": opts,
            "l2": "per-sweep working set ~56 B/node x n > 126 MB L2 (no flush needed)",
            "parallelism": par}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str, cfg: int):
    """DRAM bytes per launch of the sweep kernel from the committed `ncu --set
    full` capture of the same configuration (profiles/rb_sweep_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "rb_sweep_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"{kernel}@config{cfg}")
        if not isinstance(e, dict):
            return None
        return e.get("dram_bytes_per_launch") * e.get("colour_launches_per_sweep", 1)
    except Exception:
        return None


# ------------------------------------------------------------- oracle arm
class OracleSampler:
    """The oracle (as it stands, plain C, one thread) on the full grid of the
    workload: time step 1 from x(0), a fixed number of natural-order SOR sweeps."""

    def __init__(self, cfg, g, omega):
        from oracle import netlist, nodal, pwl
        self.cfg, self.n = cfg, g.n
        self.h, self.omega = g.h, omega
        nl = netlist.from_grid(g)
        self.o = nodal.NodalOracle(nl)
        nl.ra = nl.rb = nl.rg = None     # the branch list is not needed any more (memory)
        self.It = pwl.node_currents_table(nl, g.h, 1)
        self.t_one = self._time(1)              # call overhead + 1 sweep

    def _time(self, k):
        t0 = time.perf_counter()
        self.o.transient(self.h, 1, tol=0.0, omega=self.omega, Itab=self.It, max_sweeps=k)
        return time.perf_counter() - t0

    def per_sweep(self):
        """Seconds per sweep: grow the sweep count until a call takes >= 0.3 s
        (small grids), the difference to the 1-sweep call removes the overhead."""
        k = 3
        while True:
            t = self._time(k)
            if t >= 0.3 or k >= 1 << 22:
                return max((t - self.t_one) / (k - 1), 1e-9)
            k *= 4

    def run(self, k):
        t0 = time.perf_counter()
        self.o.transient(self.h, 1, tol=0.0, omega=self.omega, Itab=self.It, max_sweeps=k)
        dt = time.perf_counter() - t0
        return {"value": self.n * k / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"config{self.cfg} full grid ({self.n} nodes), time step 1 from x(0), {k} fixed "
                          f"natural-order SOR sweeps (omega={self.omega}) in the plain-C oracle "
                          f"(oracle/nodal.c), single thread, {dt:.1f} s"}, dt


def oracle_sample(cfg: int, g=None, seconds: float = 12.0, omega: float = 1.98):
    if g is None:
        g = make_grid(cfg)
    s = OracleSampler(cfg, g, omega)
    per = s.per_sweep()
    k = max(2, int(seconds / per))
    return s.run(k)[0]


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.workload
    g = make_grid(cfg)
    T = window_of(cfg, g, args.tsteps)
    omega, omega_src = omega_of(args, cfg)
    if omega is None:
        omega, omega_src = FALLBACK_OMEGA, "fixed (reference arm: no GPU to estimate it)"
    transport = args.transport or ("nccl" if world > 1 else "copy")
    conf = config_dict(cfg, g, T, args.tol, omega, omega_src, args.method, dict(kv.split("=", 1) for kv in args.opt),
                       world, args.scaling, transport, args.slabs)
    s = OracleSampler(cfg, g, omega)
    per = s.per_sweep()
    budget = args.ref_seconds or max(2.0, 90.0 / max(1, args.steps + args.warmup))
    k = max(1, int(budget / per))
    for _ in range(args.warmup):
        s.run(max(1, min(k, int(5.0 / per))))
    vals, t_all = [], 0.0
    for _ in range(args.steps):
        r, dt = s.run(k)
        t_all += dt
        vals.append(r["value"])
    v = float(args.steps) * g.n * k / t_all / 1e9 if t_all > 0 else 0.0
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_all / max(args.steps, 1), "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded BASELINE.json recipe, gridgen)",
            "config": conf,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"each bench step: {r['sample']}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- b200 arm
def verify_p2p(P, g, rank, world, make_group, T, tol, omega):
    """First window (T time steps from x(0)) with the NCCL transport and with
    the peer-memory exchange fused into the sweep: owned voltages and per-step
    sweep counts must be identical on every rank.  Returns (ok, reason), the
    same on every rank."""
    import numpy as np
    import torch
    import torch.distributed as dist
    res, why = {}, ""
    for p2p in (False, True):
        try:
            grp = make_group(p2p=p2p)
            try:
                r = grp.transient(g.h, T, tol=tol, omega=omega, max_sweeps=200000)
                V = np.concatenate([v.reshape(-1) for _, v in grp.owned_voltages(g)])
                res[p2p] = (V, np.asarray(r.sweeps).copy())
            finally:
                grp.close()
        except Exception as e:  # noqa: BLE001 -- any failure selects NCCL
            why = f"{'p2p' if p2p else 'nccl'} raised {type(e).__name__}: {e}"[:200]
            break
    ok = len(res) == 2 and all(np.array_equal(a, b) for a, b in zip(res[False], res[True]))
    if len(res) == 2 and not ok:
        why = "owned voltages or sweep counts differ from the nccl transport"
    flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                        device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0 and ok:
        why = "another rank's check failed"
    return bool(flag.item()), why


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1409_7166_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.workload
    g = make_grid(cfg, world, args.scaling)
    T = window_of(cfg, g, args.tsteps)
    TOT = g.steps
    tol = args.tol
    stream = torch.cuda.current_stream()
    opts = dict(kv.split("=", 1) for kv in args.opt)
    fuse = int(opts.get("fuse", 2))
    transport = args.transport or ("auto" if world > 1 else "copy")
    iopts = {k: int(v) for k, v in opts.items()}
    tr = {"p2p": transport in ("p2p", "auto"), "note": None}

    def make_group(device=True, p2p=None):
        # slab partition over the ranks, exchange after every sweep launch
        # inside the library (pg_group_transient): NCCL halo send/recv + norm
        # allreduce, or the peer-memory exchange fused into the sweep kernel
        if tr["p2p"] if p2p is None else p2p:
            return P.SlabGroup.p2p(g, rank, world, fuse=fuse, stream=stream, device=device, options=iopts)
        return P.SlabGroup.nccl(g, rank, world, fuse=fuse, stream=stream, device=device)

    if world > 1:
        grp = make_group(p2p=False if transport == "auto" else None)
        G = grp.grids[0]
        sp = grp.specs[0]
        my_nodes = g.layers * (sp.y1 - sp.y0) * g.nx
    elif args.slabs > 1:
        grp = P.SlabGroup.local(g, args.slabs, fuse=fuse, stream=stream,
                                transport="p2p" if tr["p2p"] else "copy", options=iopts if tr["p2p"] else None)
        G = grp.grids[0]
        my_nodes = g.n
    else:
        grp = None
        mk = P.Grid.from_mesh_grid if hasattr(g, "gx") else P.Grid.from_edge_grid
        G = mk(g, device=True)
        G.set_stream(stream)
        my_nodes = g.n
    for k, v in opts.items():
        for q in (grp.grids if grp is not None else [G]):
            q.set_option(k, int(v))
    t_om = time.perf_counter()
    omega, omega_src = omega_of(args, cfg)
    if omega is None and args.tune_omega and grp is None:
        omega, _ = G.tune_omega(g.h, steps=8, tol=tol, n=8, d_omega=4e-4)
    elif omega is None:
        _, omega = G.estimate_omega(g.h, 8000)
    if world > 1:
        t = torch.tensor([omega], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        omega = float(t.item())
    t_om = time.perf_counter() - t_om
    if world > 1 and transport == "auto":
        # the fused peer-memory exchange is the product path; before it is
        # timed, its first window is compared bit for bit with the NCCL
        # transport's (both equal the single grid, tests/test_gpu_slab.py,
        # test_gpu_p2p.py) and every rank falls back to NCCL unless all agree
        grp.close()
        ok, why = verify_p2p(P, g, rank, world, make_group, T, tol, omega)
        tr["p2p"] = ok
        tr["note"] = "p2p (equal to nccl on the first window)" if ok else f"nccl (p2p check failed: {why})"
        grp = make_group()
        G = grp.grids[0]
        for k, v in opts.items():
            G.set_option(k, int(v))
    elif world > 1:
        tr["note"] = transport

    state = {"done": 0}

    def window():
        """The next window of T time steps (continuing the transient, or
        restarting it from x(0) when the remaining steps do not fill a window)."""
        cont = 0 < state["done"] and state["done"] + T <= TOT
        if not cont:
            state["done"] = 0
        s0 = state["done"]
        if grp is not None:
            r = grp.transient(g.h, T, tol=tol, omega=omega, max_sweeps=200000, cont=cont)
        else:
            r = G.transient(g.h, T, tol=tol, omega=omega, method=args.method, max_sweeps=200000, cont=cont)
        state["done"] = s0 + T
        return r, s0

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def set_timing(on):
        for q in (grp.grids if grp is not None else [G]):
            q.set_option("timing", 1 if on else 0)

    # the production configuration (CUDA-graph batches, programmatic dependent
    # launch of consecutive sweeps) with option "timing": an event pair on
    # `stream` around every time step's sweep launches (read after the run, no
    # extra synchronisation) gives the sweep kernel's time inside the timed region
    set_timing(True)
    win_ms = {}          # first time step of the window -> device ms (first pass over the transient)

    def timed_window():
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r, s0 = window()
        e1.record(stream)
        e1.synchronize()
        win_ms.setdefault(s0, e0.elapsed_time(e1))
        return r

    for _ in range(args.warmup):
        timed_window()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    sweeps = launches = 0
    sweep_ms = 0.0
    sweep_launches = 0
    sweeps_per_tstep = []
    for _ in range(args.steps):
        r = timed_window()
        sweeps += int(r.stats.sweeps_total)
        launches += int(r.stats.kernel_launches)
        sweep_ms += float(r.stats.sweep_ms)
        sweep_launches += int(r.stats.sweep_launches)
        sweeps_per_tstep.append(r.sweeps[1:])
    ev1.record(stream)
    barrier()
    ck = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t1 = ms
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    node_sweeps = float(my_nodes) * sweeps
    tot = torch.tensor([node_sweeps], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tot)
    value = float(tot.item()) / (ms_max * 1e-3) / 1e9

    # roofline of the sweep kernel: one launch = one streaming pass over the
    # grid performing F sweeps; algorithmic bytes per launch = 56 B x n
    peak, peak_src = peaks()
    avg_launch_ms = sweep_ms / max(sweep_launches, 1)
    F = int(r.stats.sweeps_per_launch)
    if hasattr(g, "gx"):
        grids = grp.grids if grp is not None else [G]   # local group: one launch = all slabs
        launch_nodes = sum(q.info()["layers"] * q.info()["ny"] * q.info()["nx"] for q in grids)
        bytes_per_launch = BYTES_PER_NODE_PASS * launch_nodes
        kname = "k_rb_sweep2" if F == 2 and int(opts.get("pipe", 1)) else "k_rb_sweep_fused"
        if grp is None and sweep_launches == args.steps * T and sweeps > sweep_launches:
            # cluster-resident sweep (small meshes): one launch runs all sweeps of a
            # time step with V and the constants in shared memory, HBM once per step
            kname = "k_rb_cluster"
            F = sweeps / max(sweep_launches, 1)
        bpn = f"{BYTES_PER_NODE_PASS} B per node per launch of {F} sweeps"
    else:
        # CSR sweep (one launch per colour per sweep): rowptr 4 + b 8 + 1/d 8 +
        # V read + write 16 per row, column index 4 + value 8 per entry
        # (gathered neighbour values counted as cache hits)
        launch_nodes = g.n
        nnz = 2 * int(np.count_nonzero(np.asarray(g.eu) != np.asarray(g.ev)))
        bytes_per_launch = 36 * g.n + 12 * nnz
        kname = "k_csr_sweep"
        bpn = "36 B per row + 12 B per off-diagonal entry per sweep"
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    traffic = ncu_traffic(kname, cfg) if grp is None else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": kname, "bytes_per_launch": bytes_per_launch, "algorithmic_bytes": bpn,
            "bytes_per_node_per_launch": bytes_per_launch / launch_nodes, "sweeps_per_launch": F,
            "bytes_per_node_sweep": bytes_per_launch / launch_nodes / F, "avg_launch_us": avg_launch_ms * 1e3,
            "kernel_node_sweeps_per_s": launch_nodes * F / (avg_launch_ms * 1e-3) / 1e9,
            "sweep_share_of_step": sweep_ms / t1 if t1 > 0 else None, "peak_source": peak_src,
            "traffic_source": ("ncu --set full of this kernel on this config, dram__bytes_read.sum + "
                               "dram__bytes_write.sum per launch (profiles/rb_sweep_traffic.json)")
            if traffic else None,
            "timing": "avg_launch_us = sum over time steps of the CUDA-event time around the step's "
                      "sweep launches (graph batches, programmatic dependent launch; includes the batch "
                      "bookkeeping kernel and queued launches that exit after convergence) / launches "
                      "that did work, inside the timed region"}
    if kname == "k_rb_cluster":
        roof["note"] = ("cluster-resident kernel: all sweeps of a time step in one launch with V and the "
                        "node constants in distributed shared memory; HBM is read once per time step, the "
                        "sweep rate is bound by cluster-barrier latency, not by HBM (DESIGN.md section 7)")

    # e2e: the public C-ABI calls a user makes, with HOST buffers (pinned): the
    # grid built from host arrays (H2D inside pg_create_*), the loads set, one
    # window of T steps from x(0), the voltages read back (D2H) -- every rep
    e2e = None
    nrep = max(1, min(args.steps, 2))
    if not args.no_e2e and grp is not None and world > 1:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        h2d = d2h = 0

        def e2e_rep():
            nonlocal h2d, d2h
            H = make_group(device=False)
            if not tr["p2p"]:
                for k, v in opts.items():
                    H.grids[0].set_option(k, int(v))
            rr = H.transient(g.h, T, tol=tol, omega=omega, max_sweeps=200000)
            H.owned_voltages(g)
            sm = H.specs[0]
            h2d = 8 * g.layers * (sm.hi - sm.lo) * g.nx * 4
            d2h = 8 * g.layers * (sm.hi - sm.lo) * g.nx
            H.close()
            return int(rr.stats.sweeps_total)

        if args.warmup > 0:
            e2e_rep()      # untimed: the first group maps its pool memory and captures its graphs
        barrier()
        e0.record(stream)
        e_sweeps = 0
        for _ in range(nrep):
            e_sweeps += e2e_rep()
        e1.record(stream)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ns = torch.tensor([float(my_nodes) * e_sweeps], dtype=torch.float64, device="cuda")
        dist.all_reduce(ns)
        e2e = {"value": float(ns.item()) / (float(te.item()) * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()) / nrep, "per_rank_bytes": True,
               "step": f"slab grid from host arrays + exchange group + time steps 1..{T} + owned voltages "
                       f"read back (after one untimed rep)"}
    elif not args.no_e2e and args.slabs <= 1:
        pin = {}
        for name in ("gx", "gy", "gz", "cap", "lz", "eu", "ev", "eg"):
            a = getattr(g, name, None)
            if a is not None:
                pin[name] = torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        s = g.sources
        for name, a in (("pad_node", g.pad_node), ("pad_g", g.pad_g), ("pad_l", getattr(g, "pad_l", None)),
                        ("src_node", s.node), ("src_ptr", s.ptr), ("src_t", s.t), ("src_i", s.i)):
            if a is not None:
                pin[name] = torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        h2d = sum(v.nbytes for v in pin.values())
        out = torch.empty(g.n, dtype=torch.float64).pin_memory().numpy()
        d2h = out.nbytes

        def e2e_rep():
            if hasattr(g, "gx"):
                H = P.Grid.mesh(g.layers, g.ny, g.nx, pin["gx"], pin["gy"], pin["gz"], pin["cap"],
                                pin["pad_node"], pin["pad_g"], g.vdd, pin.get("lz"), pin.get("pad_l"))
            else:
                H = P.Grid.csr(g.n, pin["eu"], pin["ev"], pin["eg"], pin["cap"], pin["pad_node"], pin["pad_g"],
                               g.vdd)
            H.set_stream(stream)
            for k, v in opts.items():
                H.set_option(k, int(v))
            H.set_sources(pin["src_node"], pin["src_ptr"], pin["src_t"], pin["src_i"])
            rr = H.transient(g.h, T, tol=tol, omega=omega, method=args.method, max_sweeps=200000)
            H.voltages(out)
            H.close()
            return int(rr.stats.sweeps_total)

        if args.warmup > 0:
            e2e_rep()      # untimed: the first grid maps its pool memory, like the bench's warm-up steps
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e_sweeps = 0
        for _ in range(nrep):
            e_sweeps += e2e_rep()
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        e2e = {"value": float(g.n) * e_sweeps / (ems * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": ems / nrep,
               "step": (f"pg_create_{'mesh' if hasattr(g, 'gx') else 'csr'} + pg_set_sources from pinned host "
                        f"arrays, pg_transient over time steps 1..{T} from x(0), pg_get_voltages into pinned "
                        f"host memory, pg_destroy (after one untimed rep)")}

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = oracle_sample(cfg, g, seconds=12.0, omega=omega)
        except Exception as e:  # never let the baseline kill the line
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    spt = np.concatenate(sweeps_per_tstep) if sweeps_per_tstep else np.zeros(1)
    full = None
    starts = list(range(0, TOT - T + 1, T))
    if TOT % T == 0 and all(s in win_ms for s in starts):
        full = sum(win_ms[s] for s in starts) / TOT
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE.json recipe, gridgen)",
            "config": config_dict(cfg, g, T, tol, omega, omega_src, args.method, opts, world, args.scaling,
                                  transport, args.slabs),
            "detail": {"ms_per_time_step": ms_max / args.steps / T,
                       "full_transient_ms_per_time_step": full,
                       "full_transient_note": (f"all {TOT} time steps, sum of the CUDA-event times of the "
                                               f"{len(starts)} windows of the first pass (warm-up windows "
                                               f"included) / {TOT}") if full is not None else None,
                       "sweeps_per_time_step_mean": float(spt.mean()),
                       "sweeps_per_time_step_max": int(spt.max()),
                       "omega_time_s": round(t_om, 3),
                       "transport": tr["note"]},
            "clocks": ck, "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if grp is not None:
        grp.close()   # the group owns its slab grids (releases the exchange first)
    else:
        G.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
