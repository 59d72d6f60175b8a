"""Benchmark: topology-based power-grid transient (arxiv 1409.7166) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload K] [--tsteps T] [--omega w] [--method rbsor|jacobi]
                    [--scaling weak|strong] [--opt key=value ...]

One bench "step" = one full pass of the hot path over the workload: a
pg_transient call (Algorithm 1: per backward-Euler time step the fused RHS
kernels, red-black SOR sweeps (F = 2 per launch) to tol = 1e-10 V, inductor
update) over T time steps of the BASELINE.json configuration (N = 1: config 1,
4 x 1024 x 1024 RC mesh, h = 5 ps, 500 steps).  N > 1 (torchrun, one rank per
GPU): the mesh is split into row slabs, one per GPU, advanced by
pg_group_transient with an NCCL ghost-row exchange and norm allreduce after
every sweep launch; weak scaling stacks N copies of the config's rows.
Inputs are seeded synthetic grids with the BASELINE.json distributions
(DESIGN.md §6), resident in HBM before the timed region (the ~235 MB per-pass
working set exceeds the 126 MB L2).

Metric: node-sweeps per second (GNode-sweeps/s), whole job; ms per time step
is reported in `config`.  `roofline` is for the dominant kernel
(k_rb_sweep2, the two-sweep pipeline; k_csr_sweep on CSR grids, k_rb_cluster
on meshes small enough for one cluster): algorithmic bytes per launch (56 B
per node: V read + write, gx, gy, gz, b, 1/d, once per launch of F sweeps) /
its CUDA-event duration inside the timed region (event pair per time step
around the sweep launches; graphs and PDL stay on).
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
DEFAULT_OMEGA = {0: 1.9, 1: 1.98, 2: 1.98, 3: 1.99, 4: 1.99}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", type=int, default=None, help="BASELINE.json config index")
    ap.add_argument("--tsteps", type=int, default=None, help="time steps per bench step")
    ap.add_argument("--omega", type=float, default=None)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--method", default="rbsor", choices=["rbsor", "jacobi"])
    ap.add_argument("--slabs", type=int, default=1,
                    help="N = 1 only: split the mesh into this many row slabs advanced by the "
                         "single-process group (pg_group_local): the multi-GPU protocol's "
                         "exchange cost measured on one GPU")
    ap.add_argument("--transport", default=None, choices=["nccl", "copy", "p2p"],
                    help="slab exchange: nccl (N > 1 default), copy (--slabs default), or p2p: "
                         "fused into the sweep kernel over peer memory (CUDA IPC for N > 1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = config rows x N (fixed work per GPU), strong = config split")
    ap.add_argument("--opt", action="append", default=[],
                    help="library option key=value (pg_set_option), e.g. fuse=2, lag=3, kernel=4")
    ap.add_argument("--ref-seconds", type=float, default=None,
                    help="--impl reference: oracle seconds per bench step (default: ~60 s in total)")
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
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            smax = m
            sm.append(s)
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ workloads
def make_grid(cfg: int, world: int = 1, scaling: str = "weak"):
    """BASELINE config `cfg`; for N > 1 ranks under weak scaling the mesh is N
    copies of the config's row count stacked (same per-GPU work), under strong
    scaling the config itself is split."""
    import gridgen
    if world > 1 and scaling == "weak":
        L, NY, NX = gridgen.CONFIGS[cfg]["dims"]
        return gridgen.config_grid(cfg, dims=(L, NY * world, NX))
    return gridgen.config_grid(cfg)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """dram bytes per launch of the sweep kernel from the committed ncu
    capture of the same configuration (profiles/rb_sweep_traffic.json), if any."""
    p = os.path.join(ROOT, "profiles", "rb_sweep_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(kernel) if isinstance(d.get(kernel), dict) else None
        return None if e is None else e.get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------- oracle arm
def oracle_sample(cfg: int, g=None, seconds: float = 12.0, omega: float = 1.98):
    """Time the oracle (as it stands) on a bounded sample of the workload:
    the full grid, time step 1, fixed natural-order SOR sweeps (single thread)."""
    import numpy as np
    from oracle import netlist, nodal, pwl
    if g is None:
        g = make_grid(cfg)
    nl = netlist.from_grid(g)
    o = nodal.NodalOracle(nl)
    It = pwl.node_currents_table(nl, g.h, 1)
    # calibrate sweeps to ~seconds of work: grow the sweep count until a run
    # takes >= 0.3 s (small grids), the difference to a 1-sweep run removes setup
    t0 = time.perf_counter()
    o.transient(g.h, 1, tol=0.0, omega=omega, Itab=It, max_sweeps=1)
    t_one = time.perf_counter() - t0
    kt = 4
    while True:
        t0 = time.perf_counter()
        o.transient(g.h, 1, tol=0.0, omega=omega, Itab=It, max_sweeps=kt)
        t_k = time.perf_counter() - t0
        if t_k >= 0.3 or kt >= 1 << 20:
            break
        kt *= 4
    per = max(t_k - t_one, 1e-9) / (kt - 1)
    k = max(2, int(seconds / per))
    t0 = time.perf_counter()
    o.transient(g.h, 1, tol=0.0, omega=omega, Itab=It, max_sweeps=k)
    dt = time.perf_counter() - t0
    return {"value": g.n * k / dt / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"config{cfg} full grid ({g.n} nodes), time step 1, {k} fixed natural-order "
                      f"SOR sweeps (omega={omega}) in the plain-C oracle, single thread, {dt:.1f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.workload if args.workload is not None else 1
    g = make_grid(cfg)
    omega = args.omega or DEFAULT_OMEGA.get(cfg, 1.9)   # fixed sweeps: omega only sets the arithmetic
    per_step = args.ref_seconds or max(2.0, 60.0 / max(1, args.steps + args.warmup))
    for _ in range(args.warmup):
        oracle_sample(cfg, g, seconds=min(per_step, 5.0), omega=omega)
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = oracle_sample(cfg, g, seconds=per_step, omega=omega)
        t_all += time.perf_counter() - t0
        vals.append(r["value"])
    v = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_all / max(args.steps, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded BASELINE.json recipe)",
            "config": {"workload": f"config{cfg}", "nodes": g.n},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- b200 arm
def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1409_7166_b200 as P

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.workload if args.workload is not None else 1
    g = make_grid(cfg, world, args.scaling)
    T = args.tsteps or g.steps
    tol = args.tol
    stream = torch.cuda.current_stream()
    opts = dict(kv.split("=", 1) for kv in args.opt)
    fuse = int(opts.get("fuse", 2))
    p2p = args.transport == "p2p"
    iopts = {k: int(v) for k, v in opts.items()}

    def make_group(device=True):
        # slab partition over the ranks, exchange after every sweep launch
        # inside the library (pg_group_transient): NCCL halo send/recv + norm
        # allreduce, or the peer-memory exchange fused into the sweep kernel
        if p2p:
            return P.SlabGroup.p2p(g, rank, world, fuse=fuse, stream=stream, device=device, options=iopts)
        return P.SlabGroup.nccl(g, rank, world, fuse=fuse, stream=stream, device=device)

    if world > 1:
        grp = make_group()
        G = grp.grids[0]
        sp = grp.specs[0]
        my_nodes = g.layers * (sp.y1 - sp.y0) * g.nx
    elif args.slabs > 1:
        grp = P.SlabGroup.local(g, args.slabs, fuse=fuse, stream=stream, transport="p2p" if p2p else "copy",
                                options=iopts if p2p else None)
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
    # relaxation factor: Young's optimum from the library's Jacobi power
    # iteration (§IV-D refers to Young), unless given; not timed
    t_om = time.perf_counter()
    if args.omega:
        omega, omega_src = args.omega, "--omega"
    elif args.method == "jacobi":
        omega, omega_src = DEFAULT_OMEGA.get(cfg, 1.9), "DEFAULT_OMEGA"
    else:
        _, omega = G.estimate_omega(g.h, 8000)
        if world > 1:
            t = torch.tensor([omega], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            omega = float(t.item())
        omega_src = "Young (pg_estimate_omega, 8000 Jacobi sweeps)"
    t_om = time.perf_counter() - t_om

    def solve():
        if grp is not None:
            return grp.transient(g.h, T, tol=tol, omega=omega, max_sweeps=200000)
        return G.transient(g.h, T, tol=tol, omega=omega, method=args.method, max_sweeps=200000)

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
    for _ in range(args.warmup):
        solve()
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
        r = solve()
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
    else:
        # CSR sweep (one launch per colour per sweep): rowptr 8 + b 8 + 1/d 8 +
        # V read + write 16 per row, column index 4 + value 8 per entry
        # (gathered neighbour values counted as cache hits)
        launch_nodes = g.n
        nnz = 2 * int(np.count_nonzero(np.asarray(g.eu) != np.asarray(g.ev)))
        bytes_per_launch = 40 * g.n + 12 * nnz
        kname = "k_csr_sweep"
    achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": ncu_traffic(kname) if hasattr(g, "gx") and cfg == 1 else None,
            "kernel": kname, "bytes_per_launch": bytes_per_launch,
            "bytes_per_node_per_launch": bytes_per_launch / launch_nodes, "sweeps_per_launch": F,
            "bytes_per_node_sweep": bytes_per_launch / launch_nodes / F, "avg_launch_us": avg_launch_ms * 1e3,
            "kernel_node_sweeps_per_s": launch_nodes * F / (avg_launch_ms * 1e-3) / 1e9,
            "sweep_share_of_step": sweep_ms / t1 if t1 > 0 else None, "peak_source": peak_src,
            "timing": "avg_launch_us = sum over time steps of the CUDA-event time around the step's "
                      "sweep launches (graph batches, programmatic dependent launch; includes the batch "
                      "bookkeeping kernel and queued launches that exit after convergence) / launches "
                      "that did work, inside the timed region"}
    if kname == "k_rb_cluster":
        roof["note"] = ("cluster-resident kernel: all sweeps of a time step in one launch with V and the "
                        "node constants in distributed shared memory; HBM is read once per time step, the "
                        "sweep rate is bound by cluster-barrier latency, not by HBM (DESIGN.md section 7)")

    # e2e: public C-ABI call with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and grp is not None:
        # public API with host buffers: this rank's slab built from host arrays,
        # NCCL group set up, transient, owned voltages read back
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        e_sweeps = 0
        nrep = max(1, min(args.steps, 2))
        h2d = d2h = 0
        for _ in range(nrep):
            H = make_group(device=False)
            if not p2p:
                for k, v in opts.items():
                    H.grids[0].set_option(k, int(v))
            rr = H.transient(g.h, T, tol=tol, omega=omega, max_sweeps=200000)
            Vo = H.owned_voltages(g)
            sm = H.specs[0]
            h2d = 8 * g.layers * (sm.hi - sm.lo) * g.nx * 4
            d2h = 8 * g.layers * (sm.hi - sm.lo) * g.nx
            H.close()
            e_sweeps += int(rr.stats.sweeps_total)
        e1.record(stream)
        barrier()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ns = torch.tensor([float(my_nodes) * e_sweeps], dtype=torch.float64, device="cuda")
        dist.all_reduce(ns)
        e2e = {"value": float(ns.item()) / (float(te.item()) * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()) / nrep, "per_rank_bytes": True}
    elif not args.no_e2e and args.slabs <= 1:
        pin = {}
        for name in ("gx", "gy", "gz", "cap", "lz"):
            a = getattr(g, name, None)
            if a is not None:
                pt = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                pin[name] = pt.numpy()
        h2d = sum(v.nbytes for v in pin.values()) + g.pad_node.nbytes + g.pad_g.nbytes
        s = g.sources
        h2d += s.node.nbytes + s.ptr.nbytes + s.t.nbytes + s.i.nbytes
        out = torch.empty(g.n, dtype=torch.float64).pin_memory().numpy()
        d2h = out.nbytes
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e_sweeps = 0
        for _ in range(max(1, min(args.steps, 2))):
            if hasattr(g, "gx"):
                H = P.Grid.mesh(g.layers, g.ny, g.nx, pin["gx"], pin["gy"], pin["gz"], pin["cap"],
                                g.pad_node, g.pad_g, g.vdd, pin.get("lz"), g.pad_l)
            else:
                H = P.Grid.from_edge_grid(g)
            H.set_stream(stream)
            for k, v in opts.items():
                H.set_option(k, int(v))
            H.set_sources(s.node, s.ptr, s.t, s.i)
            rr = H.transient(g.h, T, tol=tol, omega=omega, method=args.method, max_sweeps=200000)
            H.voltages(out)
            H.close()
            e_sweeps += int(rr.stats.sweeps_total)
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1)
        te = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nrep = max(1, min(args.steps, 2))
        e2e = {"value": float(g.n) * e_sweeps * world / (float(te.item()) * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()) / nrep}

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = oracle_sample(cfg, g, seconds=12.0, omega=omega)
        except Exception as e:  # never let the baseline kill the line
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    spt = np.concatenate(sweeps_per_tstep) if sweeps_per_tstep else np.zeros(1)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE.json recipe, gridgen)",
            "config": {"workload": f"config{cfg}" + (f" x{world} rows (weak scaling)" if world > 1 and
                                                     args.scaling == "weak" else ""), "nodes": g.n,
                       "mesh": [g.layers, g.ny, g.nx] if hasattr(g, "gx") else None,
                       "h_s": g.h, "time_steps_per_bench_step": T, "tol_V": tol, "omega": omega,
                       "omega_source": omega_src, "omega_estimate_s": round(t_om, 3),
                       "method": args.method, "options": opts, "ms_per_time_step": ms_max / args.steps / T,
                       "sweeps_per_time_step_mean": float(spt.mean()),
                       "sweeps_per_time_step_max": int(spt.max()),
                       "l2": "per-sweep working set ~56 B/node x n > 126 MB L2 (no flush needed)",
                       "parallelism": (f"slab{world}: rows split over {world} GPUs, "
                                       + ("ghost rows and norm exchanged by the sweep kernel over peer "
                                          "memory (CUDA IPC)" if p2p else
                                          "NCCL ghost-row exchange + norm allreduce per sweep launch"))
                       if world > 1
                       else (f"1 GPU, {args.slabs} row slabs exchanged in one process ("
                             + ("pg_group_local_p2p: peer-memory exchange in the sweep kernel"
                                if p2p else "pg_group_local: copies") + ")"
                             if args.slabs > 1 else "1 GPU")},
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
