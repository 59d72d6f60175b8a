"""Summarise bench.py JSON lines (stdin) in one line each (tuning runs)."""
import json
import sys

for ln in sys.stdin:
    try:
        d = json.loads(ln)
    except Exception:
        print(ln.strip()[:300])
        continue
    r, c = d["roofline"], d.get("detail") or d["config"]
    print(f"{d['config']['workload']} value={d['value']:.1f} GNs/s ms/tstep={c['ms_per_time_step']:.3f} "
          f"sweeps/tstep={c['sweeps_per_time_step_mean']:.1f} F={r['sweeps_per_launch']} "
          f"launch_us={r['avg_launch_us']:.1f} GB/s={r['achieved']:.0f} frac={r['frac']:.3f} "
          f"kern_GNs={r['kernel_node_sweeps_per_s']:.1f} share={r['sweep_share_of_step']:.3f} "
          f"clk={d['clocks'].get('sm_mhz')}")
