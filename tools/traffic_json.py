"""Record the DRAM traffic of one sweep-kernel launch from an ncu --set full
capture into profiles/rb_sweep_traffic.json (read by bench.py for
roofline.traffic).  usage: python tools/traffic_json.py rep.ncu-rep key workload algorithmic_bytes"""
import csv, json, os, subprocess, sys

rep, key, workload, alg = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
d = dict(zip(rows[0], rows[2]))
f = lambda k: float(d[k])
rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
# ncu reports MB for these (units row)
units = dict(zip(rows[0], rows[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd *= scale.get(units["dram__bytes_read.sum"], 1)
wr *= scale.get(units["dram__bytes_write.sum"], 1)
stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): round(float(v), 3)
          for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
          and float(v) > 0.01}
e = {"kernel": d.get("Kernel Name", key), "workload": workload, "source": rep,
     "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
     "algorithmic_bytes_per_launch": alg, "traffic_over_algorithmic": (rd + wr) / alg,
     "duration_us_under_ncu": f("gpu__time_duration.sum") * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                                                           "second": 1e6}.get(units["gpu__time_duration.sum"], 1.0),
     "registers": f("launch__registers_per_thread"), "grid": d["launch__grid_size"], "block": d["launch__block_size"],
     "issue_active_pct": round(f("smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
     "dram_cycles_active_pct": round(f("dram__cycles_active.avg.pct_of_peak_sustained_elapsed"), 1),
     "fp64_pipe_pct": round(f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
     "instructions": f("smsp__inst_executed.sum"), "stalls_per_issued_instruction": stalls}
p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "rb_sweep_traffic.json")
j = json.load(open(p)) if os.path.exists(p) else {}
j[key] = e
json.dump(j, open(p, "w"), indent=1)
print(json.dumps(e, indent=1))
