"""Write the roofline inputs of one ncu --set full capture of the sampling
kernel to profiles/ncu_latest.json (read by bench.py for `traffic`):
    python scripts/ncu_json.py gpurun_out/prof_TAG.ncu-rep TAG WORKLOAD SHOTS"""
import csv
import io
import json
import os
import subprocess
import sys

rep, tag, workload, shots = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u, v = rows[0], rows[1], rows[2]


def val(name):
    i = h.index(name)
    x = float(v[i].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
             "ns": 1e-9, "s": 1.0}.get(u[i], 1.0)
    return x * scale


d = {"capture": tag, "workload": workload, "shots_per_launch": shots,
     "kernel": "gs::sample_kernel",
     "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
     "dram_read_bytes": val("dram__bytes_read.sum"),
     "dram_write_bytes": val("dram__bytes_write.sum"),
     "duration_s_serialised": val("gpu__time_duration.sum"),
     "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
     "fp64_pipe_pct": val("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
     "warp_instructions": val("smsp__inst_executed.sum"),
     "warps_active_per_sm": val("sm__warps_active.avg.per_cycle_active")}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "ncu_latest.json"), "w") as fh:
    json.dump(d, fh, indent=1)
print(json.dumps(d))
