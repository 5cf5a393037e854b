"""Write the roofline inputs of one ncu --set full capture (one chunk's
section launches: narrow_kernel / wide_kernel) to profiles/ncu_latest.json,
read by bench.py for `traffic` and the issue utilisation:
    python scripts/ncu_json.py gpurun_out/prof_TAG.ncu-rep TAG WORKLOAD SHOTS_IN_CAPTURE"""
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
h, u = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6,
         "ns": 1e-9, "s": 1.0, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def val(r, name):
    i = h.index(name)
    try:
        x = float(r[i].replace(",", "")) * SCALE.get(u[i], 1.0)
    except ValueError:
        return 0.0
    return 0.0 if x != x else x     # ncu prints -nan for metrics it could not collect


kernels = []
for r in rows[2:]:
    if len(r) != len(h):
        continue
    kernels.append({
        "kernel": r[h.index("Kernel Name")].split("(")[0],
        "duration_s": val(r, "gpu__time_duration.sum"),
        "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
        "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": val(r, "smsp__inst_executed.sum"),
        "warps_active_per_sm": val(r, "sm__warps_active.avg.per_cycle_active"),
        "smem_wavefront_pct": val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed")})
tot_t = sum(k["duration_s"] for k in kernels) or 1.0
dom = max(kernels, key=lambda k: k["duration_s"])
d = {"capture": tag, "workload": workload, "shots_in_capture": shots,
     "dram_bytes_per_shot": sum(k["dram_bytes"] for k in kernels) / shots,
     "issue_active_pct": sum(k["issue_active_pct"] * k["duration_s"] for k in kernels) / tot_t,
     "fp64_pipe_pct": sum(k["fp64_pipe_pct"] * k["duration_s"] for k in kernels) / tot_t,
     "smem_wavefront_pct": sum(k["smem_wavefront_pct"] * k["duration_s"] for k in kernels) / tot_t,
     "dram_gbs_serialised": sum(k["dram_bytes"] for k in kernels) / tot_t / 1e9,
     "dominant_kernel": dom["kernel"], "dominant_share": dom["duration_s"] / tot_t,
     "kernels": kernels}
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "ncu_latest.json"), "w") as fh:
    json.dump(d, fh, indent=1)
print(json.dumps({k: v for k, v in d.items() if k != "kernels"}))
