"""Sparse chi form (GS_SPARSE) against the dense forms on a few workloads:
device shots/s through run_batch (chi="sparse" / "dense" / "auto").
    python scripts/sparse_point.py [--shots N]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_23037_b200 import SamplerConfig, parse_circuit, run_batch  # noqa: E402
from paper_2512_23037_b200.msc import config4_circuit, msc_d5_circuit  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402


def cancelled_t(nq):
    body = "".join("H %d\nT %d\nDEPOLARIZE1(0.001) %d\nT_DAG %d\nH %d\n" % (q, q, q, q, q)
                   for q in range(nq))
    return parse_circuit(body + "M " + " ".join(map(str, range(nq))) + "\nDETECTOR rec[-1]\n")


ap = argparse.ArgumentParser()
ap.add_argument("--shots", type=int, default=1 << 18)
args = ap.parse_args()
work = [("cancelled_t_24", cancelled_t(24), ("sparse", "auto")),
        ("cancelled_t_16", cancelled_t(16), ("sparse", "dense")),
        ("msc_d5_table2", apply_noise_model(msc_d5_circuit(), 1e-3), ("sparse", "dense")),
        ("config4_n64_t32", apply_noise_model(config4_circuit(64, 32, seed=96), 1e-3),
         ("sparse", "dense", "auto")),
        ("config4_n64_t24", apply_noise_model(config4_circuit(64, 24, seed=88), 1e-3),
         ("sparse", "dense", "auto")),
        ("config4_n24_t24", apply_noise_model(config4_circuit(24, 24, seed=48), 1e-3), ("sparse", "dense"))]
for name, prog, forms in work:
    for chi in forms:
        kw = dict(master_seed=7, rng="philox", postselect=True, chi=chi)
        shots = args.shots if not name.startswith("config4") else args.shots // 16
        run_batch(prog, SamplerConfig(shots=min(shots, 4096), **kw))   # warm-up
        st = run_batch(prog, SamplerConfig(shots=shots, **kw))
        print(json.dumps({"workload": name, "chi": chi, "shots": st.total_shots,
                          "device_shots_per_s": st.total_shots / max(st.device_time_s, 1e-12),
                          "preserved": st.preserved_shots, "overflow": st.overflow_count}),
              flush=True)
