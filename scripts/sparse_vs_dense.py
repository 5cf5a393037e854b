"""Counters of the sparse and dense chi forms on the same shots (Philox,
post-selection): every counter, model bytes included, should be equal --
the forms share per-entry arithmetic and differ only in norm-sum order.
    python scripts/sparse_vs_dense.py [--log2-shots 27]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_23037_b200 import SamplerConfig, run_batch  # noqa: E402
from paper_2512_23037_b200.msc import config4_circuit, msc_d5_circuit  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2-shots", type=int, default=27)
args = ap.parse_args()
work = [("msc_d5_table2", apply_noise_model(msc_d5_circuit(), 1e-3), args.log2_shots),
        ("config4_n24_t24", apply_noise_model(config4_circuit(24, 24, seed=48), 1e-3), 20),
        ("config4_n40_t32", apply_noise_model(config4_circuit(40, 32, seed=72), 1e-3), 20),
        ("config4_n56_t16", apply_noise_model(config4_circuit(56, 16, seed=72), 1e-3), 21)]
for name, prog, lg in work:
    out = {}
    for chi in ("dense", "sparse"):
        st = run_batch(prog, SamplerConfig(shots=1 << lg, master_seed=11, rng="philox",
                                           postselect=True, chi=chi))
        out[chi] = (st.total_shots, st.preserved_shots, st.discarded_shots, st.overflow_count,
                    st.logical_error_shots, st.model_bytes, st.device_time_s)
    same = out["dense"][:6] == out["sparse"][:6]
    print(json.dumps({"workload": name, "shots": 1 << lg, "equal": same,
                      "dense": out["dense"], "sparse": out["sparse"]}), flush=True)
