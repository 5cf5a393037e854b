"""Discard and logical-error rates of the MSC workloads on the B200 (Philox
stream), with Bayes-factor-1000 intervals, against PAPER.md Table 3 / the
reference's acceptance targets (tests/test_acceptance.py:186-199):
    python scripts/msc_rates.py [--shots N] > profiles/msc_rates_TAG.jsonl"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23037_b200 import SamplerConfig, run_batch, msc  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402

TARGETS = [("msc_d5_table2", msc.msc_d5_circuit, 5e-4, 0.6210),
           ("msc_d5_table2", msc.msc_d5_circuit, 1e-3, 0.8560),
           ("msc_d5_table2", msc.msc_d5_circuit, 2e-3, 0.9792),
           ("msc_d3_table2", msc.msc_d3_circuit, 1e-3, 0.313)]

ap = argparse.ArgumentParser()
ap.add_argument("--shots", type=float, default=1e9)
ap.add_argument("--seed", type=int, default=2026)
a = ap.parse_args()
for name, make, p, target in TARGETS:
    prog = apply_noise_model(make(), p)
    t0 = time.perf_counter()
    st = run_batch(prog, SamplerConfig(shots=int(a.shots), master_seed=a.seed,
                                       postselect=True, rng="philox"))
    dt = time.perf_counter() - t0
    lo, hi = st.bayes_interval
    print(json.dumps({"workload": name, "p": p, "shots": st.total_shots,
                      "discard_rate": st.discard_rate, "target_discard": target,
                      "delta_points": 100 * (st.discard_rate - target),
                      "preserved": st.preserved_shots,
                      "logical_errors": st.logical_error_shots,
                      "logical_error_rate": st.logical_error_rate,
                      "bayes_interval": [lo, hi], "wall_s": dt,
                      "shots_per_s": st.total_shots / dt}), flush=True)
