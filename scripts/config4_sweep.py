"""BASELINE config 4 sweep: random Clifford+T circuits, n in {20..64} x
T in {8..32} (chi-growth stress), p=1e-3, 10^5 shots per point through
``run_batch`` (entry capacity 4096 with up to 3 doublings, overflow counted).

    python scripts/config4_sweep.py [--shots N] [--rng philox|splitmix] [--out f.jsonl]

Prints one JSON object per point (device and wall shots/s, overflow /
discard counts, the program's chi dimension limit and section count) and a
markdown table at the end.  Device time = the section launches (CUDA events
on the engine stream); wall = run_batch end to end (host buffers)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_23037_b200 import SamplerConfig, run_batch  # noqa: E402
from paper_2512_23037_b200.msc import config4_circuit  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402
from paper_2512_23037_b200.sampler import _program_for  # noqa: E402

NS = (20, 24, 32, 40, 48, 56, 64)
TS = (8, 16, 24, 32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shots", type=int, default=100_000)
    ap.add_argument("--p", type=float, default=1e-3)
    ap.add_argument("--rng", default="philox", choices=["philox", "splitmix"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    out = open(args.out, "w") if args.out else None
    for n in NS:
        for t in TS:
            prog = apply_noise_model(config4_circuit(n, t, seed=n + t), args.p)
            cfg = SamplerConfig(shots=args.shots, master_seed=n * 1000 + t,
                                rng=args.rng, postselect=True)
            run_batch(prog, SamplerConfig(shots=min(args.shots, 4096),
                                          master_seed=1, rng=args.rng))   # warm-up
            st = run_batch(prog, cfg)
            p = _program_for(prog, cfg.dim_limit)
            row = {"n": n, "t": t, "shots": st.total_shots,
                   "device_shots_per_s": st.device_dict()["device_shots_per_s"],
                   "wall_shots_per_s": st.throughput,
                   "overflow": st.overflow_count, "discarded": st.discarded_shots,
                   "preserved": st.preserved_shots,
                   "logical_error_shots": st.logical_error_shots,
                   "max_dim": p.dp.max_dim, "sections": p.sections(),
                   # chi="auto": truncated programs may run on the sparse form
                   "form": "sparse" if 1 in p._chi_form.values() else "dense",
                   "model_bytes_per_shot": st.model_bytes / max(st.total_shots, 1),
                   "rng": args.rng, "p": args.p}
            rows.append(row)
            line = json.dumps(row)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()
    print("\n| n | T | device shots/s | wall shots/s | overflow | discarded | chi dim limit |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        print("| %d | %d | %.3g | %.3g | %d | %d | %d |" % (
            r["n"], r["t"], r["device_shots_per_s"], r["wall_shots_per_s"],
            r["overflow"], r["discarded"], r["max_dim"]))


if __name__ == "__main__":
    main()
