"""Command-line front end mirroring ``gstab`` (ref cli.py:51-211) for the
sampling commands, running on the B200.

    python -m paper_2512_23037_b200 sample CIRCUIT --shots N [--noise p]
        [--postselect] [--seed S] [--rng splitmix|philox] [--witnesses K]
        [--chi auto|dense|sparse]
    python -m paper_2512_23037_b200 stats CIRCUIT
    python -m paper_2512_23037_b200 bench CIRCUIT --sweep batch-size|noise --values ...
    python -m paper_2512_23037_b200 msc --d 5 [--variant table2|grown|proxy] [--noise p]

Exit codes as the reference: 0 success, 2 usage error, 3 parse error
(ref cli.py:24-27).  ``sample`` writes the reference ``RunStats.as_dict``
JSON (ref sampler.py:133-149) to stdout or --out and a summary to stderr.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

from .circuit import ParseError, compute_stats, parse_circuit
from .noise import NoiseModelError, apply_noise_model

EXIT_OK, EXIT_VALIDATION, EXIT_USAGE, EXIT_PARSE = 0, 1, 2, 3


def _load(path):
    try:
        with open(path) as fh:
            return parse_circuit(fh.read())
    except ParseError as exc:
        print("parse error in %s: %s" % (path, exc), file=sys.stderr)
        sys.exit(EXIT_PARSE)
    except OSError as exc:
        print("error: %s" % exc, file=sys.stderr)
        sys.exit(EXIT_USAGE)


def _emit(payload: str, out):
    if out:
        with open(out, "w") as fh:
            fh.write(payload)
    else:
        sys.stdout.write(payload)


def cmd_sample(a):
    from .sampler import SamplerConfig, run_batch
    prog = _load(a.circuit)
    if a.noise is not None:
        try:
            prog = apply_noise_model(prog, a.noise)
        except NoiseModelError as exc:
            print("error: %s" % exc, file=sys.stderr)
            return EXIT_USAGE
    try:
        cfg = SamplerConfig(shots=a.shots, master_seed=a.seed, batch_size=a.batch_size,
                            entry_capacity=a.entry_capacity,
                            threads=a.threads or int(os.environ.get("SOFT_THREADS", "1")),
                            postselect=a.postselect, rng=a.rng, device=a.device, chi=a.chi)
    except ValueError as exc:
        print("error: %s" % exc, file=sys.stderr)
        return EXIT_USAGE
    st = run_batch(prog, cfg, witnesses=a.witnesses)
    d = st.as_dict()
    if a.witnesses:
        d = dict(d, witnesses=st.witnesses)
    _emit(json.dumps(d, indent=2) + "\n", a.out)
    print("shots=%d preserved=%d discard_rate=%.4f errors=%d ler=%.3e "
          "interval=[%.3e, %.3e] overflow=%d throughput=%.0f/s device=%.0f/s "
          "backend=b200" % (d["total_shots"], d["preserved_shots"],
                            d["discard_rate"], d["logical_error_shots"],
                            d["logical_error_rate"], d["bayes_lo"], d["bayes_hi"],
                            d["overflow_count"], d["throughput"],
                            st.device_dict()["device_shots_per_s"]), file=sys.stderr)
    return EXIT_OK


def cmd_stats(a):
    d = compute_stats(_load(a.circuit)).as_dict()
    width = max(len(k) for k in d)
    for k, v in d.items():
        print("%-*s  %s" % (width, k, v), file=sys.stderr)
    _emit(json.dumps(d, indent=2) + "\n", a.out)
    return EXIT_OK


def cmd_bench(a):
    from .sampler import SamplerConfig, throughput_bench
    prog = _load(a.circuit)
    try:
        vals = [float(v) for v in a.values.split(",") if v.strip()]
    except ValueError:
        print("error: malformed --values %r" % a.values, file=sys.stderr)
        return EXIT_USAGE
    lines = ["value,shots_per_s,discard_rate"]
    if a.shots > 0:
        cfg = SamplerConfig(shots=a.shots, master_seed=a.seed,
                            entry_capacity=a.entry_capacity,
                            postselect=a.postselect, rng=a.rng,
                            batch_size=a.batch_size, chi=a.chi)
        try:
            rows = throughput_bench(prog, cfg, a.sweep, vals)
        except NoiseModelError as exc:
            print("error: %s" % exc, file=sys.stderr)
            return EXIT_USAGE
        lines += ["%g,%.2f,%.6f" % r for r in rows]
    _emit("\n".join(lines) + "\n", a.out)
    return EXIT_OK


def cmd_msc(a):
    from . import msc
    make = {("table2", 5): msc.msc_d5_circuit, ("table2", 3): msc.msc_d3_circuit,
            ("grown", 5): lambda: msc.msc_grown_circuit(5),
            ("proxy", 5): lambda: msc.msc_circuit(5), ("proxy", 3): lambda: msc.msc_circuit(3)}
    if (a.variant, a.d) not in make:
        print("error: no %s circuit at d=%d" % (a.variant, a.d), file=sys.stderr)
        return EXIT_USAGE
    prog = make[(a.variant, a.d)]()
    if a.noise:
        prog = apply_noise_model(prog, a.noise)
    _emit(prog.serialize(), a.out)
    return EXIT_OK


def build_parser():
    ap = argparse.ArgumentParser(prog="paper_2512_23037_b200",
                                 description="B200 sampler for noisy Clifford+T circuits")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("sample", help="run shots and report statistics")
    s.add_argument("circuit")
    s.add_argument("--shots", type=int, required=True)
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--threads", type=int, default=None, help="accepted, ignored")
    s.add_argument("--batch-size", type=int, default=None,
                   help="shots resident per launch (default 2^22)")
    s.add_argument("--noise", type=float, default=None)
    s.add_argument("--postselect", action=argparse.BooleanOptionalAction, default=False)
    s.add_argument("--entry-capacity", type=int, default=4096)
    s.add_argument("--rng", choices=("splitmix", "philox"), default="splitmix")
    s.add_argument("--device", type=int, default=0)
    s.add_argument("--witnesses", type=int, default=0)
    s.add_argument("--chi", choices=("auto", "dense", "sparse"), default="auto",
                   help="chi form (DESIGN.md §3): sparse for supports far below 2^k")
    s.add_argument("--out", default=None)
    s.set_defaults(fn=cmd_sample)
    t = sub.add_parser("stats", help="circuit statistics")
    t.add_argument("circuit")
    t.add_argument("--out", default=None)
    t.set_defaults(fn=cmd_stats)
    b = sub.add_parser("bench", help="throughput sweep (CSV)")
    b.add_argument("circuit")
    b.add_argument("--sweep", choices=("batch-size", "noise"), required=True)
    b.add_argument("--values", required=True)
    b.add_argument("--shots", type=int, default=10000)
    b.add_argument("--batch-size", type=int, default=None,
                   help="wave size for --sweep noise (default 2^22)")
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--postselect", action=argparse.BooleanOptionalAction, default=False)
    b.add_argument("--entry-capacity", type=int, default=4096)
    b.add_argument("--rng", choices=("splitmix", "philox"), default="splitmix")
    b.add_argument("--chi", choices=("auto", "dense", "sparse"), default="auto")
    b.add_argument("--out", default=None)
    b.set_defaults(fn=cmd_bench)
    m = sub.add_parser("msc", help="emit a magic-state-cultivation circuit text")
    m.add_argument("--d", type=int, default=5, choices=(3, 5))
    m.add_argument("--variant", default="table2", choices=("table2", "grown", "proxy"),
                   help="table2: the paper's Table 2 shape (msc_d5_circuit / msc_d3_circuit)")
    m.add_argument("--noise", type=float, default=None)
    m.add_argument("--out", default=None)
    m.set_defaults(fn=cmd_msc)
    return ap


def main(argv=None):
    a = build_parser().parse_args(argv)
    return a.fn(a)
