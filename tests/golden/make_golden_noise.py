"""Golden noisy circuit texts written by the REAL reference's uniform
depolarizing transformer (ref gstab/noise.py:104-194) for every BASELINE
workload, so ``tests/test_noise_golden.py`` can pin this repo's
``apply_noise_model`` byte-for-byte against it (CPU only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_noise.py

Writes ``noise_texts.json.gz``: a list of {name, p, base, noisy}, where
``base`` is the noiseless text serialized by the reference's own parser
(gstab.circuit.parse_circuit(...).serialize()) and ``noisy`` is
gstab.noise.apply_noise_model(base, p).serialize().
"""

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def workloads():
    from paper_2512_23037_b200 import msc
    out = [
        ("config1_random_n8_t4", msc.config1_circuit(1), 1e-3),
        ("injection_d3_3_rounds", msc.injection_circuit(3, 3), 5e-4),
        ("config4_random_n32_t24", msc.config4_circuit(32, 24, seed=56), 1e-3),
        ("config4_random_n64_t32", msc.config4_circuit(64, 32, seed=96), 1e-3),
        ("msc_d5_grown_proxy", msc.msc_grown_circuit(5), 1e-3),
        ("msc_d3_proxy", msc.msc_circuit(3), 1e-3),
    ]
    if hasattr(msc, "msc_d5_circuit"):   # the Table-2 circuits
        out += [("msc_d3", msc.msc_d3_circuit(), 1e-3),
                ("msc_d5", msc.msc_d5_circuit(), 1e-3),
                ("msc_d5_p5e-4", msc.msc_d5_circuit(), 5e-4),
                ("msc_d5_p2e-3", msc.msc_d5_circuit(), 2e-3)]
    return out


def main():
    sys.path.insert(0, "/root/reference/pkg/src")
    os.environ.setdefault("GSTAB_BACKEND", "python")
    from gstab.circuit import parse_circuit
    from gstab.noise import apply_noise_model
    out = []
    for name, prog, p in workloads():
        ref = parse_circuit(prog.serialize())
        out.append({"name": name, "p": p, "base": ref.serialize(),
                    "noisy": apply_noise_model(ref, p).serialize()})
        print(name, len(out[-1]["noisy"].splitlines()), "lines")
    with gzip.open(os.path.join(HERE, "noise_texts.json.gz"), "wt") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
