"""Generate golden parity fixtures by running the REAL reference in the build
container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``gstab`` read-only from ``/root/reference/pkg/src`` (numpy backend)
and writes ``tests/golden/*.json.gz``.  The GPU box never reads
``/root/reference``; only these committed fixtures travel.  Programs are
stored as circuit text so every consumer re-parses them with this repo's own
parser.

Fixture files
  rng.json.gz        SplitMix64 / derive_seed / Philox known answers
  shots.json.gz      per-shot ShotResult fields (status, record, observables,
                     discarded detector, overflow instruction) for fuzz suites
                     and hand-written semantic programs, postselect on/off
  states.json.gz     per-instruction tableau + amplitude snapshots (observer)
  counters.json.gz   run_batch counters incl. overflow/rerun cases
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("GSTAB_BACKEND", "python")

from gstab import backend  # noqa: E402
from gstab.circuit import parse_circuit  # noqa: E402
from gstab.fuzz import generate_program, generate_suite  # noqa: E402
from gstab.noise import apply_noise_model  # noqa: E402
from gstab.sampler import (SamplerConfig, ShotContext, ShotRng,  # noqa: E402
                           derive_seed, run_batch, run_shot)

SEMANTIC_PROGRAMS = [
    "M 0\n",
    "X_ERROR(1) 0\nM 0\nDETECTOR rec[-1]\n",
    "X_ERROR(1) 0\nM 0\nDETECTOR rec[-1]\nOBSERVABLE_INCLUDE(0) rec[-1]\n",
    "H 0\nM 0\nX rec[-1] 0\nM 0\n",
    "X 0\nM 0\nH 1\nZ rec[-1] 1\nCZ rec[-1] 1\nH 1\nM 1\n",
    "X 0\nMR 0\nM 0\n",
    "H 0\nR 0\nM 0\n",
    "H 0\nCX 0 1\nMPP Z0*Z1 X0*X1\n",
    "MPP(1.0) Z0\n",
    "H 0\nMPP(0.3) X0 Z0*Z1 Y0\nM 0 1\n",
    "H 0\nH 1\nT 0\nT 1\nM 0\n",
    "H 0\nDEPOLARIZE1(0.3) 0\nM 0\nDETECTOR rec[-1]\nOBSERVABLE_INCLUDE(0) rec[-1]\n",
    "H 0\nCX 0 1\nDEPOLARIZE1(0.1) 0 1\nT 0\nM 0\nM 1\n"
    "DETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-1]\n",
    "H 0\nDEPOLARIZE1(0.4) 0\nM 0\nDETECTOR rec[-1]\n"
    "X_ERROR(0.3) 0\nM 0\nDETECTOR rec[-1] rec[-2]\n",
    "H 0\nCX 0 1\nCX 1 2\nT 0\nT 2\nDEPOLARIZE1(0.02) 0 1 2\n"
    "M 0\nM 1\nM 2\nDETECTOR rec[-2] rec[-3]\nOBSERVABLE_INCLUDE(0) rec[-1]\n",
    # repeated targets compose by OR; DEPOLARIZE2 letters; Y error
    "H 0 1 2\nT 0 1 2\nDEPOLARIZE1(0.5) 0 0 1\nDEPOLARIZE2(0.5) 1 2 0 2\n"
    "Y_ERROR_PLACEHOLDER\n",
    # SWAP-controlled feedback quirk -> Z (ref sampler.py:195-203)
    "H 0\nM 0\nH 1\nSWAP rec[-1] 1\nH 1\nM 1\n",
    # REPEAT with lookbacks and observables on two keys
    "REPEAT 3 {\n  H 0\n  T 0\n  CX 0 1\n  M 1\n  DETECTOR rec[-1]\n}\n"
    "M 0\nOBSERVABLE_INCLUDE(0) rec[-1]\nOBSERVABLE_INCLUDE(3) rec[-2]\n",
    # T layer on GHZ-like state, measurement of products
    "H 0\nCX 0 1\nCX 0 2\nCX 0 3\nT 0 1 2 3\nT_DAG 1\nH_XY 2\nH_NXY 3\n"
    "MPP X0*X1*X2*X3 Z0*Z1\nT 0 1\nM 0 1 2 3\n",
    "H 0 1 2 3\nT 0\nT 1\nT 2\nT 3\nS 0\nS_DAG 1\nT 0\nT_DAG 1\nCZ 0 2\n"
    "SWAP 1 3\nT 2 3\nMPP Y0*X2 Z1*Z3\nR 0\nM 0 1 2 3\n",
]
SEMANTIC_PROGRAMS = [p.replace("Y_ERROR_PLACEHOLDER\n", "M 0 1 2\n")
                     for p in SEMANTIC_PROGRAMS]


def shot_fields(res):
    return {"status": res.status.value,
            "observables": {str(k): v for k, v in sorted(res.observables.items())},
            "discarded_detector": res.discarded_detector,
            "overflow_instruction": res.overflow_instruction,
            "record": res.record}


def run_shots(text, master, shots, postselect, capacity=4096):
    prog = parse_circuit(text)
    ctx = ShotContext(prog.num_qubits, capacity)
    out = []
    for shot in range(shots):
        ctx.reset(derive_seed(master, shot))
        out.append(shot_fields(run_shot(prog, ctx, postselect=postselect,
                                        keep_record=True)))
    return out


class Snap:
    def __init__(self):
        self.snaps = []

    def on_random_pauli(self, i, err):
        pass

    def on_measurement(self, i, p, outcome, prob_plus):
        pass

    def after_instruction(self, i, instr, state):
        t = state.tableau
        self.snaps.append({
            "i": i,
            "ph": [int(v) for v in t.ph],
            "xs": [int(v) for v in t.xs],
            "zs": [int(v) for v in t.zs],
            "idx": [int(v) for v in state.idx],
            "amp": [[float(a.real), float(a.imag)] for a in state.amp]})


def dump(name, obj):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


def config1_program(seed: int) -> str:
    """BASELINE config 1: random Clifford+T, 8 qubits, 4 T, 2 mid-circuit M,
    TICK after each op, final M 0..7 + observable."""
    rng = random.Random(seed)
    one = ("H", "S", "S_DAG", "X", "Y", "Z", "H_XY", "H_NXY")
    two = ("CX", "CZ", "SWAP")
    n = 8
    ops = []
    for _ in range(40):
        if rng.random() < 0.45:
            a, b = rng.sample(range(n), 2)
            ops.append("%s %d %d" % (rng.choice(two), a, b))
        else:
            ops.append("%s %d" % (rng.choice(one), rng.randrange(n)))
    for k in range(4):
        ops.insert(rng.randrange(5, len(ops)),
                   "%s %d" % (rng.choice(("T", "T_DAG")), rng.randrange(n)))
    for k in range(2):
        ops.insert(rng.randrange(len(ops) // 2, len(ops)), "M %d" % rng.randrange(n))
    lines = []
    for op in ops:
        lines.append(op)
        lines.append("TICK")
    lines.append("M " + " ".join(str(q) for q in range(n)))
    lines.append("DETECTOR rec[-9]")
    lines.append("OBSERVABLE_INCLUDE(0) rec[-1]")
    return "\n".join(lines) + "\n"


def main():
    assert backend.name() == "python", backend.name()
    r = ShotRng(0)
    rng_fx = {
        "splitmix_seed0": [r.next_u64() for _ in range(3)],
        "derive_seed": [[m, s, derive_seed(m, s)] for m, s in
                        ((0, 0), (0, 1), (1, 0), (12345, 678), (2**63, 2**40))],
        "philox_kat": [
            {"key": [0, 0], "ctr": [0, 0, 0, 0],
             "out": [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]},
            {"key": [0xFFFFFFFF, 0xFFFFFFFF], "ctr": [0xFFFFFFFF] * 4,
             "out": [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]}],
    }
    dump("rng.json.gz", rng_fx)

    shots_fx = []
    # hand-written semantics
    for i, text in enumerate(SEMANTIC_PROGRAMS):
        for post in (False, True):
            shots_fx.append({"name": "sem%d" % i, "text": text, "master": 7 + i,
                             "postselect": post, "capacity": 4096,
                             "shots": run_shots(text, 7 + i, 24, post)})
    # overflow at tiny capacity (ref tests/test_sampler.py:123-129)
    text = "H 0\nH 1\nT 0\nT 1\nM 0\n"
    shots_fx.append({"name": "overflow", "text": text, "master": 0,
                     "postselect": False, "capacity": 2,
                     "shots": run_shots(text, 0, 4, False, capacity=2)})
    # fuzz suites: default envelope (noise + feedback) and T-free
    for seed, count, kw in ((20260825, 60, {}), (99, 30, {"max_t": 0}),
                            (5, 30, {"max_qubits": 6, "max_gates": 60,
                                     "max_t": 12})):
        for j, prog in enumerate(generate_suite(seed, count, **kw)):
            text = prog.serialize()
            post = j % 2 == 1
            shots_fx.append({"name": "fuzz%d_%d" % (seed, j), "text": text,
                             "master": seed + j, "postselect": post,
                             "capacity": 4096,
                             "shots": run_shots(text, seed + j, 12, post)})
    # config 1 (noisy), 200 shots bit-exact records
    base = parse_circuit(config1_program(1))
    noisy = apply_noise_model(base, 1e-3).serialize()
    shots_fx.append({"name": "config1", "text": noisy, "master": 2026,
                     "postselect": False, "capacity": 4096,
                     "shots": run_shots(noisy, 2026, 200, False)})
    noisy2 = apply_noise_model(base, 2e-2).serialize()
    shots_fx.append({"name": "config1_p2e-2_post", "text": noisy2, "master": 3,
                     "postselect": True, "capacity": 4096,
                     "shots": run_shots(noisy2, 3, 200, True)})
    dump("shots.json.gz", shots_fx)

    states_fx = []
    rng = random.Random(4242)
    progs = [SEMANTIC_PROGRAMS[k] for k in (10, 15, 18, 19)]
    progs += [generate_program(rng, max_qubits=7, max_gates=40, max_t=8).serialize()
              for _ in range(12)]
    for i, text in enumerate(progs):
        prog = parse_circuit(text)
        for shot in range(2):
            ctx = ShotContext(prog.num_qubits, 4096)
            ctx.reset(derive_seed(11, shot))
            obs = Snap()
            res = run_shot(prog, ctx, postselect=False, observer=obs,
                           keep_record=True)
            states_fx.append({"text": text, "master": 11, "shot": shot,
                              "result": shot_fields(res), "snaps": obs.snaps})
    dump("states.json.gz", states_fx)

    counters_fx = []
    cases = [
        ("H 0\nCX 0 1\nDEPOLARIZE1(0.1) 0 1\nT 0\nM 0\nM 1\n"
         "DETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-1]\n",
         dict(shots=300, master_seed=5, postselect=True)),
        ("H 0\nH 1\nT 0\nT 1\nM 0\n",
         dict(shots=5, master_seed=1, entry_capacity=2, rerun_on_overflow=True)),
        ("H 0\nH 1\nT 0\nT 1\nM 0\n",
         dict(shots=5, master_seed=1, entry_capacity=2, rerun_on_overflow=False)),
        ("H 0 1 2\nT 0 1 2\nM 0\n",
         dict(shots=20, master_seed=2, entry_capacity=2,
              max_capacity_doublings=1)),
        ("H 0\nDEPOLARIZE1(0.3) 0\nM 0\nDETECTOR rec[-1]\n"
         "OBSERVABLE_INCLUDE(0) rec[-1]\n",
         dict(shots=400, master_seed=3, postselect=True)),
        (noisy2, dict(shots=400, master_seed=9, postselect=True)),
        (noisy2, dict(shots=400, master_seed=9, postselect=False)),
    ]
    for text, kw in cases:
        st = run_batch(parse_circuit(text), SamplerConfig(**kw))
        counters_fx.append({"text": text, "config": kw, "counters": {
            "total": st.total_shots, "preserved": st.preserved_shots,
            "discarded": st.discarded_shots, "overflow": st.overflow_count,
            "error_shots": st.logical_error_shots,
            "per_observable": {str(k): v for k, v in st.logical_errors.items()}}})
    dump("counters.json.gz", counters_fx)


if __name__ == "__main__":
    main()
