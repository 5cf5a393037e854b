"""Pin the CPU oracle (oracle/gstab_oracle.py) to the golden fixtures that
tests/golden/make_golden.py produced by running the real reference."""

import numpy as np
import pytest

from oracle import gstab_oracle as orc
from paper_2512_23037_b200.circuit import parse_circuit


def test_rng_known_answers(golden_rng):
    assert [orc.splitmix_u64(0, k) for k in range(3)] == golden_rng["splitmix_seed0"]
    for m, s, want in golden_rng["derive_seed"]:
        assert orc.sha1_seed(m, s) == want
    for kat in golden_rng["philox_kat"]:
        assert list(orc.philox4x32_10(kat["ctr"], kat["key"])) == kat["out"]


def _oracle_shots(fx):
    prog = parse_circuit(fx["text"])
    flat = list(prog.flat())
    out = []
    for shot in range(len(fx["shots"])):
        res = orc.run_one_shot(flat, prog.num_qubits,
                               orc.DrawStream("splitmix", fx["master"], shot),
                               fx["capacity"], fx["postselect"])
        out.append({"status": res["status"],
                    "observables": {str(k): v for k, v in
                                    sorted(res["observables"].items())},
                    "discarded_detector": res["discarded_detector"],
                    "overflow_instruction": res["overflow_instruction"],
                    "record": res["record"]})
    return out


def test_oracle_shot_results_bit_exact(golden_shots):
    for fx in golden_shots:
        assert _oracle_shots(fx) == fx["shots"], fx["name"]


def test_oracle_states_match(golden_states):
    for fx in golden_states:
        prog = parse_circuit(fx["text"])
        flat = list(prog.flat())
        for snap in fx["snaps"]:
            res = orc.run_one_shot(flat, prog.num_qubits,
                                   orc.DrawStream("splitmix", fx["master"], fx["shot"]),
                                   4096, False, stop_after=snap["i"], snapshot=True)
            st = res["state"]
            assert st["xs"] == snap["xs"] and st["zs"] == snap["zs"]
            assert st["ph"] == snap["ph"]
            assert st["idx"] == snap["idx"]
            np.testing.assert_array_equal(np.array(st["amp"]), np.array(snap["amp"]))


def test_oracle_counters(golden_counters):
    for fx in golden_counters:
        kw = dict(fx["config"])
        shots = kw.pop("shots")
        got = orc.run_counters(parse_circuit(fx["text"]), shots, **kw)
        assert got["total"] == fx["counters"]["total"]
        for k in ("preserved", "discarded", "overflow", "error_shots"):
            assert got[k] == fx["counters"][k], k
        assert {str(k): v for k, v in got["per_observable"].items()} == \
            fx["counters"]["per_observable"]


def test_oracle_config1_golden_prefix():
    """The oracle reproduces the reference's config-1 records (first 1500 of
    the 1e5 golden shots; the GPU test checks all of them)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden",
                             "config1_records.npz"))
    prog = parse_circuit(str(g["text"]))
    flat = list(prog.flat())
    m = int(g["num_measurements"])
    want = np.unpackbits(g["records"][:1500], axis=1, bitorder="little")[:, :m]
    code = {"preserved": 1, "discarded": 2, "overflow": 3}
    for s in range(1500):
        r = orc.run_one_shot(flat, prog.num_qubits,
                             orc.DrawStream("splitmix", int(g["master"]), s), 4096, True)
        assert code[r["status"]] == g["status"][s]
        rec = np.zeros(m, dtype=np.uint8)
        rec[:len(r["record"])] = r["record"]
        assert np.array_equal(rec, want[s]), s
