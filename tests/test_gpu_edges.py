"""GPU edge cases: empty runs, Clifford-only programs, records larger than
the shared-memory slot (global record path), REPEAT-heavy programs, the
chi-dimension limit (OVERFLOW vs UNSUPPORTED), 64-qubit masks."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import gstab_oracle as orc
from paper_2512_23037_b200 import SamplerConfig, parse_circuit, run_batch, sample
from paper_2512_23037_b200.sampler import _records_before


def _oracle(prog, master, shots, cap, post, mode="splitmix"):
    flat = list(prog.flat())
    return [orc.run_one_shot(flat, prog.num_qubits, orc.DrawStream(mode, master, s),
                             cap, post) for s in range(shots)]


def _check(prog, master, shots, cfg_kw, cap):
    cfg = SamplerConfig(shots=shots, master_seed=master, **cfg_kw)
    b = sample(prog, cfg)
    ref = _oracle(prog, master, shots, cap, cfg.postselect, cfg.rng)
    for s in range(shots):
        got = b.result(s, measured=_records_before(prog, b, s))
        assert got.status.value == ref[s]["status"], s
        assert got.record == ref[s]["record"], s


def test_zero_shots_and_empty_program():
    st = run_batch(parse_circuit("M 0\n"), SamplerConfig(shots=0))
    assert st.total_shots == 0 and st.discard_rate == 0.0
    st = run_batch(parse_circuit("H 0\n"), SamplerConfig(shots=100))
    assert st.preserved_shots == 100 and st.logical_error_shots == 0


def test_clifford_only_program():
    prog = parse_circuit("H 0\nCX 0 1\nS 1\nDEPOLARIZE1(0.2) 0 1\nM 0 1\n"
                         "DETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-1]\n")
    _check(prog, 4, 64, dict(postselect=True), 4096)


def test_records_beyond_shared_memory_slot():
    # 20000 measurements -> 2.5 KB of record bits per shot (global path)
    text = "H 0\nREPEAT 10000 {\n  X_ERROR(0.01) 0 1\n  M 0 1\n  DETECTOR rec[-2] rec[-4]\n}\n"
    prog = parse_circuit("M 0 1\n" + text)
    _check(prog, 2, 8, dict(postselect=False), 4096)
    b = sample(prog, SamplerConfig(shots=16, master_seed=3, postselect=True))
    assert b.records.shape[1] == (prog.num_measurements + 63) // 64
    # the same in every kernel form (warp per shot: record words beyond the
    # 32 register slots go to the global buffer; block per shot; sparse)
    from paper_2512_23037_b200 import _lib
    for extra in (_lib.GS_WIDE_ONLY, _lib.GS_WIDE_ONLY | _lib.GS_CHI_BLOCK, _lib.GS_SPARSE):
        got = sample(prog, SamplerConfig(shots=8, master_seed=2), extra_flags=extra)
        ref = sample(prog, SamplerConfig(shots=8, master_seed=2))
        assert np.array_equal(got.status, ref.status) and np.array_equal(got.records, ref.records)


def test_dimension_limit_overflow_and_unsupported():
    prog = parse_circuit("H 0 1 2 3 4 5\nT 0 1 2 3 4 5\nM 0\n")   # k reaches 6
    # capacity 8 < 2^4: the reference overflows at the 4th T -> OVERFLOW
    _check(prog, 1, 4, dict(entry_capacity=8, rerun_on_overflow=False, max_dim=3), 8)
    # capacity large, dimension limit 3: not representable -> loud error
    with pytest.raises(RuntimeError):
        run_batch(prog, SamplerConfig(shots=4, max_dim=3))


def test_64_qubit_masks():
    rng = random.Random(64)
    lines = ["H " + " ".join(str(q) for q in range(64))]
    for _ in range(60):
        a, b = rng.sample(range(64), 2)
        lines.append("CX %d %d" % (a, b))
    lines += ["T 63", "T_DAG 0", "DEPOLARIZE1(0.05) 63 0 31", "M 63 0 32",
              "MPP X63*Z0*Y31", "DETECTOR rec[-1]", "OBSERVABLE_INCLUDE(5) rec[-2]"]
    prog = parse_circuit("\n".join(lines) + "\n")
    assert prog.num_qubits == 64
    _check(prog, 9, 48, dict(postselect=True), 4096)
    _check(prog, 9, 48, dict(postselect=True, chi="sparse"), 4096)


def test_witnesses_replay_to_logical_errors():
    """Witness shot indices (preserved shots with a flipped observable) must
    replay through run_shot to an error, and their count equals the counter."""
    from paper_2512_23037_b200 import ShotContext, derive_seed, run_shot
    from paper_2512_23037_b200.msc import msc_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(msc_circuit(3), 2e-3)
    st = run_batch(prog, SamplerConfig(shots=20000, master_seed=6, postselect=True),
                   witnesses=64)
    assert len(st.witnesses) == min(64, st.logical_error_shots)
    for w in st.witnesses[:8]:
        ctx = ShotContext(prog.num_qubits, 4096 * 8)
        ctx.reset(derive_seed(6, w))
        r = run_shot(prog, ctx, postselect=True)
        assert r.status.value == "preserved" and any(r.observables.values())


def test_cli_sample_json_schema(tmp_path):
    import json
    from paper_2512_23037_b200.cli import main
    path = tmp_path / "c.stim"
    path.write_text("H 0\nCX 0 1\nM 0 1\nDETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-1]\n")
    out = tmp_path / "o.json"
    assert main(["sample", str(path), "--shots", "1000", "--noise", "0.01",
                 "--postselect", "--out", str(out)]) == 0
    d = json.loads(out.read_text())
    assert d["total_shots"] == 1000
    assert set(d) >= {"preserved_shots", "discard_rate", "bayes_lo", "throughput"}
    # the sparse chi form through the CLI: the same counters
    out2 = tmp_path / "o2.json"
    assert main(["sample", str(path), "--shots", "1000", "--noise", "0.01",
                 "--postselect", "--chi", "sparse", "--out", str(out2)]) == 0
    d2 = json.loads(out2.read_text())
    for k in ("total_shots", "preserved_shots", "discarded_shots", "logical_error_shots"):
        assert d2[k] == d[k], k


def _cancelled_t(nq: int, noise: bool) -> str:
    """T gates that cancel back to a one-entry support.
    The static span keeps every T coordinate until the final measurements
    (DESIGN.md §8), so the dense chi needs nq dimensions."""
    body = "".join("H %d\nT %d\n%sT_DAG %d\nH %d\n"
                   % (q, q, "DEPOLARIZE1(0.02) %d\n" % q if noise else "", q, q)
                   for q in range(nq))
    return body + "M " + " ".join(map(str, range(nq))) + "\nDETECTOR rec[-1]\n"


def test_cancelled_t_span_beyond_dim_limit_runs_sparse():
    """Past the dense dimension limit the default (chi="auto") runs the
    whole program on the sparse form, like the reference's map; forcing the
    dense forms stays loud; a raised dense limit runs too."""
    from paper_2512_23037_b200 import UnsupportedCircuitError
    prog = parse_circuit(_cancelled_t(22, True))
    cfg = SamplerConfig(shots=8, master_seed=5, chi="dense")
    assert cfg.dim_limit == 20
    with pytest.raises(UnsupportedCircuitError) as ei:
        run_batch(prog, cfg)
    assert ei.value.limit == 20 and ei.value.instruction is not None
    # auto -> sparse: the records equal the reference restatement's (sparse
    # map, one or two entries per shot), in both random streams
    for rng in ("splitmix", "philox"):
        _check(prog, 5, 8, dict(postselect=True, rng=rng), 32768)
        st = run_batch(prog, SamplerConfig(shots=4096, master_seed=5, rng=rng))
        assert st.total_shots == 4096 and st.overflow_count == 0
    # the dense block form with the limit raised to the span agrees
    _check(prog, 5, 8, dict(max_dim=22, postselect=True), 32768)
    # the advisor's noiseless repro: 24 blocks, every shot preserved
    prog24 = parse_circuit(_cancelled_t(24, False))
    st = run_batch(prog24, SamplerConfig(shots=5, master_seed=1))
    assert st.preserved_shots == 5 and st.overflow_count == 0
    _check(prog24, 1, 5, dict(), 32768)


def test_long_noise_stretch_inside_a_wide_section_splitmix():
    """More than 2,048 noise locations (the wide kernel's SplitMix fire-bit
    ring) inserted before one op of a warp-per-shot section: every location
    must still be tested and applied in order (records equal the oracle's)."""
    body = ["H 0 1 2 3 4 5", "T 0 1 2 3 4 5"]                 # chi dimension 6: wide
    body += ["REPEAT 350 {", "  H 6 7", "  DEPOLARIZE1(0.004) 0 1 2 3 4 5 6 7", "}"]
    body += ["CX 0 6 1 7", "M 0 1 2 3 4 5 6 7", "DETECTOR rec[-1] rec[-2]",
             "OBSERVABLE_INCLUDE(0) rec[-3]"]
    prog = parse_circuit("\n".join(body) + "\n")
    from paper_2512_23037_b200.compiler import compile_program
    dp = compile_program(prog)
    assert dp.num_locations > 2048
    for post in (False, True):
        _check(prog, 12, 48, dict(postselect=post), 4096)
        _check(prog, 12, 48, dict(postselect=post, chi="sparse"), 4096)   # same noise scan


def test_narrow_limit5_records_beyond_register_words():
    """The kn=5 narrow build keeps up to 4 record words per lane in
    registers; a program with more measurements inside a k=5 narrow section
    takes the global record buffer -- same records as the oracle's."""
    from paper_2512_23037_b200 import _lib
    from paper_2512_23037_b200.engine import Engine, Program, get_engine
    from paper_2512_23037_b200.compiler import compile_program
    from paper_2512_23037_b200.sampler import ShotBatch
    text = ("H 0 1 2 3 4\nT 0 1 2 3 4\nREPEAT 140 {\n  X_ERROR(0.2) 5\n  M 5\n}\n"
            "M 0 1 2 3 4\nDETECTOR rec[-1] rec[-6]\nOBSERVABLE_INCLUDE(0) rec[-2]\n")
    prog = parse_circuit(text)
    dp = compile_program(prog)
    assert dp.num_measurements > 128 and dp.max_dim == 5
    p = Program(dp)
    eng = get_engine(0)
    for mode, extra in (("splitmix", 0), ("philox", _lib.GS_RNG_PHILOX)):
        par = Engine.params(21, 0, 64, 32768, _lib.GS_POSTSELECT | _lib.GS_NARROW_K5 | extra)
        status, aux, rec, obs = eng.run_records(p, par)
        b = ShotBatch(status, aux, rec, obs, list(dp.obs_keys), dp.num_measurements)
        ref = _oracle(prog, 21, 64, 32768, True, mode)
        for s in range(64):
            got = b.result(s, measured=_records_before(prog, b, s))
            assert got.status.value == ref[s]["status"], (mode, s)
            assert got.record == ref[s]["record"], (mode, s)


def test_thousand_location_instruction_across_the_ring_splitmix():
    """One noise instruction of 1,000 locations (repeated targets: 32-33
    fire-bit words) behind a long stretch of small ones, inserted before one
    op of a wide section: the ring keeps the whole instruction live until it
    is complete (records equal the oracle's)."""
    rep = " ".join(["7"] * 1000)
    body = ["H 0 1 2 3 4 5", "T 0 1 2 3 4 5",
            "REPEAT 90 {", "  H 6", "  DEPOLARIZE1(0.003) 0 1 2 3 4 5 6", "}",
            "X_ERROR(0.003) " + rep, "DEPOLARIZE1(0.01) 6",
            "REPEAT 40 {", "  DEPOLARIZE1(0.003) 0 1 2 3 4 5 6", "}",
            "M 0 1 2 3 4 5 6 7", "DETECTOR rec[-1] rec[-2]", "OBSERVABLE_INCLUDE(0) rec[-3]"]
    prog = parse_circuit("\n".join(body) + "\n")
    for post in (False, True):
        _check(prog, 31, 48, dict(postselect=post), 4096)
        _check(prog, 31, 48, dict(postselect=post, chi="sparse"), 4096)
