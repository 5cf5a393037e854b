"""The sparse chi form (run flag GS_SPARSE, gs_sparse.cuh): the whole program
warp per shot on a list of the nonzero entries.  Parity with the oracle and
with the dense forms is also covered by the storage-variant parametrisations
of test_gpu_parity.py (goldens, snapshots, dumps, random programs)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import gstab_oracle as orc
from paper_2512_23037_b200 import SamplerConfig, compile_program, parse_circuit, run_batch
from paper_2512_23037_b200 import _lib
from paper_2512_23037_b200.engine import Engine, Program, get_engine


def _config4(n, t):
    from paper_2512_23037_b200.msc import config4_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    return apply_noise_model(config4_circuit(n, t, seed=n + t), 1e-3)


@pytest.mark.parametrize("n,t", [(24, 24), (40, 32), (56, 16)])
def test_sparse_equals_dense_on_config4(n, t):
    """Records, statuses (overflow points included) and observables of the
    sparse form equal the dense forms' shot for shot (the same per-entry
    arithmetic; only norm-sum orders differ), at capacity 32768."""
    prog = _config4(n, t)
    dp = compile_program(prog, max_dim=20)
    p = Program(dp)
    eng = get_engine(0)
    for flags in (_lib.GS_RNG_PHILOX, 0):
        par = Engine.params(17, 0, 512, 32768, flags | _lib.GS_POSTSELECT)
        dense = eng.run_records(p, par)
        par = Engine.params(17, 0, 512, 32768, flags | _lib.GS_POSTSELECT | _lib.GS_SPARSE)
        sp = eng.run_records(p, par)
        for x, y in zip(dense, sp):
            assert np.array_equal(x, y), (n, t, flags)


def test_sparse_counters_and_model_bytes_equal_dense():
    """Counters -- model bytes included (the same per-entry accounting) --
    of a mixed run equal the dense forms'."""
    from paper_2512_23037_b200.msc import msc_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(msc_circuit(3), 2e-3)
    p = Program(compile_program(prog))
    eng = get_engine(0)
    base = _lib.GS_RNG_PHILOX | _lib.GS_POSTSELECT
    c0 = eng.run_counters(p, Engine.params(3, 0, 1 << 16, 32768, base))
    c1 = eng.run_counters(p, Engine.params(3, 0, 1 << 16, 32768, base | _lib.GS_SPARSE))
    assert np.array_equal(c0, c1)


def test_sparse_overflow_at_the_capacity_matches_oracle():
    """A small capacity makes shots overflow inside T layers: the overflow
    instruction and every record before it equal the oracle's."""
    prog = _config4(24, 16)
    flat = list(prog.flat())
    p = Program(compile_program(prog))
    eng = get_engine(0)
    cap = 64
    status, aux, rec, obs = eng.run_records(p, Engine.params(5, 0, 24, cap, _lib.GS_SPARSE))
    n_ovf = 0
    for s in range(24):
        ref = orc.run_one_shot(flat, prog.num_qubits, orc.DrawStream("splitmix", 5, s), cap, False)
        want = {orc.PRESERVED: 1, orc.DISCARDED: 2, orc.OVERFLOW: 3}[ref["status"]]
        assert int(status[s]) == want, s
        if want == 3:
            n_ovf += 1
            assert int(aux[s]) == ref["overflow_instruction"], s
    assert n_ovf > 0


def test_sparse_rejects_capacities_beyond_its_index_field():
    p = Program(compile_program(parse_circuit("H 0\nT 0\nM 0\n")))
    with pytest.raises(RuntimeError):
        get_engine(0).run_counters(p, Engine.params(1, 0, 8, 1 << 17, _lib.GS_SPARSE))


def test_sparse_hash_table_survives_many_builds():
    """Lists of up to 256 entries (k = 8; > 32 entries take the hash-table
    path, <= 32 the warp-match path) through 240 butterflies per shot, on
    one block of warps (blocks=1): every warp fills and clears its table
    ~70,000 times; results equal the dense form's."""
    text = ("H 0 1 2 3 4 5 6 7\nT 0 1 2 3 4 5 6 7\nREPEAT 60 {\n  H 0 1 2 3 4 5 6 7\n"
            "  T 0 1 2 3 4 5 6 7\n  CX 0 1 2 3 4 5 6 7\n}\nM 0 1 2 3 4 5 6 7\n")
    prog = parse_circuit(text)
    p = Program(compile_program(prog))
    assert p.dp.max_dim == 8
    eng = get_engine(0)
    a = eng.run_records(p, Engine.params(2, 0, 4096, 4096, _lib.GS_RNG_PHILOX))
    b = eng.run_records(p, Engine.params(2, 0, 4096, 4096, _lib.GS_RNG_PHILOX | _lib.GS_SPARSE, blocks=1))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_auto_form_on_a_truncated_program_whose_shots_overflow():
    """Config-4 n=64, T=24 is truncated at the dense limit (k 20) but every
    shot overflows before reaching it: chi="auto" probes both forms (no
    UNSUPPORTED shot), keeps the faster, and its counters equal the sparse
    form's and the dense form's."""
    prog = _config4(64, 24)
    kw = dict(shots=2048, master_seed=3, rng="philox", postselect=True)
    a = run_batch(prog, SamplerConfig(**kw))
    s = run_batch(prog, SamplerConfig(chi="sparse", **kw))
    d = run_batch(prog, SamplerConfig(chi="dense", **kw))
    assert a.overflow_count == 2048
    for o in (s, d):
        assert (a.total_shots, a.preserved_shots, a.discarded_shots, a.overflow_count,
                a.model_bytes) == (o.total_shots, o.preserved_shots, o.discarded_shots,
                                   o.overflow_count, o.model_bytes)


def _cancelled(nq):
    body = "".join("H %d\nT %d\nT_DAG %d\nH %d\n" % (q, q, q, q) for q in range(nq))
    return parse_circuit(body + "M " + " ".join(map(str, range(nq))) + "\n")


def test_sparse_span_limits():
    """k = 30 (the u32-coordinate limit) runs sparse; a 31-dimensional span
    is truncated even for the sparse form and stays loud; the largest
    capacity the index field allows (2^16) runs."""
    from paper_2512_23037_b200 import UnsupportedCircuitError
    st = run_batch(_cancelled(30), SamplerConfig(shots=256, master_seed=2))
    assert st.preserved_shots == 256
    with pytest.raises(UnsupportedCircuitError):
        run_batch(_cancelled(31), SamplerConfig(shots=8, master_seed=2))
    st = run_batch(_cancelled(24), SamplerConfig(shots=256, master_seed=2, chi="sparse",
                                                entry_capacity=1 << 13))
    assert st.preserved_shots == 256


def test_sparse_witnesses_equal_dense():
    """Rare-failure witnesses (preserved shots with a flipped observable)
    are the same shot indices on both forms."""
    from paper_2512_23037_b200.msc import msc_d3_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(msc_d3_circuit(), 5e-3)
    kw = dict(shots=1 << 16, master_seed=9, rng="philox", postselect=True)
    # a cap above the error count collects every witness (which ones fill a
    # smaller cap depends on the order shots finish)
    a = run_batch(prog, SamplerConfig(**kw), witnesses=1 << 14)
    b = run_batch(prog, SamplerConfig(chi="sparse", **kw), witnesses=1 << 14)
    assert 0 < a.logical_error_shots < 1 << 14
    assert a.witnesses == b.witnesses
    assert a.logical_error_shots == b.logical_error_shots
