"""Compiler flags of the T ops (CPU): the reduced form (TF_RED) and fused
pairs (TF_FUSE) the wide kernel relies on.

TF_RED marks a BUTTERFLY / GROW whose b-coefficient divided by the gate's
global phase is purely imaginary; payload word 12 carries the sign of
ss = Im(b' ) and T/T_DAG, and the device computes c v + i ss w with the
phase e^{+-i pi/8} counted separately (gs_sweeps.cuh t_mix).  The full
constants a, b i^{xi_s} stay in words 7-10, so the reduced ones must
reproduce them: a = phase * c, b i^{xi_s} = phase * i * ss.
"""

import cmath
import math
import random

from paper_2512_23037_b200 import msc
from paper_2512_23037_b200.compiler import (OP_END, OP_T, T_BUTTERFLY, T_DIAG,
                                            TF_FUSE, TF_FUSEQ, TF_RED, compile_program,
                                            decode_header)
from paper_2512_23037_b200.noise import apply_noise_model

from tests_helpers import random_program


def _f64(w):
    import struct
    return struct.unpack("<d", struct.pack("<Q", int(w)))[0]


def _t_ops(dp):
    ops = dp.ops
    pc = 0
    while True:
        kind, ln, k, fl, _ = decode_header(int(ops[pc]))
        if kind == OP_END:
            return
        if kind == OP_T:
            yield pc, k, fl, [int(x) for x in ops[pc + 1:pc + ln]]
        pc += ln


def _programs():
    yield apply_noise_model(msc.msc_grown_circuit(5), 1e-3)
    yield apply_noise_model(msc.msc_circuit(3), 1e-3)
    for seed in range(12):
        yield msc.config4_circuit(8 + 4 * (seed % 5), 6 + seed, seed=seed)


def test_reduced_form_reproduces_the_full_constants():
    c, s = math.cos(math.pi / 8), math.sin(math.pi / 8)
    n_red = n_full = 0
    for prog in _programs():
        dp = compile_program(prog)
        for pc, k, fl, w in _t_ops(dp):
            case, xis = fl & 3, (fl >> 2) & 3
            a = complex(_f64(w[6]), _f64(w[7]))
            bxs = complex(_f64(w[8]), _f64(w[9]))
            red = bool(fl & TF_RED)
            assert red == (case != T_DIAG and xis % 2 == 0), (pc, fl)
            if not red:
                n_full += 1
                continue
            n_red += 1
            dagger = bool(w[11] & 2)
            ss = -s if w[11] & 1 else s
            phase = cmath.exp((-1j if dagger else 1j) * math.pi / 8)
            assert abs(phase * c - a) < 1e-15
            assert abs(phase * 1j * ss - bxs) < 1e-15
    assert n_red > 50 and n_full > 0


def _noise_pcs(dp):
    return {int(dp.tables[dp.noise_off + 4 * m]) & 0xFFFFFFFF for m in range(dp.num_noise)}


def test_fused_pairs_share_dimension_and_form():
    n_q = 0
    for prog in _programs():
        dp = compile_program(prog)
        noise = _noise_pcs(dp)
        tops = list(_t_ops(dp))
        by_pc = {pc: (k, fl, w) for pc, k, fl, w in tops}
        pcs = [pc for pc, *_ in tops]
        for i, (pc, k, fl, w) in enumerate(tops):
            if not fl & (TF_FUSE | TF_FUSEQ):
                continue
            assert not (fl & TF_FUSE and fl & TF_FUSEQ)
            assert (fl & 3) == T_BUTTERFLY and k >= 2
            nxt = pcs[i + 1]
            k2, fl2, w2 = by_pc[nxt]
            # the partner is the very next op, a BUTTERFLY of the same
            # dimension and form with a different partner vector
            assert nxt == pc + 1 + len(w)
            assert (fl2 & 3) == T_BUTTERFLY and k2 == k
            assert (fl2 & TF_RED) == (fl & TF_RED)
            assert (w2[5] & 0xFFFFFFFF) != (w[5] & 0xFFFFFFFF)
            assert not fl2 & (TF_FUSE | TF_FUSEQ)
            # TF_FUSE: no noise before the partner; TF_FUSEQ: noise there
            # (the device fuses only when none of it fires)
            assert (nxt in noise) == bool(fl & TF_FUSEQ)
            n_q += bool(fl & TF_FUSEQ)
    assert n_q > 0


def test_random_programs_compile_both_forms():
    rng = random.Random(5)
    seen = set()
    for _ in range(40):
        prog = random_program(rng)
        for _, _, fl, _ in _t_ops(compile_program(prog)):
            seen.add((fl & 3, bool(fl & TF_RED)))
    # both forms occur (the non-reduced one when xi_s is odd)
    assert (T_BUTTERFLY, True) in seen and (T_BUTTERFLY, False) in seen


def test_static_span_keeps_cancelled_t_coordinates():
    """ADVICE r01 (medium), pinned: H q; T q; T_DAG q; H q on 24 distinct
    qubits has a one-entry support per noiseless shot in the reference, but
    the shot-invariant span grows by one coordinate per qubit until the
    final measurements.  Past the dimension limit the compile truncates at
    the first T that would exceed it (shots reaching it end UNSUPPORTED or
    OVERFLOW, never silently wrong); at the span's size it compiles whole."""
    from paper_2512_23037_b200 import compile_program, parse_circuit
    text = "".join("H %d\nT %d\nT_DAG %d\nH %d\n" % (q, q, q, q) for q in range(24))
    text += "M " + " ".join(map(str, range(24))) + "\n"
    prog = parse_circuit(text)
    cut = compile_program(prog, max_dim=20)
    assert cut.max_dim == 20
    flat = list(prog.flat())
    assert flat[cut.truncated_at].name == "T" and flat[cut.truncated_at].targets[0] == 20
    whole = compile_program(prog, max_dim=24)
    assert whole.truncated_at is None and whole.max_dim == 24


def test_actions_1q_equals_action_on_random_tableaux():
    """The noise tables' batched single-qubit actions (column reads, gamma =
    delta) equal the general pauli_action restatement row by row."""
    import random
    from paper_2512_23037_b200.compiler import _XZTableau
    rng = random.Random(5)
    for n in (3, 9, 30, 64):
        tab = _XZTableau(n)
        for _ in range(6 * n):
            g = rng.choice(("H", "S", "S_DAG", "H_XY", "X", "CX", "CZ", "SWAP"))
            qs = rng.sample(range(n), 2) if g in ("CX", "CZ", "SWAP") else [rng.randrange(n)]
            tab.gate(g, qs)
        qmask = sum(1 << q for q in rng.sample(range(n), min(n, 12)))
        got = tab.actions_1q(qmask)
        for (q, lx), act in got.items():
            assert act == tab.action(lx << q, (1 - lx) << q, 0), (n, q, lx)
