"""Workload generators for the BASELINE configs.

The paper's magic-state-cultivation circuits are not shipped with the
reference (tests/test_acceptance.py:41-42), so they are built
here on the triangular 6.6.6 color code (same patch construction as the
reference's test helper, ref tests/conftest.py:98-114):

  msc_d5_circuit()     the headline (BASELINE config 5): Table 2's shape --
                       42 qubits, 741 gates, 477 2Q, 93 measurements, 72
                       T/T_DAG, T-depth 6 -- injection at d=3, a d=3 window,
                       growth to d=5, two check windows; discard 62.5 /
                       85.8 / 97.9 % at p = 5e-4 / 1e-3 / 2e-3 (paper 62.1 /
                       85.6 / 97.92)
  msc_d3_circuit()     BASELINE config 2: 15 qubits, 137 gates, 22 T;
                       discard 31.0 % at p=1e-3 (paper 31.3 %)
  msc_grown_circuit(5) the round-1 headline proxy (d=3 check, growth, one d=5
                       check, final half-check; 542 gates, 72 T)
  msc_circuit(d)       the simplest proxy (prepare |+_L>, inject, x full
                       T-checks at distance d; d=5: 96 T)
  injection_circuit, config1_circuit, config4_circuit  BASELINE configs 3, 1, 4

Noiselessly every detector and the observable are deterministic (tested);
the Table-2 circuits also have fault distance >= 3 for the observable on the
Clifford proxy (tests/fault_dem.py).  Shape deviations from Table 2 are
reported by ``compute_stats`` and listed in DESIGN.md §8.
"""

from __future__ import annotations

import random

from .circuit import parse_circuit


def color_code_patch(d: int):
    """(qubit sites, faces) of the triangular 6.6.6 color code of distance d:
    sites (r, c), 0 <= c <= r < 3(d-1)/2+1; plaquette centres at
    (r+c) % 3 == 1; every other site is a data qubit."""
    if d < 3 or d % 2 == 0:
        raise ValueError("d must be an odd integer >= 3")
    rows = 3 * (d - 1) // 2 + 1
    sites = [(r, c) for r in range(rows) for c in range(r + 1)]
    centres = [s for s in sites if (s[0] + s[1]) % 3 == 1]
    data = [s for s in sites if (s[0] + s[1]) % 3 != 1]
    index = {s: i for i, s in enumerate(data)}
    faces = []
    for r, c in centres:
        ring = ((r - 1, c - 1), (r - 1, c), (r, c - 1), (r, c + 1),
                (r + 1, c), (r + 1, c + 1))
        faces.append(sorted(index[s] for s in ring if s in index))
    return data, faces


def _pure_errors(nq: int, faces):
    """For each face f a qubit set e_f with |e_f & face_g| odd iff g == f
    (GF(2) right inverse of the face incidence matrix)."""
    rows = []
    for i, f in enumerate(faces):
        m = 0
        for q in f:
            m |= 1 << q
        rows.append([m, 1 << i])
    # reduce to echelon form over GF(2); keep the combination masks
    pivots = []
    for r in rows:
        for pv, pm, pb in pivots:
            if r[0] >> pb & 1:
                r[0] ^= pv
                r[1] ^= pm
        if r[0] == 0:
            raise ValueError("dependent faces")
        b = (r[0] & -r[0]).bit_length() - 1
        pivots.append((r[0], r[1], b))
    # back-substitute so every pivot bit appears in exactly one row
    red = [list(p) for p in pivots]
    for i in range(len(red) - 1, -1, -1):
        vi, mi, bi = red[i]
        for j in range(len(red)):
            if j != i and red[j][0] >> bi & 1:
                red[j][0] ^= vi
                red[j][1] ^= mi
    # solution for face f: qubits = pivots of rows whose combo contains f
    errs = []
    for f in range(len(faces)):
        e = 0
        for v, m, b in red:
            if m >> f & 1:
                e |= 1 << b
        errs.append(sorted(q for q in range(nq) if e >> q & 1))
    return errs


class _Builder:
    def __init__(self):
        self.lines: list[str] = []
        self.meas = 0

    def op(self, text: str):
        self.lines.append(text)

    def tick(self):
        self.lines.append("TICK")

    def measure(self, name: str, qs):
        self.lines.append("%s %s" % (name, " ".join(map(str, qs))))
        self.meas += len(qs)
        return list(range(self.meas - len(qs), self.meas))

    def rec(self, absolute: int) -> str:
        return "rec[%d]" % (absolute - self.meas)


class _Patch:
    """Qubit roles of one color-code patch inside the 42-qubit layout."""

    def __init__(self, data, faces, zanc, xanc, sub0, sub2):
        self.data, self.faces = data, faces
        self.zanc, self.xanc = zanc, xanc
        self.sub0, self.sub2 = sub0, sub2


class _Cultivation:
    """Gadgets shared by the proxies."""

    def __init__(self, b: _Builder, chk: int, flg):
        self.b, self.chk, self.flg = b, chk, list(flg)

    def z_round(self, P: _Patch, detect):
        """Z-face round; ``detect`` = True (every face), False, or the set of
        face indices whose outcome is deterministic."""
        b = self.b
        b.op("R " + " ".join(map(str, P.zanc)))
        b.tick()
        for layer in range(6):
            pairs = []
            for f, face in enumerate(P.faces):
                if layer < len(face):
                    pairs += [face[layer], P.zanc[f]]
            if pairs:
                b.op("CX " + " ".join(map(str, pairs)))
                b.tick()
        ms = b.measure("MR", P.zanc)
        b.tick()
        self._detect(ms, detect)
        return ms

    def x_round(self, P: _Patch, detect):
        b = self.b
        b.op("R " + " ".join(map(str, P.xanc)))
        b.tick()
        b.op("H " + " ".join(map(str, P.xanc)))
        b.tick()
        for layer in range(6):
            pairs = []
            for f, face in enumerate(P.faces):
                if layer < len(face):
                    pairs += [P.xanc[f], face[layer]]
            if pairs:
                b.op("CX " + " ".join(map(str, pairs)))
                b.tick()
        b.op("H " + " ".join(map(str, P.xanc)))
        b.tick()
        ms = b.measure("MR", P.xanc)
        b.tick()
        self._detect(ms, detect)
        return ms

    def _detect(self, ms, detect):
        for f, m in enumerate(ms):
            if detect is True or (detect and f in detect):
                self.b.op("DETECTOR " + self.b.rec(m))

    def t_layer(self, P: _Patch, undo: bool):
        b = self.b
        first, second = ("T", "T_DAG") if undo else ("T_DAG", "T")
        if P.sub0:
            b.op("%s %s" % (first, " ".join(map(str, P.sub0))))
        if P.sub2:
            b.op("%s %s" % (second, " ".join(map(str, P.sub2))))
        b.tick()

    def x_parity(self, P: _Patch, observable: bool):
        """X^n parity of the data block read out through a cat state on the
        check ancilla and the flag qubits (flags end deterministic 0 and
        catch hook errors); each cat qubit drives one segment of data CXs so
        the segments run in parallel."""
        b, chk, flg = self.b, self.chk, self.flg
        cat = [chk] + flg
        b.op("R " + " ".join(map(str, cat)))
        b.tick()
        b.op("H %d" % chk)
        b.tick()
        for f in flg:
            b.op("CX %d %d" % (chk, f))
            b.tick()
        seg = [P.data[i::len(cat)] for i in range(len(cat))]
        for layer in range(max(len(s_) for s_ in seg)):
            pairs = []
            for a, s_ in zip(cat, seg):
                if layer < len(s_):
                    pairs += [a, s_[layer]]
            b.op("CX " + " ".join(map(str, pairs)))
            b.tick()
        for f in reversed(flg):
            b.op("CX %d %d" % (chk, f))
            b.tick()
        b.op("H %d" % chk)
        b.tick()
        ms = b.measure("MR", [chk])
        fms = b.measure("MR", flg) if flg else []
        b.tick()
        if observable:
            b.op("OBSERVABLE_INCLUDE(0) " + b.rec(ms[0]))
        else:
            b.op("DETECTOR " + b.rec(ms[0]))
        for m in fms:
            b.op("DETECTOR " + b.rec(m))

    def prepare_plus(self, P: _Patch, allq):
        """R all, H data, one Z round without detectors, then Pauli-frame
        feedback on a pure-error set per face: |+_L> with every face +1."""
        b = self.b
        b.op("R " + " ".join(map(str, allq)))
        b.tick()
        b.op("H " + " ".join(map(str, P.data)))
        b.tick()
        zm = self.z_round(P, detect=False)
        nd = max(P.data) + 1
        for f, e in enumerate(_pure_errors(nd, P.faces)):
            for q in e:
                b.op("X %s %d" % (b.rec(zm[f]), q))
        b.tick()

    def inject(self, P: _Patch, inj: int):
        """T on the logical Z-parity through an ancilla, MR + DETECTOR."""
        b = self.b
        b.op("R %d" % inj)
        b.tick()
        for q in P.data:
            b.op("CX %d %d" % (q, inj))
        b.tick()
        b.op("T %d" % inj)
        b.tick()
        for q in reversed(P.data):
            b.op("CX %d %d" % (q, inj))
        b.tick()
        im = b.measure("MR", [inj])
        b.tick()
        b.op("DETECTOR " + b.rec(im[0]))

    def check(self, P: _Patch, rounds: int = 1):
        """One cultivation check: T_DAG/T layer, X^n parity (DETECTOR), undo
        layer, then ``rounds`` Z+X syndrome rounds with detectors."""
        self.t_layer(P, undo=False)
        self.x_parity(P, observable=False)
        self.t_layer(P, undo=True)
        for _ in range(rounds):
            self.z_round(P, detect=True)
            self.x_round(P, detect=True)

    def final(self, P: _Patch):
        """Final half-check: T layer + X^n parity into OBSERVABLE_INCLUDE(0)."""
        self.t_layer(P, undo=False)
        self.x_parity(P, observable=True)


def _layout(d: int, flags: int):
    sites, faces = color_code_patch(d)
    nd, nf = len(sites), len(faces)
    data = list(range(nd))
    zanc = list(range(nd, nd + nf))
    xanc = list(range(nd + nf, nd + 2 * nf))
    inj = nd + 2 * nf
    chk = inj + 1
    flg = list(range(chk + 1, chk + 1 + flags))
    sub0 = [q for q, (r, c) in enumerate(sites) if (r + c) % 3 == 0]
    sub2 = [q for q, (r, c) in enumerate(sites) if (r + c) % 3 == 2]
    P = _Patch(data, faces, zanc, xanc, sub0, sub2)
    return sites, P, inj, chk, flg, data + zanc + xanc + [inj, chk] + flg


def msc_circuit(d: int = 5, *, checks: int | None = None, flags: int | None = None,
                final_observable: bool = True, rounds_after_injection: int = 1):
    """Noiseless MSC-like cultivation proxy of distance ``d`` (3 or 5), all
    checks at the final distance.

    Defaults: d=3 -> 1 full check + final half-check on 15 qubits
    (22 T, T-depth 4 as in Table 2); d=5 -> 2 full checks + final
    half-check on 42 qubits (19 data, 9+9 check ancillas, injection, check
    and 3 flag qubits; 96 T, T-depth 6).  See ``msc_grown_circuit`` for the
    d=3 -> d=5 growth variant with Table 2's 72 T.
    """
    if checks is None:
        checks = 1 if d == 3 else 2
    if flags is None:
        flags = 0 if d == 3 else 3
    sites, P, inj, chk, flg, allq = _layout(d, flags)
    b = _Builder()
    g = _Cultivation(b, chk, flg)
    g.prepare_plus(P, allq)
    g.inject(P, inj)
    for _ in range(rounds_after_injection):
        g.z_round(P, detect=True)
        g.x_round(P, detect=True)
    for _ in range(checks):
        g.check(P)
    if final_observable:
        g.final(P)
    return parse_circuit("\n".join(b.lines) + "\n")


def _grown_init(sites, inner_rows: int):
    """|0> / |+> pattern of the data qubits added by the growth.

    The d_to logical pair is kept as Z_L = Z on the left boundary (c == 0)
    and X_L = X on the diagonal boundary (c == r); both restrict to logicals
    of the inner patch, so new qubits on the left boundary start in |0>, on
    the diagonal in |+>.  The others are split so that as many grown faces
    as possible have a deterministic first outcome (Z faces whose new qubits
    are all |0>, X faces whose new qubits are all |+>)."""
    new = [q for q, (r, c) in enumerate(sites) if r >= inner_rows]
    fixed0 = {q for q in new if sites[q][1] == 0}
    fixedp = {q for q in new if sites[q][0] == sites[q][1]}
    return new, fixed0, fixedp


def msc_grown_circuit(d: int = 5, *, d_inner: int = 3, inner_checks: int = 1,
                      checks: int = 1, flags: int = 3,
                      rounds_after_injection: int = 1, rounds_after_growth: int = 1,
                      final_observable: bool = True):
    """MSC proxy with the paper's injection -> cultivate at d=3 -> grow to
    d=5 -> cultivate structure (Table 2 d=5: 42 qubits,
    72 T, T-depth 6 = 1 injection T + 2 layers x 7 + 3 layers x 19).

    The inner d_inner patch is the top corner (rows < 3(d_inner-1)/2+1) of
    the distance-d triangle, so it reuses the first data qubits and the
    corner faces.  Growth: the new data qubits start in |0> or |+>
    (``_grown_init``), one Z and one X round of every distance-d face
    follows, faces with a deterministic outcome get DETECTORs and every
    other face is fixed to +1 by Pauli-frame feedback on a pure error that
    commutes with the kept logical pair -- the logical state of the inner
    patch is carried over exactly (Z_L and X_L commute with every measured
    face).  Noiselessly every detector and the observable are
    deterministic (tested).
    """
    sites, P, inj, chk, flg, allq = _layout(d, flags)
    inner_rows = 3 * (d_inner - 1) // 2 + 1
    isites, ifaces = color_code_patch(d_inner)
    assert sites[:len(isites)] == isites
    ni = len(isites)
    # inner faces = outer faces whose centre lies in the corner, restricted
    # to inner data (same order as color_code_patch(d_inner))
    outer_of = []
    for f, face in enumerate(P.faces):
        inner = [q for q in face if q < ni]
        if inner and sorted(inner) in [sorted(x) for x in ifaces]:
            outer_of.append((ifaces.index(sorted(inner)), f))
    outer_of.sort()
    assert [i for i, _ in outer_of] == list(range(len(ifaces)))
    Pi = _Patch(list(range(ni)), ifaces, [P.zanc[f] for _, f in outer_of],
                [P.xanc[f] for _, f in outer_of],
                [q for q in P.sub0 if q < ni], [q for q in P.sub2 if q < ni])
    b = _Builder()
    g = _Cultivation(b, chk, flg)
    # --- inner stage: prepare, inject, cultivate at d_inner
    g.prepare_plus(Pi, allq)
    g.inject(Pi, inj)
    for _ in range(rounds_after_injection):
        g.z_round(Pi, detect=True)
        g.x_round(Pi, detect=True)
    for _ in range(inner_checks):
        g.check(Pi)
    # --- growth to distance d
    new, zero, plus = _grown_init(sites, inner_rows)
    free = [q for q in new if q not in zero and q not in plus]
    # a grown face is deterministic only if its inner part is empty or an
    # inner face (a stabilizer of the inner code)
    inner_ok = [not [q for q in face if q < ni] or
                sorted(q for q in face if q < ni) in [sorted(x) for x in ifaces]
                for face in P.faces]
    best = None
    for m in range(1 << len(free)):
        z_ = zero | {q for i, q in enumerate(free) if not m >> i & 1}
        p_ = plus | {q for i, q in enumerate(free) if m >> i & 1}
        zdet = [f for f, face in enumerate(P.faces)
                if inner_ok[f] and all(q in z_ for q in face if q >= ni)]
        xdet = [f for f, face in enumerate(P.faces)
                if inner_ok[f] and all(q in p_ for q in face if q >= ni)]
        key = len(zdet) + len(xdet)
        if best is None or key > best[0]:
            best = (key, sorted(p_), zdet, xdet)
    _, plus_q, zdet, xdet = best
    if plus_q:
        b.op("H " + " ".join(map(str, plus_q)))
        b.tick()
    zm = g.z_round(P, detect=set(zdet))
    xm = g.x_round(P, detect=set(xdet))
    nd = len(P.data)
    left = [q for q in P.data if sites[q][1] == 0]
    diag = [q for q in P.data if sites[q][0] == sites[q][1]]
    # pure errors that also commute with the kept logical representative
    xerr = _pure_errors(nd, P.faces + [left])[:len(P.faces)]
    zerr = _pure_errors(nd, P.faces + [diag])[:len(P.faces)]
    for f in range(len(P.faces)):
        if f not in zdet:
            for q in xerr[f]:
                b.op("X %s %d" % (b.rec(zm[f]), q))
        if f not in xdet:
            for q in zerr[f]:
                b.op("Z %s %d" % (b.rec(xm[f]), q))
    b.tick()
    for _ in range(rounds_after_growth):
        g.z_round(P, detect=True)
        g.x_round(P, detect=True)
    # --- cultivation at distance d
    for _ in range(checks):
        g.check(P)
    if final_observable:
        g.final(P)
    return parse_circuit("\n".join(b.lines) + "\n")


def random_clifford_t(n: int, gates: int, t_count: int, mid_measurements: int,
                      seed: int, *, tick: bool = True, plus_start: bool = False):
    """Random Clifford+T circuit (BASELINE configs 1 and 4): ``gates``
    Cliffords from {H,S,S_DAG,X,Y,Z,H_XY,H_NXY,CX,CZ,SWAP}, ``t_count``
    T/T_DAG and ``mid_measurements`` M at random positions, TICK after each
    op, final M on all qubits, one detector on the first mid-circuit
    measurement and OBSERVABLE_INCLUDE(0) on the last qubit."""
    rng = random.Random(seed)
    one = ("H", "S", "S_DAG", "X", "Y", "Z", "H_XY", "H_NXY")
    two = ("CX", "CZ", "SWAP")
    ops = []
    for _ in range(gates):
        if n >= 2 and rng.random() < 0.45:
            a, c = rng.sample(range(n), 2)
            ops.append("%s %d %d" % (rng.choice(two), a, c))
        else:
            ops.append("%s %d" % (rng.choice(one), rng.randrange(n)))
    for _ in range(t_count):
        ops.insert(rng.randrange(1, len(ops) + 1),
                   "%s %d" % (rng.choice(("T", "T_DAG")), rng.randrange(n)))
    for _ in range(mid_measurements):
        ops.insert(rng.randrange(len(ops) // 2, len(ops) + 1),
                   "M %d" % rng.randrange(n))
    lines = ["H " + " ".join(str(q) for q in range(n)), "TICK"] if plus_start else []
    for o in ops:
        lines.append(o)
        if tick:
            lines.append("TICK")
    lines.append("M " + " ".join(str(q) for q in range(n)))
    if mid_measurements:
        lines.append("DETECTOR rec[-%d]" % (n + mid_measurements))
    lines.append("OBSERVABLE_INCLUDE(0) rec[-1]")
    return parse_circuit("\n".join(lines) + "\n")


def injection_circuit(d: int = 3, rounds: int = 3):
    """BASELINE config 3: color-code T-state injection followed by ``rounds``
    Z+X syndrome rounds with detectors and a final T-check whose X^n parity
    is the observable (post-selection on every detector)."""
    return msc_circuit(d, checks=0, flags=0, rounds_after_injection=rounds)


def config1_circuit(seed: int = 1):
    """BASELINE config 1: random Clifford+T on 8 qubits, 40 Cliffords, 4 T,
    2 mid-circuit M (noise is added with apply_noise_model(p=1e-3))."""
    return random_clifford_t(8, 40, 4, 2, seed)


def config4_circuit(n: int, t_count: int, seed: int = 0):
    """BASELINE config 4: chi-growth stress, random Clifford+T with n qubits
    and ``t_count`` T gates, 3n Cliffords and n//8 mid-circuit M."""
    return random_clifford_t(n, 3 * n, t_count, max(1, n // 8), seed,
                             plus_start=True)


# ======================================================================
# Table-2 cultivation circuits (msc_d3_circuit / msc_d5_circuit)
# ======================================================================
#
# Built op by op into a qubit-level ASAP schedule (``_Layers``): every op is
# placed in the earliest TICK layer after the previous op on each of its
# qubits (so the circuit is exactly the program-order circuit), measurements
# never move before an earlier measurement (record order is program order),
# and classically controlled Pauli corrections run at the start of a layer
# after their measurement.  Detectors and observables are written with
# absolute record indices and emitted as lookbacks after their last
# measurement.


class _Layers:
    def __init__(self):
        self.ops = []            # (layer, phase, seq, name, targets)
        self.ready = {}
        # preparation (R, then optional single-qubit gates) deferred to the
        # layers right before the qubit's next op: ALAP, so a freshly reset
        # ancilla does not idle (and collect errors) before it is used
        self.pending = {}
        self.nmeas = 0
        self.meas_at = []        # layer of each measurement
        self.seq = 0
        self.notes = []          # (layer, seq, text builder)

    def _at(self, qs):
        return max([self.ready.get(q, 0) + len(self.pending.get(q, ()))
                    for q in qs] + [0])

    def _flush(self, qs, L):
        """Place the pending preparation of qs in the layers before L."""
        for q in qs:
            pend = self.pending.pop(q, None)
            if pend:
                for k, name in enumerate(pend):
                    self._put(L - len(pend) + k, 1, name, (q,))

    def _put(self, layer, phase, name, targets):
        self.ops.append((layer, phase, self.seq, name, tuple(targets)))
        self.seq += 1

    def gate(self, name, *qs):
        """One gate on qubits qs (1 or 2 targets)."""
        L = self._at(qs)
        self._flush(qs, L)
        self._put(L, 1, name, qs)
        for q in qs:
            self.ready[q] = L + 1

    def gates(self, name, qs):
        for q in qs:
            self.gate(name, q)

    def layer(self, named):
        """Single-qubit gates [(name, q), ...] in one common layer."""
        L = self._at([q for _, q in named])
        self._flush([q for _, q in named], L)
        for name, q in named:
            self._put(L, 1, name, (q,))
            self.ready[q] = L + 1

    def cx(self, pairs):
        for c, t in pairs:
            self.gate("CX", c, t)

    def reset(self, qs, then=()):
        """R (followed by the single-qubit gates `then`) on each qubit of qs,
        deferred to just before the qubit's next op."""
        for q in qs:
            if q in self.pending:
                raise ValueError("qubit %d reset twice" % q)
            self.pending[q] = ["R"] + list(then)

    def measure(self, name, qs, by_ready=False):
        """M / MR of each qubit; returns absolute record indices (in the
        order of qs).  by_ready: record them in the order the qubits become
        free, so none waits on a later-ready one (records stay in program
        order, which is this order)."""
        if by_ready:
            order = sorted(range(len(qs)), key=lambda i: (self._at((qs[i],)), i))
            got = self.measure(name, [qs[i] for i in order])
            out = [0] * len(qs)
            for k, i in enumerate(order):
                out[i] = got[k]
            return out
        out = []
        for q in qs:
            L = self._at((q,))
            self._flush((q,), L)
            self._put(L, 1, name, (q, "#%d" % self.nmeas))
            self.ready[q] = L + 1
            self.meas_at.append(L)
            out.append(self.nmeas)
            self.nmeas += 1
        return out

    def mpp(self, term):
        qs = [int(t[1:]) for t in term.split("*")]
        L = self._at(qs)
        self._flush(qs, L)
        self._put(L, 1, "MPP", (term, "#%d" % self.nmeas))
        for q in qs:
            self.ready[q] = L + 1
        self.meas_at.append(L)
        self.nmeas += 1
        return self.nmeas - 1

    def feedback(self, pauli, m, q):
        """Pauli on q iff measurement m returned -1 (noiseless frame update)."""
        if q in self.pending:
            raise ValueError("feedback on a qubit awaiting preparation")
        L = max(self.ready.get(q, 0), self.meas_at[m] + 1)
        self._put(L, 0, pauli, ("@%d" % m, q))
        self.ready[q] = L

    def note(self, kind, ms):
        L = max(self.meas_at[m] for m in ms)
        self.notes.append((L, self.seq, kind, tuple(ms)))
        self.seq += 1

    # -- dynamical decoupling ----------------------------------------
    def pad_dd(self, qubits, count):
        """Insert `count` single-qubit gates as identity sequences (X X, or
        X Y Z once when count is odd) on `qubits` inside their idle windows
        (consecutive non-empty layers with no op on the qubit, between two of
        its ops).  A gate replaces the idle DEPOLARIZE1 of its layer by the
        same DEPOLARIZE1 after the gate, so the noisy circuit's channels
        are unchanged; the unitary is the identity up to a global phase."""
        if count <= 0:
            return
        if count == 1:
            raise ValueError("cannot pad a single gate")
        nonempty = sorted({op[0] for op in self.ops if op[1] == 1})
        busy = {}
        for L, ph, s, name, tg in self.ops:
            qs = [int(t[1:]) for t in tg[0].split("*")] if name == "MPP" else tg
            for q in qs:
                if isinstance(q, int):
                    busy.setdefault(q, set()).add(L)
        windows = []
        for q in qubits:
            b = sorted(busy.get(q, ()))
            for a, c in zip(b, b[1:]):
                run = [L for L in nonempty if a < L < c]
                if len(run) >= 2:
                    windows.append((len(run), q, run))
        windows.sort(key=lambda w: (-w[0], w[1]))
        seqs = []
        rem = count
        if rem % 2:
            seqs.append(("X", "Y", "Z"))
            rem -= 3
        seqs += [("X", "X")] * (rem // 2)
        placed = 0
        wi = 0
        # round-robin over the longest windows, one sequence per window visit
        slots = [list(w[2]) for w in windows]
        while placed < len(seqs):
            if not windows:
                raise ValueError("no idle windows left for dynamical decoupling")
            _, q, _ = windows[wi % len(windows)]
            run = slots[wi % len(windows)]
            sq = seqs[placed]
            if len(run) >= len(sq):
                for g, L in zip(sq, run[:len(sq)]):
                    self._put(L, 1, g, (q,))
                del run[:len(sq)]
                placed += 1
            wi += 1
            if wi > 100000:
                raise ValueError("dynamical decoupling does not fit")

    # -- emission -----------------------------------------------------
    def text(self):
        """Circuit text: layers in order, TICK after each; measurement
        records numbered in emission order (ids -> indices), detectors and
        observables after the layer of their last measurement."""
        layers = {}
        for op in self.ops:
            layers.setdefault(op[0], []).append(op)
        notes = {}
        for n in self.notes:
            notes.setdefault(n[0], []).append(n)
        index = {}
        lines = []
        count = 0
        for L in sorted(set(layers) | set(notes)):
            ops = sorted(layers.get(L, []), key=lambda o: (o[1], o[2]))
            prev = None
            for _, ph, _, name, tg in ops:
                if ph == 0:
                    m, q = int(tg[0][1:]), tg[1]
                    lines.append("%s rec[%d] %d" % (name, index[m] - count, q))
                    prev = None
                    continue
                if name == "MPP":
                    index[int(tg[1][1:])] = count
                    lines.append("MPP " + tg[0])
                    count += 1
                    prev = None
                    continue
                if name in ("M", "MR"):
                    index[int(tg[1][1:])] = count
                    count += 1
                    tg = tg[:1]
                if prev == name:
                    lines[-1] += " " + " ".join(map(str, tg))
                else:
                    lines.append(name + " " + " ".join(map(str, tg)))
                prev = name
            for _, _, kind, ms in sorted(notes.get(L, []), key=lambda n: n[1]):
                lb = " ".join("rec[%d]" % (index[m] - count) for m in ms)
                lines.append(("DETECTOR " if kind == "det" else "OBSERVABLE_INCLUDE(0) ") + lb)
            lines.append("TICK")
        return "\n".join(lines) + "\n"


# interleaved Z/X stabilizer-round schedules, per face: (data qubit, layer of
# its CX with the Z ancilla, layer of its CX with the X ancilla); found by a
# constraint search (distinct layers per qubit and per ancilla; even
# Z-before-X counts on every overlapping face pair): 6 CX layers at d=3,
# 7 at d=5 (a sequential Z-then-X round needs 8 / 12)
_ROUND_SCHEDULE = {
    3: [((0, 1, 2), (1, 3, 1), (2, 0, 3), (3, 2, 0)),
        ((1, 2, 0), (3, 5, 1), (5, 4, 3), (6, 3, 2)),
        ((2, 4, 1), (3, 3, 4), (4, 2, 3), (5, 5, 2))],
    9: [((0, 6, 3), (1, 5, 2), (2, 3, 4), (3, 4, 5)),
        ((1, 3, 1), (3, 6, 3), (5, 5, 2), (6, 4, 0)),
        ((2, 2, 0), (3, 1, 2), (4, 4, 5), (5, 0, 1), (7, 6, 3), (8, 3, 4)),
        ((4, 3, 1), (7, 1, 2), (10, 2, 0), (11, 0, 4)),
        ((5, 4, 3), (6, 2, 1), (8, 6, 5), (9, 0, 2), (12, 5, 4), (13, 1, 6)),
        ((7, 0, 5), (8, 1, 0), (11, 3, 1), (12, 2, 3), (15, 5, 2), (16, 6, 4)),
        ((9, 1, 3), (13, 3, 2), (17, 4, 1), (18, 2, 4)),
        ((10, 5, 3), (11, 6, 2), (14, 4, 5), (15, 3, 4)),
        ((12, 0, 1), (13, 4, 0), (16, 2, 3), (17, 3, 2))],
}


class _Cult2:
    """Gadgets of the Table-2 circuits on one color-code patch."""

    def __init__(self, S: _Layers, data, faces, zanc, xanc, sites):
        self.S, self.data, self.faces = S, list(data), [list(f) for f in faces]
        self.zanc, self.xanc, self.sites = list(zanc), list(xanc), sites

    def sub(self, k):
        return [q for q in self.data if (self.sites[q][0] + self.sites[q][1]) % 3 == k]

    def encode_t(self):
        """|T_L> on the distance-3 patch by unitary encoding: T|+> on the
        input qubit, copied onto a weight-3 logical X representative that
        avoids the face pivots, then (I + X_f) on every face through its
        pivot (a qubit of that face only)."""
        S, data, faces = self.S, self.data, self.faces
        pivots = []
        for i, f in enumerate(faces):
            only = [q for q in f if all(q not in g for j, g in enumerate(faces) if j != i)]
            pivots.append(only[0])
        # weight-3 X logical (odd, even overlap with every face) avoiding pivots
        rest = [q for q in data if q not in pivots]
        logical = None
        for a in range(len(rest)):
            for b in range(a + 1, len(rest)):
                for c in range(b + 1, len(rest)):
                    L = {rest[a], rest[b], rest[c]}
                    if all(len(L & set(f)) % 2 == 0 for f in faces):
                        logical = sorted(L)
                        break
                if logical:
                    break
            if logical:
                break
        src = logical[0]
        S.reset([src], then=("H", "T"))
        S.reset(pivots, then=("H",))
        S.reset([q for q in data if q != src and q not in pivots])
        S.cx([(src, q) for q in logical[1:]])
        # fan-outs, scheduled so that each layer touches disjoint qubits
        fans = [[(p, q) for q in f if q != p] for p, f in zip(pivots, faces)]
        for k in range(max(len(x) for x in fans)):
            for i, x in enumerate(fans):
                if x:
                    S.cx([x[(k + i) % len(x)]]) if k < len(x) else None

    def round(self, detect=True):
        """Z- and X-stabilizer measurement of every face, separate ancillas,
        interleaved in the face's CX schedule (_ROUND_SCHEDULE: each data
        qubit meets one ancilla per layer, and for every Z face f and X face
        g the shared qubits see Z_f before X_g an even number of times, so
        both ancillas measure exactly their stabilizer): R ancillas, X
        ancillas to |+>, CX data->Z-ancilla / X-ancilla->data, X-basis
        readout; DETECTORs on the faces in `detect` (True: all)."""
        S = self.S
        fs = range(len(self.faces))
        S.reset([self.zanc[f] for f in fs])
        S.reset([self.xanc[f] for f in fs], then=("H",))
        sched = _ROUND_SCHEDULE[len(self.faces)]
        cx = []
        for f in fs:
            for q, lz, lx in sched[f]:
                cx.append((lz, f, 0, (q, self.zanc[f])))
                cx.append((lx, f, 1, (self.xanc[f], q)))
        for _, _, _, pair in sorted(cx):
            S.cx([pair])
        S.gates("H", [self.xanc[f] for f in fs])
        ms = S.measure("MR", [self.zanc[f] for f in fs] + [self.xanc[f] for f in fs],
                       by_ready=True)
        zm = dict(zip(fs, ms[:len(fs)]))
        xm = dict(zip(fs, ms[len(fs):]))
        for m in sorted(ms):
            f = ms.index(m)
            key = ("z", f) if f < len(fs) else ("x", f - len(fs))
            if detect is True or (detect and key in detect):
                S.note("det", [m])
        return zm, xm

    def t_layer(self, undo):
        """T_DAG on sublattice 0 and T on sublattice 2 (the undo swaps them),
        all in one layer: the H_XY check conjugated into an X check with
        physical H_XY / H_NXY."""
        first, second = ("T", "T_DAG") if undo else ("T_DAG", "T")
        self.S.layer([(first, q) for q in self.sub(0)] + [(second, q) for q in self.sub(2)])

    def cat_check(self, cat, detect=True):
        """X^n of the data through a cat state on `cat` (root first): each
        cat qubit drives one contiguous segment of data CXs; the root is
        read out in the X basis (the check), the others in Z (flags: a cat
        qubit X error, e.g. a hook, shows here)."""
        S = self.S
        S.reset(cat[:1], then=("H",))
        S.reset(cat[1:])
        S.cx([(cat[0], c) for c in cat[1:]])
        n = len(self.data)
        seg = [self.data[i * n // len(cat):(i + 1) * n // len(cat)] for i in range(len(cat))]
        for k in range(max(len(s) for s in seg)):
            for c, s in zip(cat, seg):
                if k < len(s):
                    S.cx([(c, s[k])])
        S.cx([(cat[0], c) for c in reversed(cat[1:])])
        S.gate("H", cat[0])
        ms = S.measure("MR", cat, by_ready=True)
        if detect:
            for m in ms:
                S.note("det", [m])
        return ms

    def _fold_tree(self, root):
        """CX pairs (parent, child), in time order, of a doubling fan tree
        over the data rooted at `root`: back-propagated from the end, the
        root's operator reaches one new qubit per infected qubit per layer
        (3 layers for 7 qubits), so the pairs are emitted latest-last."""
        rest = [q for q in self.data if q != root]
        infected = [root]
        rounds = []
        while rest:
            links = []
            for p in list(infected):
                if rest:
                    c = rest.pop(0)
                    links.append((p, c))
                    infected.append(c)
            rounds.append(links)
        return [e for links in reversed(rounds) for e in links]

    def fold_check(self, root, detect=True):
        """X^n of the data folded onto data qubit `root` by a CX fan tree
        (root's X spreads to every data qubit), read out non-destructively
        in the X basis (H, M, H) and unfolded."""
        S = self.S
        tree = self._fold_tree(root)
        S.cx(tree)
        S.gate("H", root)
        m = S.measure("M", [root])[0]
        S.gate("H", root)
        S.cx(list(reversed(tree)))
        if detect:
            S.note("det", [m])
        return m

    def fold_inject(self, root):
        """T_L = T on the logical Z parity: Z^n folded onto data qubit
        `root` by a CX fan-in tree (data controls, parent targets), T on the
        root, unfold."""
        S = self.S
        tree = [(c, p) for p, c in self._fold_tree(root)]
        S.cx(tree)
        S.gate("T", root)
        S.cx(list(reversed(tree)))

    def prepare_plus(self):
        """|+_L>: R and H on the data, one Z round (random outcomes, no
        detectors), Pauli-frame feedback on a pure error of each face."""
        S = self.S
        S.reset(self.data, then=("H",))
        S.reset(self.zanc)
        width = max(len(f) for f in self.faces)
        sched = _ROUND_SCHEDULE[len(self.faces)]
        cx = []
        for f in range(len(self.faces)):
            for q, lz, _ in sched[f]:
                cx.append((lz, f, (q, self.zanc[f])))
        for _, _, pair in sorted(cx):
            S.cx([pair])
        zm = S.measure("MR", self.zanc, by_ready=True)
        for f, e in enumerate(_pure_errors(max(self.data) + 1, self.faces)):
            for q in e:
                S.feedback("X", zm[f], q)

    def observable(self, record=True):
        """Noiseless MPP of X on every data qubit: the H_XY logical in the
        rotated frame (between the T_DAG/T layer and its undo); the first one
        of a window is OBSERVABLE_INCLUDE(0), the second one (record=False)
        closes the window as DETECTOR(first xor second)."""
        m = self.S.mpp("*".join("X%d" % q for q in self.data))
        if record:
            self.S.note("obs", [m])
        return m


def _d5_layout():
    sites, faces = color_code_patch(5)
    nd, nf = len(sites), len(faces)
    data = list(range(nd))
    zanc = list(range(nd, nd + nf))
    xanc = list(range(nd + nf, nd + 2 * nf))
    cat = list(range(nd + 2 * nf, nd + 2 * nf + 5))
    return sites, data, faces, zanc, xanc, cat


def _finish(S, target_1q, dd_qubits):
    prog = parse_circuit(S.text())
    from .circuit import compute_stats
    st = compute_stats(prog)
    need = target_1q - (st.total_gates - st.two_qubit_gates)
    if need:
        S.pad_dd(dd_qubits, need)
        prog = parse_circuit(S.text())
    return prog


def msc_d5_circuit(*, dd: bool = True, cats=((2, 2), (3, 3), (2, 1))):
    """Magic-state cultivation at d=5 with the paper's Table 2 shape (42
    qubits, 741 gates, 477 two-qubit gates, 93 measurements, 72 T/T_DAG on
    the 19 data qubits, T-depth 6, depth 92 vs 94):

      inject    |T_L> at d=3 by unitary encoding (T|+> on one data qubit)
      round     one d=3 stabilizer round (interleaved Z/X, 6 CX layers)
      window    T_DAG/T layer, two flagged cat checks of X^7, undo layer
      grow      new data: Bell pairs on the two boundaries that carry the
                kept logicals, |0>/|+> elsewhere; two d=5 rounds, Pauli-frame
                feedback restoring every face to +1
      window A  T_DAG/T layer, noiseless MPP of X^19 (the rotated-frame H_XY
                logical) -> OBSERVABLE_INCLUDE(0), two flagged cat checks,
                a second noiseless MPP -> DETECTOR(first xor second), undo
      rounds    two d=5 rounds
      window B  T_DAG/T layer, two cat checks (the second unflagged)

    Under the reference's uniform noise model (apply_noise_model) every
    detector and the observable are deterministic without noise, and no
    fault set of weight <= 2 flips the observable undetected on the Clifford
    proxy (tests/fault_dem.py); single-qubit gate count padded to Table 2 by
    identity dynamical-decoupling sequences on idle data (noise-neutral).
    `cats` = cat sizes of the checks of the three windows."""
    sites, data, faces, zanc, xanc, cat = _d5_layout()
    S = _Layers()
    inner_rows = 4
    ni = 7
    ifaces = color_code_patch(3)[1]
    outer_of = []
    for f, face in enumerate(faces):
        inner = sorted(q for q in face if q < ni)
        if inner in [sorted(x) for x in ifaces]:
            outer_of.append(f)
    P3 = _Cult2(S, range(ni), ifaces, [zanc[f] for f in outer_of],
                [xanc[f] for f in outer_of], sites)
    P5 = _Cult2(S, data, faces, zanc, xanc, sites)
    # --- d=3: inject, one round, double check
    P3.encode_t()
    P3.round(detect=True)
    P3.t_layer(undo=False)
    pool = cat + zanc[3:]     # checks borrow idle face ancillas beyond the 5 cat qubits

    def window_cats(sizes):
        out, k = [], 0
        for m in sizes:
            out.append(pool[k:k + m])
            k += m
        return out

    for c in window_cats(cats[0]):
        P3.cat_check(c)
    P3.t_layer(undo=True)
    # --- growth to d=5: the new data qubits on the two boundaries that carry
    # the kept logicals (Z_L on c == 0, X_L on r == c) start as Bell pairs
    # (PAPER.md:297-303), so Z_L and X_L of the d=5 code equal the d=3 ones
    # on the state; the other new qubits start in |0> or |+>, chosen to make
    # the most first-round faces deterministic
    new = [q for q, (r, c) in enumerate(sites) if r >= inner_rows]
    left = [q for q in data if sites[q][1] == 0]
    diag = [q for q in data if sites[q][0] == sites[q][1]]
    bell = [tuple(q for q in left if q in new), tuple(q for q in diag if q in new)]
    assert all(len(b) == 2 for b in bell)
    paired = {q for b in bell for q in b}
    free = [q for q in new if q not in paired]
    inner_ok = [not [q for q in face if q < ni] or
                sorted(q for q in face if q < ni) in [sorted(x) for x in ifaces]
                for face in faces]

    def det_part(face, basis_set):
        part = [q for q in face if q >= ni]
        for a, b in bell:
            if (a in part) != (b in part):
                return False
        return all(q in basis_set or q in paired for q in part)

    best = None
    for m in range(1 << len(free)):
        z_ = {q for i, q in enumerate(free) if not m >> i & 1}
        p_ = {q for i, q in enumerate(free) if m >> i & 1}
        zdet = [f for f, face in enumerate(faces) if inner_ok[f] and det_part(face, z_)]
        xdet = [f for f, face in enumerate(faces) if inner_ok[f] and det_part(face, p_)]
        key = len(zdet) + len(xdet)
        if best is None or key > best[0]:
            best = (key, sorted(p_), sorted(z_), zdet, xdet)
    _, plus_q, zero_q, zdet, xdet = best
    S.reset(zero_q)
    S.reset(plus_q, then=("H",))
    for a, b in bell:
        S.reset([a], then=("H",))
        S.reset([b])
        S.cx([(a, b)])
    det = {("z", f) for f in zdet} | {("x", f) for f in xdet}
    zm, xm = P5.round(detect=det)
    xerr = _pure_errors(len(data), faces + [left])[:len(faces)]
    zerr = _pure_errors(len(data), faces + [diag])[:len(faces)]
    for f in range(len(faces)):
        if f not in zdet:
            for q in xerr[f]:
                S.feedback("X", zm[f], q)
        if f not in xdet:
            for q in zerr[f]:
                S.feedback("Z", xm[f], q)
    P5.round(detect=True)
    # --- d=5 double check, rotated-frame logical -> observable
    P5.t_layer(undo=False)
    m1 = P5.observable()
    for c in window_cats(cats[1]):
        P5.cat_check(c)
    m2 = P5.observable(record=False)
    S.note("det", [m1, m2])
    P5.t_layer(undo=True)
    P5.round(detect=True)
    P5.round(detect=True)
    # --- second d=5 double check
    P5.t_layer(undo=False)
    for c in window_cats(cats[2]):
        P5.cat_check(c)
    return _finish(S, 264, data) if dd else parse_circuit(S.text())


def msc_d3_circuit(*, dd: bool = True, window_a=("fold3", "fold0"), window_b=("cat",)):
    """Magic-state cultivation at d=3 with the paper's Table 2 shape (15
    qubits, 137 gates, 81 two-qubit gates, 14 measurements, 22 T/T_DAG on
    the 7 data qubits, T-depth 4): |+_L> (H on the data, a Z round,
    Pauli-frame feedback), T_L by folding Z_L onto a data qubit (T, unfold),
    a check window (T_DAG/T layer, noiseless MPP of the rotated-frame
    logical into the observable, two fold checks of X^7 rooted at different
    qubits, undo layer), one stabilizer round, and a second window with a
    flagged cat check.  Same conventions and fault-tolerance checks as
    msc_d5_circuit; depth 51 (Table 2: 39)."""
    sites, faces = color_code_patch(3)
    data = list(range(7))
    zanc, xanc, cat = [7, 8, 9], [10, 11, 12], [13, 14]
    S = _Layers()
    P = _Cult2(S, data, faces, zanc, xanc, sites)
    P.prepare_plus()
    P.fold_inject(3)
    P.t_layer(undo=False)
    P.observable()

    def run(checks):
        for c in checks:
            if c == "cat":
                P.cat_check(cat)
            else:
                P.fold_check(int(c[4:]))

    run(window_a)
    P.t_layer(undo=True)
    P.round(detect=True)
    P.t_layer(undo=False)
    run(window_b)
    return _finish(S, 56, data) if dd else parse_circuit(S.text())
