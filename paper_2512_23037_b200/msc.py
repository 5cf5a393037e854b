"""Workload generators for the BASELINE configs.

The paper's magic-state-cultivation circuits are not shipped with the
reference (tests/test_acceptance.py:41-42), so the d=3 / d=5
workloads are *proxies* built from the recipe of SURVEY.md Appendix B.2 on
the triangular 6.6.6 color code (same patch construction as the reference's
test helper, ref tests/conftest.py:98-114):

  prepare |+_L>      R all, H data, one Z-check round (MR, no detectors),
                     Pauli-frame feedback on a pure-error set per face
  inject             parity CX into an ancilla, T, uncompute, MR + DETECTOR
  T-check (x checks) T_DAG on sublattice (r+c)%3==0, T on (r+c)%3==2,
                     X^n parity on a flagged check ancilla (+ DETECTORs),
                     undo layer, then a Z and an X check round with DETECTORs
  final half-check   T layer + X^n parity into OBSERVABLE_INCLUDE(0)

Noiselessly every detector and the observable are deterministic (tested).
Deviations from the paper's Table 2 are reported by ``compute_stats`` and
documented in DESIGN.md: d=5 uses 2 full checks (96 T, T-depth 6) instead of
the paper's d=3->d=5 growth (72 T), so the proxy does *more* chi work.
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
