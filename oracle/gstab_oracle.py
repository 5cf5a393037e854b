"""CPU ORACLE — test infrastructure, NOT product code.

A from-scratch CPU restatement of the reference generalized-stabilizer shot
sampler (``/root/reference/pkg/src/gstab``), used only by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg as the checker and the timed CPU baseline.  The
product path (``paper_2512_23037_b200``) never imports this module.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference in
the build container and stores records / counters / state snapshots under
``tests/golden/``; ``tests/test_oracle.py`` checks this module against them
bit-for-bit (records, counters) and to 1e-12 (amplitudes).

Every function cites the reference lines it restates.  Numerics follow the
reference's numpy operation order (complex products, ``np.unique`` merge,
``np.add.at`` accumulation, sorted index order) so amplitudes normally come
out bit-identical.

RNG modes
  * ``"splitmix"`` — reference-compatible: seed = LE64(SHA1(LE64 master ||
    LE64 shot))[:8] (ref sampler.py:37-42); draw k (0-based) =
    mix(seed + (k+1)*0x9E3779B97F4A7C15) (ref sampler.py:45-61).
  * ``"philox"`` — production mode of the GPU engine (Philox4x32-10 keyed by
    the master seed, counter = (draw pair, shot)); defined in this repo, not
    in the reference, so parity is GPU-vs-this-restatement only.
"""

from __future__ import annotations

import hashlib
import math
import struct

import numpy as np

M64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15
PRUNE = 1e-12
I_POW = (1.0 + 0.0j, 1.0j, -1.0 + 0.0j, -1.0j)

GATE_CODE = {"I": 0, "X": 1, "Y": 2, "Z": 3, "H": 4, "S": 5, "S_DAG": 6,
             "H_XY": 7, "H_NXY": 8, "CX": 9, "CZ": 10, "SWAP": 11}
ONE_Q = ("I", "X", "Y", "Z", "H", "S", "S_DAG", "H_XY", "H_NXY")
TWO_Q = ("CX", "CZ", "SWAP")
NOISE = ("DEPOLARIZE1", "DEPOLARIZE2", "X_ERROR", "Z_ERROR")
LETTER_XZ = {"X": (1, 0), "Y": (1, 1), "Z": (0, 1)}
CODE_XZ = {1: (1, 0), 2: (1, 1), 3: (0, 1)}

PRESERVED, DISCARDED, OVERFLOW = "preserved", "discarded", "overflow"


class OracleOverflow(Exception):
    def __init__(self, needed, capacity):
        super().__init__("need %d entries, capacity %d" % (needed, capacity))
        self.needed = needed
        self.capacity = capacity


class OracleCorrupt(Exception):
    pass


# ----------------------------------------------------------------------
# RNG  (ref sampler.py:37-61)
# ----------------------------------------------------------------------

def sha1_seed(master: int, shot: int) -> int:
    d = hashlib.sha1(struct.pack("<QQ", master & M64, shot & M64)).digest()
    return struct.unpack("<Q", d[:8])[0]


def splitmix_mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix_u64(seed: int, k: int) -> int:
    """k-th output (0-based) of SplitMix64 started at ``seed``."""
    return splitmix_mix((seed + (k + 1) * GOLDEN_GAMMA) & M64)


_PH_M0, _PH_M1 = 0xD2511F53, 0xCD9E8D57
_PH_W0, _PH_W1 = 0x9E3779B9, 0xBB67AE85
M32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = _PH_M0 * c0
        p1 = _PH_M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0, p1 & M32,
                          (p0 >> 32) ^ c3 ^ k1, p0 & M32)
        k0 = (k0 + _PH_W0) & M32
        k1 = (k1 + _PH_W1) & M32
    return c0, c1, c2, c3


def philox_u64(master: int, shot: int, k: int) -> int:
    """Draw k of shot ``shot``: Philox4x32-10, key = master seed, counter =
    (k>>1 low, k>>1 high, shot low, shot high); even k takes words (0,1),
    odd k words (2,3)."""
    pair = k >> 1
    x = philox4x32_10((pair & M32, (pair >> 32) & M32, shot & M32,
                       (shot >> 32) & M32), (master & M32, (master >> 32) & M32))
    if k & 1:
        return x[2] | (x[3] << 32)
    return x[0] | (x[1] << 32)


class DrawStream:
    """Sequential uniform draws for one shot in either RNG mode."""

    __slots__ = ("mode", "seed", "master", "shot", "k")

    def __init__(self, mode, master, shot, seed=None):
        self.mode = mode
        self.master = master & M64
        self.shot = shot & M64
        self.seed = sha1_seed(master, shot) if seed is None else seed & M64
        self.k = 0

    def uniform(self) -> float:
        if self.mode == "philox":
            u = philox_u64(self.master, self.shot, self.k)
        else:
            u = splitmix_u64(self.seed, self.k)
        self.k += 1
        return (u >> 11) * (2.0 ** -53)


# ----------------------------------------------------------------------
# Pauli algebra  (ref pauli.py:141-160)
# ----------------------------------------------------------------------

def pmul(a, b):
    """Exact product of packed Paulis (x, z, e): X^x Z^z convention with the
    (-1)^{z1.x2} reordering sign, converted back to letters."""
    x1, z1, e1 = a
    x2, z2, e2 = b
    x, z = x1 ^ x2, z1 ^ z2
    e = (e1 + e2 + 2 * (z1 & x2).bit_count() + (x1 & z1).bit_count()
         + (x2 & z2).bit_count() - (x & z).bit_count())
    return x, z, e & 3


def anticommutes(x1, z1, x2, z2) -> bool:
    return ((x1 & z2).bit_count() + (z1 & x2).bit_count()) & 1 == 1


def _row_mask(xs, zs, qx, qz) -> int:
    """Bit j set iff row j anticommutes with (qx, qz) (ref _kernels_py.py:20)."""
    par = (np.bitwise_count(xs & np.uint64(qz))
           + np.bitwise_count(zs & np.uint64(qx))) & 1
    m = 0
    for j in np.flatnonzero(par):
        m |= 1 << int(j)
    return m


def _bits(mask):
    while mask:
        low = mask & -mask
        yield low.bit_length() - 1
        mask ^= low


def _pm_signs(idx, mask) -> np.ndarray:
    """(-1)^popcount(idx & mask) as float64 (ref _kernels_py.py:108-110)."""
    return 1.0 - 2.0 * (np.bitwise_count(idx & np.uint64(mask))
                        & np.uint64(1)).astype(np.float64)


# ----------------------------------------------------------------------
# per-shot state: tableau + sorted sparse amplitudes
# ----------------------------------------------------------------------

class ShotState:
    """Tableau rows 0..n-1 destabilizers, n..2n-1 stabilizers, phases in
    {0,2} (ref tableau.py:45-56); amplitudes as parallel sorted arrays
    (ref state.py:52-58)."""

    def __init__(self, n: int, capacity: int):
        self.n = n
        self.capacity = capacity
        self.x = np.zeros(2 * n, dtype=np.uint64)
        self.z = np.zeros(2 * n, dtype=np.uint64)
        self.ph = np.zeros(2 * n, dtype=np.uint8)
        for q in range(n):
            self.x[q] = np.uint64(1 << q)
            self.z[n + q] = np.uint64(1 << q)
        self.idx = np.zeros(1, dtype=np.uint64)
        self.amp = np.ones(1, dtype=np.complex128)

    # -- tableau ------------------------------------------------------

    def row(self, j):
        return int(self.x[j]), int(self.z[j]), int(self.ph[j])

    def clifford(self, gate: str, qs) -> None:
        """Row conjugation rules of ref _kernels_py.py:30-86 (tableau.py:83)."""
        xs, zs = self.x, self.z
        m1 = np.uint64(1 << qs[0])
        a_x = (xs & m1) != 0
        a_z = (zs & m1) != 0
        if gate == "I":
            return
        if gate == "X":
            flip = a_z
        elif gate == "Y":
            flip = a_x ^ a_z
        elif gate == "Z":
            flip = a_x
        elif gate == "H":
            flip = a_x & a_z
            sw = (xs ^ zs) & m1
            xs ^= sw
            zs ^= sw
        elif gate in ("S", "S_DAG", "H_XY", "H_NXY"):
            flip = {"S": a_x & a_z, "S_DAG": a_x & ~a_z,
                    "H_XY": a_z & ~a_x, "H_NXY": a_x | a_z}[gate]
            zs ^= xs & m1
        else:
            m2 = np.uint64(1 << qs[1])
            b_x = (xs & m2) != 0
            b_z = (zs & m2) != 0
            if gate == "CX":
                flip = a_x & b_z & ~(b_x ^ a_z)
                xs[a_x] ^= m2
                zs[b_z] ^= m1
            elif gate == "CZ":
                flip = a_x & b_x & (a_z ^ b_z)
                zs[a_x] ^= m2
                zs[b_x] ^= m1
            elif gate == "SWAP":
                both = m1 | m2
                for arr in (xs, zs):
                    d = ((arr & m1) != 0) ^ ((arr & m2) != 0)
                    arr[d] ^= both
                return
            else:
                raise ValueError("unknown gate %r" % gate)
        self.ph[flip] ^= 2

    def action(self, qx, qz, qe):
        """(beta, delta, xi0) of Pauli Q on the basis |b_alpha>
        (ref tableau.py:117-146)."""
        n = self.n
        beta = _row_mask(self.x[n:], self.z[n:], qx, qz)
        delta = _row_mask(self.x[:n], self.z[:n], qx, qz)
        d = (0, 0, 0)
        for k in _bits(beta):
            d = pmul(d, self.row(k))
        r = pmul((d[0], d[1], (-d[2]) & 3), (qx, qz, qe))
        gamma = _row_mask(self.x[:n], self.z[:n], r[0], r[1])
        m = (0, 0, 0)
        for k in _bits(gamma):
            m = pmul(m, self.row(n + k))
        if (m[0], m[1]) != (r[0], r[1]):
            raise RuntimeError("stabilizer decomposition failed")
        return beta, delta, (r[2] - m[2]) & 3

    def pivot(self, px, pz, pe, outcome: int) -> None:
        """Measurement collapse of the tableau (ref tableau.py:165-200)."""
        n = self.n
        am = _row_mask(self.x, self.z, px, pz)
        beta = am >> n
        t = (beta & -beta).bit_length() - 1
        sx, sz, se = self.row(n + t)
        am &= ~((1 << (n + t)) | (1 << t))
        if am:
            sel = np.zeros(2 * n, dtype=bool)
            for j in _bits(am):
                sel[j] = True
            xj, zj = self.x[sel], self.z[sel]
            x3, z3 = xj ^ np.uint64(sx), zj ^ np.uint64(sz)
            e = (self.ph[sel].astype(np.int64) + se + (sx & sz).bit_count()
                 + 2 * np.bitwise_count(zj & np.uint64(sx)).astype(np.int64)
                 + np.bitwise_count(xj & zj).astype(np.int64)
                 - np.bitwise_count(x3 & z3).astype(np.int64))
            self.x[sel], self.z[sel] = x3, z3
            self.ph[sel] = (e & 3).astype(np.uint8)
        self.x[t], self.z[t], self.ph[t] = sx, sz, se
        self.x[n + t], self.z[n + t] = px, pz
        self.ph[n + t] = (pe + (0 if outcome == 1 else 2)) & 3

    # -- amplitudes ---------------------------------------------------

    def pauli(self, ex, ez, ee) -> None:
        """Hermitian Pauli error: permute indices up to phase and re-sort
        (ref state.py:88-102, 289-292)."""
        if ex == 0 and ez == 0:
            if ee == 2:
                self.amp = -self.amp
            return
        beta, delta, xi0 = self.action(ex, ez, ee)
        ph = I_POW[xi0] * _pm_signs(self.idx, delta)
        self.idx = self.idx ^ np.uint64(beta)
        self.amp = self.amp * ph
        order = np.argsort(self.idx, kind="stable")
        self.idx, self.amp = self.idx[order], self.amp[order]

    def t_gate(self, q: int, dagger: bool) -> None:
        """T = a I + b Z_q branching with pair merge (ref state.py:104-129,
        294-306).  Coefficients are built exactly as the reference does."""
        c, s = math.cos(math.pi / 8), math.sin(math.pi / 8)
        if dagger:
            phase = complex(math.cos(-math.pi / 8), math.sin(-math.pi / 8))
            a, b = phase * c, 1j * phase * s
        else:
            phase = complex(math.cos(math.pi / 8), math.sin(math.pi / 8))
            a, b = phase * c, -1j * phase * s
        beta, delta, xi0 = self.action(0, 1 << q, 0)
        xi = I_POW[xi0] * _pm_signs(self.idx, delta)
        if beta == 0:
            if xi0 & 1:
                raise OracleCorrupt("imaginary Z eigenvalue in T update")
            self.amp = self.amp * (a + b * xi)
            return
        keys = np.concatenate([self.idx, self.idx ^ np.uint64(beta)])
        vals = np.concatenate([a * self.amp, b * xi * self.amp])
        uniq, inv = np.unique(keys, return_inverse=True)
        acc = np.zeros(len(uniq), dtype=np.complex128)
        np.add.at(acc, inv, vals)
        keep = np.abs(acc) > PRUNE
        uniq, acc = uniq[keep], acc[keep]
        if len(uniq) > self.capacity:
            raise OracleOverflow(len(uniq), self.capacity)
        if len(uniq) == 0:
            raise OracleCorrupt("all amplitudes pruned to zero")
        self.idx, self.amp = uniq, acc

    def measure(self, px, pz, pe, u: float) -> int:
        """Measure Hermitian Pauli; returns +1/-1 (ref state.py:133-208)."""
        beta, delta, xi0 = self.action(px, pz, pe)
        if beta == 0:
            if xi0 & 1:
                raise OracleCorrupt("imaginary eigenvalue for Hermitian Pauli")
            lam = I_POW[xi0].real * _pm_signs(self.idx, delta)
            plus = lam > 0
            pp = float(np.sum(np.abs(self.amp[plus]) ** 2))
            out = 1 if u < pp else -1
            if (pp if out == 1 else 1.0 - pp) < 1e-12:
                raise OracleCorrupt("selected measurement branch has ~zero weight")
            keep = plus if out == 1 else ~plus
            self.idx, self.amp = self.idx[keep], self.amp[keep]
        else:
            t = (beta & -beta).bit_length() - 1
            hi = ((self.idx >> np.uint64(t)) & np.uint64(1)) == 1
            reps = np.unique(np.where(hi, self.idx ^ np.uint64(beta), self.idx))
            part = reps ^ np.uint64(beta)
            v1, v2 = self._lookup(reps), self._lookup(part)
            xp = I_POW[xi0] * _pm_signs(part, delta)
            wp = v1 + xp * v2
            wm = v1 - xp * v2
            pp = float(0.5 * np.sum(np.abs(wp) ** 2))
            out = 1 if u < pp else -1
            if (pp if out == 1 else 1.0 - pp) < 1e-12:
                raise OracleCorrupt("selected measurement branch has ~zero weight")
            w = wp if out == 1 else wm
            keep = np.abs(w) > PRUNE
            self.pivot(px, pz, pe, out)
            self.idx, self.amp = reps[keep], w[keep]
        if len(self.idx) == 0:
            raise OracleCorrupt("post-measurement state is empty")
        self.amp = self.amp / math.sqrt(float(np.sum(np.abs(self.amp) ** 2)))
        return out

    def _lookup(self, keys):
        pos = np.minimum(np.searchsorted(self.idx, keys), len(self.idx) - 1)
        hit = self.idx[pos] == keys
        return np.where(hit, self.amp[pos], 0.0 + 0.0j)

    def snapshot(self):
        return {"xs": [int(v) for v in self.x], "zs": [int(v) for v in self.z],
                "ph": [int(v) for v in self.ph],
                "idx": [int(v) for v in self.idx],
                "amp": [(float(a.real), float(a.imag)) for a in self.amp]}


# ----------------------------------------------------------------------
# noise draws  (ref noise.py:60-101)
# ----------------------------------------------------------------------

def sample_error(kind, targets, p, rand):
    ex = ez = 0
    if kind == "DEPOLARIZE1":
        for q in targets:
            fire = rand() < p
            code = min(1 + int(rand() * 3), 3)
            if fire:
                bx, bz = CODE_XZ[code]
                ex |= bx << q
                ez |= bz << q
    elif kind == "DEPOLARIZE2":
        for i in range(0, len(targets), 2):
            a, b = targets[i], targets[i + 1]
            fire = rand() < p
            pick = min(1 + int(rand() * 15), 15)
            if fire:
                for qq, code in ((a, pick & 3), (b, pick >> 2)):
                    if code:
                        bx, bz = CODE_XZ[code]
                        ex |= bx << qq
                        ez |= bz << qq
    elif kind == "X_ERROR":
        for q in targets:
            if rand() < p:
                ex |= 1 << q
    elif kind == "Z_ERROR":
        for q in targets:
            if rand() < p:
                ez |= 1 << q
    return ex, ez


# ----------------------------------------------------------------------
# one shot  (ref sampler.py:169-276)
# ----------------------------------------------------------------------

def _is_rec(t):
    return hasattr(t, "offset")


def run_one_shot(flat, n, stream: DrawStream, capacity, postselect,
                 stop_after=None, snapshot=False):
    """Interpret the flattened program for one trajectory.

    Returns a dict with status, observables, discarded_detector,
    overflow_instruction, record (and the final state snapshot on request).
    ``stop_after`` truncates after that flat instruction index.
    """
    st = ShotState(n, capacity)
    rec: list[int] = []
    obs: dict[int, int] = {}
    det = -1
    status = PRESERVED
    extra = {}
    for i, ins in enumerate(flat):
        name = ins.name
        try:
            if name in ("TICK", "QUBIT_COORDS", "SHIFT_COORDS"):
                pass
            elif name in NOISE:
                ex, ez = sample_error(name, ins.targets, ins.args[0],
                                      stream.uniform)
                if ex or ez:
                    st.pauli(ex, ez, 0)
            elif name in ("T", "T_DAG"):
                for q in ins.targets:
                    st.t_gate(q, name == "T_DAG")
            elif name in TWO_Q:
                for a, b in zip(ins.targets[0::2], ins.targets[1::2]):
                    if _is_rec(a):
                        if rec[a.offset]:
                            st.clifford("X" if name == "CX" else "Z", (b,))
                    else:
                        st.clifford(name, (a, b))
            elif name in ("X", "Z") and any(_is_rec(t) for t in ins.targets):
                for r, q in zip(ins.targets[0::2], ins.targets[1::2]):
                    if rec[r.offset]:
                        st.clifford(name, (q,))
            elif name in ONE_Q:
                for q in ins.targets:
                    st.clifford(name, (q,))
            elif name in ("M", "MR", "R"):
                for q in ins.targets:
                    out = st.measure(0, 1 << q, 0, stream.uniform())
                    bit = 0 if out == 1 else 1
                    if name != "R":
                        rec.append(bit)
                    if name != "M" and bit:
                        st.clifford("X", (q,))
            elif name == "MPP":
                fp = ins.args[0] if ins.args else 0.0
                for prod in ins.targets:
                    px = pz = 0
                    for q, letter in prod.terms:
                        bx, bz = LETTER_XZ[letter]
                        px |= bx << q
                        pz |= bz << q
                    out = st.measure(px, pz, 0, stream.uniform())
                    bit = 0 if out == 1 else 1
                    if fp > 0.0 and stream.uniform() < fp:
                        bit ^= 1
                    rec.append(bit)
            elif name == "DETECTOR":
                det += 1
                par = 0
                for t in ins.targets:
                    par ^= rec[t.offset]
                if postselect and par:
                    status = DISCARDED
                    extra["discarded_detector"] = det
                    break
            elif name == "OBSERVABLE_INCLUDE":
                key = int(ins.args[0]) if ins.args else 0
                par = 0
                for t in ins.targets:
                    par ^= rec[t.offset]
                obs[key] = obs.get(key, 0) ^ par
            else:
                raise ValueError("unexecutable instruction %s" % name)
        except OracleOverflow:
            status = OVERFLOW
            extra["overflow_instruction"] = i
            break
        if stop_after is not None and i >= stop_after:
            break
    res = {"status": status,
           "observables": obs if status == PRESERVED else {},
           "discarded_detector": extra.get("discarded_detector"),
           "overflow_instruction": extra.get("overflow_instruction"),
           "record": rec}
    if snapshot:
        res["state"] = st.snapshot()
    return res


def run_shot_with_reruns(flat, n, mode, master, shot, capacity, doublings,
                         rerun, postselect, seed=None):
    """Overflow rerun loop with capacity doubling (ref sampler.py:306-316)."""
    attempts = doublings if rerun else 0
    cap = capacity
    while True:
        res = run_one_shot(flat, n, DrawStream(mode, master, shot, seed), cap,
                           postselect)
        if res["status"] != OVERFLOW or attempts == 0:
            return res
        attempts -= 1
        cap *= 2


def empty_counters():
    return {"total": 0, "preserved": 0, "discarded": 0, "overflow": 0,
            "error_shots": 0, "per_observable": {}}


def run_counters(prog, shots, master_seed=0, *, shot_begin=0, mode="splitmix",
                 entry_capacity=4096, postselect=False, rerun_on_overflow=True,
                 max_capacity_doublings=3):
    """Aggregate counters over shots [shot_begin, shot_begin+shots)
    (ref sampler.py:283-331)."""
    flat = list(prog.flat())
    n = prog.num_qubits
    out = empty_counters()
    for shot in range(shot_begin, shot_begin + shots):
        res = run_shot_with_reruns(flat, n, mode, master_seed, shot,
                                   entry_capacity, max_capacity_doublings,
                                   rerun_on_overflow, postselect)
        out["total"] += 1
        if res["status"] == PRESERVED:
            out["preserved"] += 1
            bad = False
            for k, v in res["observables"].items():
                if v:
                    out["per_observable"][k] = out["per_observable"].get(k, 0) + 1
                    bad = True
            out["error_shots"] += bad
        elif res["status"] == DISCARDED:
            out["discarded"] += 1
        else:
            out["overflow"] += 1
    return out


def merge_counters(a, b):
    out = {k: a[k] + b[k] for k in ("total", "preserved", "discarded",
                                    "overflow", "error_shots")}
    po = dict(a["per_observable"])
    for k, v in b["per_observable"].items():
        po[k] = po.get(k, 0) + v
    out["per_observable"] = po
    return out


def _pool_chunk(args):
    text, lo, hi, kw = args
    from paper_2512_23037_b200.circuit import parse_circuit  # host parser only
    return run_counters(parse_circuit(text), hi - lo, shot_begin=lo, **kw)


def run_counters_parallel(prog, shots, processes, **kw):
    """Process-pool fan-out over contiguous shot ranges (ref
    sampler.py:362-372 pattern); used for the CPU baseline."""
    import multiprocessing as mp
    text = prog.serialize()
    step = max(1, math.ceil(shots / processes))
    begin = kw.pop("shot_begin", 0)
    chunks = [(text, begin + a, begin + min(a + step, shots), kw)
              for a in range(0, shots, step)]
    ctx = mp.get_context("fork")
    with ctx.Pool(processes) as pool:
        parts = pool.map(_pool_chunk, chunks)
    out = empty_counters()
    for p in parts:
        out = merge_counters(out, p)
    return out
