"""Static-frame compiler: CircuitProgram -> device op stream.

Why a static frame:

* The tableau's x/z bits evolve identically in every shot: noise never
  touches the tableau (ref state.py:88-102), feedback only conjugates by
  Paulis (ref sampler.py:195-209), and pivot choice depends on x/z only
  (ref tableau.py:176-193).  Per shot the tableau is therefore just the
  2n sign bits ``sigma`` (phase = 2*sigma), updated by GF(2)-affine maps
  whose masks are computed here once.
* Every phase the reference derives from the tableau, ``xi0`` of
  ``pauli_action`` (ref tableau.py:117-146), is ``xi_s + 2*par(sigma & M)``
  for a static ``xi_s`` and mask ``M``.
* The amplitude support of every shot lies in ``c ^ span(B)`` for a basis
  ``B`` that is also shot-invariant: T gates add static betas, measurements
  remove one static dimension.  Only the offset ``c`` (a u64) and the dense
  amplitude array over the ``2^k`` coordinates are per shot.  Absent
  reference entries are exact zeros in the dense array, so every reference
  numeric step (merge, prune at 1e-12, pair-merge, filter, renormalise) maps
  1:1 onto a dense pass (ref state.py:104-129, 162-208, 294-311).
* RNG draw offsets are static per instruction (ref sampler.py:180-230,
  noise.py:60-101), so noise firing can be pre-scanned per shot.

Encoding: ``ops`` is a u64 stream of variable-length records
``[header, payload...]``; header = kind | len<<8 | k<<16 | flags<<24 |
flat_instruction<<32.  Noise instructions are *not* in the stream: the
``tables`` array holds, besides letter tables and record index lists, a noise
instruction table (insertion pc, location range, qubit mask, letter table)
and the insertion pc of every 32-location word of the fire bitset; ``locs``
holds two words (draw index | qubits | kind, threshold) per noise location.  The layout is mirrored
by ``csrc/gs_kernels.cu`` and by the CPU frame model in tests.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .circuit import (GATES_1Q, GATES_2Q, NOISE_OPS, PauliProduct, Rec)

MAX_QUBITS = 64
DEFAULT_MAX_DIM = 20

# op kinds
OP_END = 0
OP_T = 1
OP_MEAS = 2
OP_NOISE = 3
OP_FEEDBACK = 4
OP_DETECTOR = 5
OP_OBSERVABLE = 6
OP_GROW_LIMIT = 7

# T cases
T_DIAG, T_BUTTERFLY, T_GROW = 0, 1, 2
TF_FUSE = 1 << 4     # T flag: apply together with the next (BUTTERFLY) op
# T flag: BUTTERFLY / GROW with b' = b / phase purely imaginary (xi_s even):
# the wide kernel runs it as c v + i ss w with the global phase
# e^{+-i pi/8} counted instead of multiplied in (gs_sweeps.cuh t_mix);
# payload word 12: bit 0 = ss < 0, bit 1 = T_DAG
TF_RED = 1 << 5
# T flag: like TF_FUSE, but noise is inserted before the partner; the
# device fuses only when none of it fires for the shot
TF_FUSEQ = 1 << 6
# measurement cases
M_DET, M_PIVOT_SPAN, M_PIVOT_NOSPAN = 0, 1, 2
# measurement flags (bits of the header flag byte, above the 2-bit case and
# 2-bit xi_s)
MF_RECORD = 1 << 4
MF_FLIP = 1 << 5
MF_RESET = 1 << 6
MF_COMPACT = 1 << 7
# noise kinds in location words
NK_DEP1, NK_DEP2, NK_XERR, NK_ZERR = 0, 1, 2, 3
OWNER_LIMIT = 1 << 14     # noise instructions addressable from a location word
_NOISE_KIND = {"DEPOLARIZE1": NK_DEP1, "DEPOLARIZE2": NK_DEP2,
               "X_ERROR": NK_XERR, "Z_ERROR": NK_ZERR}

_LETTER_XZ = {"X": (1, 0), "Y": (1, 1), "Z": (0, 1)}

# 16-byte row component words + 8-byte amplitude index of the reference
# layout: bytes for the SURVEY §8(d) state-touch model
CHI_ENTRY_BYTES = 24


class CompileError(ValueError):
    pass


def _dbl_bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", float(v)))[0]


def _threshold(p: float) -> int:
    """Integer m-threshold so that (m * 2^-53 < p) <=> (m < T) for the
    53-bit draw m = u64 >> 11 (exact: scaling by 2^53 is exact)."""
    x = p * 9007199254740992.0
    if x >= 9007199254740992.0:
        return 1 << 53
    return int(math.ceil(x))


def geo_table(p_max: float, nlocs: int):
    """T[g] = ceil((1-p_max)^g * 2^53), g = 0..nlocs.  In Philox mode the gap
    between consecutive candidate noise locations is max{g : m < T[g]} for a
    53-bit draw m, i.e. P(gap >= g) = (1-p_max)^g (geometric skipping of a
    Bernoulli(p_max) process over the locations)."""
    q = 1.0 - p_max
    out = []
    for g in range(nlocs + 1):
        x = (q ** g) * 9007199254740992.0
        out.append(1 << 53 if x >= 9007199254740992.0 else int(math.ceil(x)))
    return out


def t_coefficients(dagger: bool):
    """T = a*I + b*Z on the branch basis, built with the reference's exact
    Python expressions so the constants are bit-identical
    (ref state.py:107-116)."""
    c = math.cos(math.pi / 8)
    s = math.sin(math.pi / 8)
    if dagger:
        phase = complex(math.cos(-math.pi / 8), math.sin(-math.pi / 8))
        return phase * c, 1j * phase * s
    phase = complex(math.cos(math.pi / 8), math.sin(math.pi / 8))
    return phase * c, -1j * phase * s


def _pmul(a, b):
    """Packed Pauli product (x, z, e) (ref pauli.py:141-155)."""
    x1, z1, e1 = a
    x2, z2, e2 = b
    x, z = x1 ^ x2, z1 ^ z2
    e = (e1 + e2 + 2 * (z1 & x2).bit_count() + (x1 & z1).bit_count()
         + (x2 & z2).bit_count() - (x & z).bit_count())
    return x, z, e & 3


def _iter_bits(m: int):
    while m:
        low = m & -m
        yield low.bit_length() - 1
        m ^= low


class _XZTableau:
    """Shot-invariant x/z part of the destabilizer/stabilizer tableau
    (rows 0..n-1 destabilizers, n..2n-1 stabilizers; ref tableau.py:45-56).
    Gate updates return the sign-flip row mask (bit j = row j) of
    ref _kernels_py.py:30-86."""

    def __init__(self, n: int):
        self.n = n
        self.x = np.zeros(2 * n, dtype=np.uint64)
        self.z = np.zeros(2 * n, dtype=np.uint64)
        for q in range(n):
            self.x[q] = np.uint64(1 << q)
            self.z[n + q] = np.uint64(1 << q)

    @staticmethod
    def _mask(flags: np.ndarray) -> int:
        return int.from_bytes(np.packbits(flags, bitorder="little").tobytes(),
                              "little")

    def gate(self, name: str, qs) -> int:
        xs, zs = self.x, self.z
        m1 = np.uint64(1 << qs[0])
        ax = (xs & m1) != 0
        az = (zs & m1) != 0
        if name == "I":
            return 0
        if name == "X":
            flip = az
        elif name == "Y":
            flip = ax ^ az
        elif name == "Z":
            flip = ax
        elif name == "H":
            flip = ax & az
            sw = (xs ^ zs) & m1
            xs ^= sw
            zs ^= sw
        elif name in ("S", "S_DAG", "H_XY", "H_NXY"):
            flip = {"S": ax & az, "S_DAG": ax & ~az, "H_XY": az & ~ax,
                    "H_NXY": ax | az}[name]
            zs ^= xs & m1
        else:
            m2 = np.uint64(1 << qs[1])
            bx = (xs & m2) != 0
            bz = (zs & m2) != 0
            if name == "CX":
                flip = ax & bz & ~(bx ^ az)
                xs[ax] ^= m2
                zs[bz] ^= m1
            elif name == "CZ":
                flip = ax & bx & (az ^ bz)
                zs[ax] ^= m2
                zs[bx] ^= m1
            elif name == "SWAP":
                both = m1 | m2
                for arr in (xs, zs):
                    d = ((arr & m1) != 0) ^ ((arr & m2) != 0)
                    arr[d] ^= both
                return 0
            else:
                raise CompileError("unknown Clifford %r" % name)
        return self._mask(flip)

    def anti(self, qx: int, qz: int, lo: int = 0, hi: int | None = None) -> int:
        hi = 2 * self.n if hi is None else hi
        par = (np.bitwise_count(self.x[lo:hi] & np.uint64(qz))
               + np.bitwise_count(self.z[lo:hi] & np.uint64(qx))) & 1
        return self._mask(par.astype(bool))

    def row(self, j: int):
        return int(self.x[j]), int(self.z[j])

    def action(self, qx: int, qz: int, qe: int):
        """Static part of pauli_action (ref tableau.py:117-146) with all row
        signs zero: returns (beta, delta, xi_s, sigma_mask) such that the
        per-shot xi0 = xi_s + 2*par(sigma & sigma_mask)."""
        n = self.n
        beta = self.anti(qx, qz, n, 2 * n)
        delta = self.anti(qx, qz, 0, n)
        d = (0, 0, 0)
        for k in _iter_bits(beta):
            d = _pmul(d, self.row(k) + (0,))
        r = _pmul((d[0], d[1], (-d[2]) & 3), (qx, qz, qe))
        gamma = self.anti(r[0], r[1], 0, n)
        m = (0, 0, 0)
        for k in _iter_bits(gamma):
            m = _pmul(m, self.row(n + k) + (0,))
        if (m[0], m[1]) != (r[0], r[1]):
            raise CompileError("stabilizer decomposition failed")
        return beta, delta, (r[2] - m[2]) & 3, beta | (gamma << n)

    def actions_1q(self, qmask: int):
        """``action`` of X_q and Z_q for every q in ``qmask`` (noise tables),
        from one conversion of the rows to Python ints: the anticommutation
        masks are column reads, and in a symplectic tableau the stabilizer
        coefficients of P are its anticommutations with the destabilizers
        (gamma = delta), checked below by rebuilding P.  Same results as
        ``action`` (tests/test_compiler_flags.py)."""
        n = self.n
        xr = [int(v) for v in self.x]
        zr = [int(v) for v in self.z]
        # column q of x / z as a 2n-bit row mask, for all 64 columns at once
        sh = np.arange(64, dtype=np.uint64)
        cols = []
        for a in (self.x, self.z):
            bits = ((a[None, :] >> sh[:, None]) & np.uint64(1)).astype(np.uint8)
            packed = np.packbits(bits, axis=1, bitorder="little")
            cols.append([int.from_bytes(row.tobytes(), "little") for row in packed])
        mask = (1 << n) - 1
        out = {}
        for q in _iter_bits(qmask):
            colx, colz = cols[0][q], cols[1][q]
            for lx, lz in ((1, 0), (0, 1)):
                qx, qz = lx << q, lz << q
                anti = colz if lx else colx          # rows anticommuting with X_q / Z_q
                beta, delta = anti >> n, anti & mask
                d = (0, 0, 0)
                for k in _iter_bits(beta):
                    d = _pmul(d, (xr[k], zr[k], 0))
                r = _pmul((d[0], d[1], (-d[2]) & 3), (qx, qz, 0))
                m = (0, 0, 0)
                for k in _iter_bits(delta):
                    m = _pmul(m, (xr[n + k], zr[n + k], 0))
                if (m[0], m[1]) != (r[0], r[1]):
                    raise CompileError("stabilizer decomposition failed")
                out[(q, lx)] = (beta, delta, (r[2] - m[2]) & 3, beta | (delta << n))
        return out

    def pivot(self, px: int, pz: int):
        """Measurement pivot (ref tableau.py:165-200).  Returns (t, sel, K):
        per shot, rows j in ``sel`` get sigma_j ^= sigma_{n+t} ^ K_j, then
        sigma_t <- old sigma_{n+t}, sigma_{n+t} <- outcome bit."""
        n = self.n
        am = self.anti(px, pz)
        beta = am >> n
        t = (beta & -beta).bit_length() - 1
        sx, sz = self.row(n + t)
        sel = am & ~((1 << (n + t)) | (1 << t))
        kmask = 0
        py = (sx & sz).bit_count()
        for j in _iter_bits(sel):
            xj, zj = self.row(j)
            x3, z3 = xj ^ sx, zj ^ sz
            e = (py + 2 * (zj & sx).bit_count() + (xj & zj).bit_count()
                 - (x3 & z3).bit_count()) & 3
            if e & 1:
                raise CompileError("non-Hermitian row product in pivot")
            if e:
                kmask |= 1 << j
            self.x[j], self.z[j] = np.uint64(x3), np.uint64(z3)
        self.x[t], self.z[t] = np.uint64(sx), np.uint64(sz)
        self.x[n + t], self.z[n + t] = np.uint64(px), np.uint64(pz)
        return t, sel, kmask


class _Span:
    """Linear span over GF(2) of the coordinate basis B (list of u64)."""

    def __init__(self):
        self.vecs: list[int] = []

    def coords(self, v: int):
        """(in_span, coordinate mask) with v = XOR_{i in mask} B[i]."""
        piv: list[tuple[int, int]] = []  # (reduced vector, combo)
        for i, b in enumerate(self.vecs):
            combo = 1 << i
            for pv, pc in piv:
                if b & (pv & -pv):
                    b ^= pv
                    combo ^= pc
            if b == 0:
                raise CompileError("basis became dependent")
            piv.append((b, combo))
        combo = 0
        for pv, pc in piv:
            if v & (pv & -pv):
                v ^= pv
                combo ^= pc
        return v == 0, combo

    def dots(self, w: int) -> int:
        """Bit i = parity(w & B[i])."""
        m = 0
        for i, b in enumerate(self.vecs):
            if (w & b).bit_count() & 1:
                m |= 1 << i
        return m

    def bit_col(self, t: int) -> int:
        m = 0
        for i, b in enumerate(self.vecs):
            if (b >> t) & 1:
                m |= 1 << i
        return m


@dataclass
class DeviceProgram:
    """Everything the device needs, plus host-side metadata used to decode
    records and dumps.  ``ops``/``tables``/``locs`` are little-endian u64."""
    num_qubits: int
    num_measurements: int
    num_detectors: int
    obs_keys: list
    max_dim: int
    num_locations: int
    num_draws: int
    ops: np.ndarray
    tables: np.ndarray
    locs: np.ndarray
    # per compiled op (same order as ops): flat instruction index, dim after
    op_instr: list = field(default_factory=list)
    # basis after each flat instruction (for dump reconstruction)
    basis_after: dict = field(default_factory=dict)
    xz_after: dict = field(default_factory=dict)
    truncated_at: int | None = None
    static_sign_bytes: int = 0
    noise_off: int = 0       # tables offset of the noise instruction table
    num_noise: int = 0
    wordpc_off: int = 0      # tables offset of the per-word insertion pcs
    num_words: int = 0
    geo_off: int = 0         # tables offset of the geometric gap table
    geo_len: int = 1         # its length (locations of the whole program + 1)
    noise_uniform: int = 1   # every location has p == p_max (no thinning)
    acc_off: int = 0         # tables offset of per-location p/p_max thresholds
    p_max: float = 0.0

    @property
    def nbytes(self) -> int:
        return int(self.ops.nbytes + self.tables.nbytes + self.locs.nbytes)


class _Emitter:
    def __init__(self):
        self.ops: list[int] = []
        self.tables: list[int] = []
        self.locs: list[int] = []
        self.op_instr: list[int] = []

    def op(self, kind, k, flags, instr, payload):
        n = 1 + len(payload)
        if n > 255:
            raise CompileError("op record too long")
        hdr = (kind | (n << 8) | ((k & 0xFF) << 16) | ((flags & 0xFF) << 24)
               | ((instr & 0xFFFFFFFF) << 32))
        self.ops.append(hdr)
        for w in payload:
            self.ops.append(int(w) & 0xFFFFFFFFFFFFFFFF)
        self.op_instr.append(instr)

    def table(self, words) -> int:
        off = len(self.tables)
        self.tables.extend(int(w) & 0xFFFFFFFFFFFFFFFF for w in words)
        return off


def compile_program(prog, *, max_dim: int = DEFAULT_MAX_DIM,
                    stop_after: int | None = None,
                    keep_frames: bool = False) -> DeviceProgram:
    """Lower a parsed program (this package's or the reference's
    ``CircuitProgram``) to the device op stream.

    ``stop_after`` truncates after that flat instruction (dump support);
    ``keep_frames`` records the basis and x/z tableau after every
    instruction so host code can rebuild reference-layout snapshots.
    """
    n = prog.num_qubits
    if not 1 <= n <= MAX_QUBITS:
        raise CompileError("num_qubits must be in 1..%d" % MAX_QUBITS)
    if max_dim > 30:
        raise CompileError("max_dim must be <= 30")
    nmask = (1 << n) - 1
    tab = _XZTableau(n)
    span = _Span()
    em = _Emitter()
    pending = 0            # folded Clifford sign flips not yet applied
    pending_gates = 0      # Clifford applications folded into ``pending``
    meas = 0
    draws = 0
    det_ordinal = 0
    obs_keys: list[int] = []
    max_k = 0
    basis_after = {}
    xz_after = {}
    truncated = None
    sign_bytes = 2 * ((2 * n + 7) // 8)
    total_static_sign = 0
    noise_ops: list = []

    def lohi(m):
        return m & nmask, (m >> n) & nmask

    def flush_words():
        nonlocal pending, pending_gates
        lo, hi = lohi(pending)
        cnt = pending_gates
        pending = 0
        pending_gates = 0
        return lo, hi, cnt

    def clifford(name, qs):
        nonlocal pending, pending_gates
        pending ^= tab.gate(name, qs)
        pending_gates += 1

    def emit_t(q, dagger, instr):
        nonlocal max_k, truncated
        beta, delta, xis, msig = tab.action(0, 1 << q, 0)
        k = len(span.vecs)
        dmask = span.dots(delta)
        a, b = t_coefficients(dagger)
        if beta == 0:
            if xis & 1:
                raise CompileError("imaginary Z eigenvalue in T update")
            case, cb = T_DIAG, 0
        else:
            ins, cb = span.coords(beta)
            case = T_BUTTERFLY if ins else T_GROW
            if not ins:
                cb = 0      # beta itself becomes basis vector k
        kind = OP_T
        if case == T_GROW and k + 1 > max_dim:
            kind = OP_GROW_LIMIT
        pre_lo, pre_hi, cnt = flush_words()
        m_lo, m_hi = lohi(msig)
        # b * i^{xi_s}: multiplying by +-1 / +-i only swaps and negates the
        # components, so this host constant is exact; the device negates it
        # when the per-shot sign parity adds 2 to xi0
        bxs = b * (1.0 + 0.0j, 1.0j, -1.0 + 0.0j, -1.0j)[xis]
        flags = case | (xis << 2)
        # b / phase = -+i s * i^{xi_s} = i ss with ss = -+s (T / T_DAG),
        # negated for xi_s = 2
        ss_neg = int((not dagger) ^ (xis == 2))
        if kind == OP_T and case != T_DIAG and xis % 2 == 0:
            flags |= TF_RED
        em.op(kind, k, flags, instr,
              [pre_lo, pre_hi, m_lo, m_hi, delta, cb | (dmask << 32),
               _dbl_bits(a.real), _dbl_bits(a.imag), _dbl_bits(bxs.real),
               _dbl_bits(bxs.imag), (cnt + 1) * sign_bytes,
               ss_neg | (int(dagger) << 1)])
        if kind == OP_GROW_LIMIT:
            truncated = instr
            return False
        if case == T_GROW:
            span.vecs.append(beta)
            max_k = max(max_k, k + 1)
        return True

    def emit_meas(px, pz, instr, record, flip_p, reset):
        nonlocal meas, draws
        beta, delta, xis, msig = tab.action(px, pz, 0)
        k = len(span.vecs)
        dmask = span.dots(delta)
        flags = 0
        vec = 0
        cb = 0
        t = 0
        i_sq = 0
        sel = kbits = 0
        tmask = 0
        if beta == 0:
            if xis & 1:
                raise CompileError("imaginary eigenvalue for Hermitian Pauli")
            case = M_DET
            if dmask:
                i_sq = dmask.bit_length() - 1
                vec = span.vecs[i_sq]
                flags |= MF_COMPACT
                span.vecs = [v ^ (vec if (dmask >> i) & 1 else 0)
                             for i, v in enumerate(span.vecs) if i != i_sq]
        else:
            t = (beta & -beta).bit_length() - 1
            tmask = span.bit_col(t)
            ins, cb = span.coords(beta)
            if not ins:
                cb = 0
            if ins:
                case = M_PIVOT_SPAN
                i_sq = tmask.bit_length() - 1
                vec = span.vecs[i_sq]
                flags |= MF_COMPACT
                span.vecs = [v ^ (vec if (tmask >> i) & 1 else 0)
                             for i, v in enumerate(span.vecs) if i != i_sq]
            else:
                case = M_PIVOT_NOSPAN
                vec = beta
                span.vecs = [v ^ (beta if (v >> t) & 1 else 0)
                             for v in span.vecs]
            t2, sel, kbits = tab.pivot(px, pz)
            assert t2 == t
        u_draw = draws
        draws += 1
        slot = 0
        if record:
            flags |= MF_RECORD
            slot = meas
            meas += 1
        flip_thr = 0
        if flip_p > 0.0:
            flags |= MF_FLIP
            flip_thr = _threshold(flip_p)
            draws += 1
        rst_lo = rst_hi = 0
        if reset:
            flags |= MF_RESET
            rst_lo, rst_hi = lohi(tab.gate("X", (reset[0],)))
        pre_lo, pre_hi, cnt = flush_words()
        m_lo, m_hi = lohi(msig)
        s_lo, s_hi = lohi(sel)
        k_lo, k_hi = lohi(kbits)
        em.op(OP_MEAS, k, case | (xis << 2) | flags, instr,
              [pre_lo, pre_hi, m_lo, m_hi, delta, dmask | (tmask << 32),
               cb | (t << 32) | (i_sq << 40), vec, s_lo, s_hi, k_lo, k_hi,
               slot | (u_draw << 32), flip_thr, rst_lo, rst_hi,
               (cnt + 1 + (1 if reset else 0)) * sign_bytes])

    def emit_noise(name, targets, p, instr):
        nonlocal draws
        kind = _NOISE_KIND[name]
        thr = _threshold(p)
        loc0 = len(em.locs) // 2
        # owning noise instruction index in bits 50..63 of every location
        # word (device O(1) owner lookup; the device bisects the noise table
        # when the program has more than OWNER_LIMIT noise instructions)
        kword = kind | ((len(noise_ops) << 2) if len(noise_ops) < OWNER_LIMIT else 0)
        if kind == NK_DEP2:
            pairs = list(zip(targets[0::2], targets[1::2]))
            for j, (a, b) in enumerate(pairs):
                em.locs += [(draws + 2 * j) | (a << 32) | (b << 40)
                            | (kword << 48), thr]
            draws += 2 * len(pairs)
        elif kind == NK_DEP1:
            for j, q in enumerate(targets):
                em.locs += [(draws + 2 * j) | (q << 32) | (kword << 48), thr]
            draws += 2 * len(targets)
        else:
            for j, q in enumerate(targets):
                em.locs += [(draws + j) | (q << 32) | (kword << 48), thr]
            draws += len(targets)
        nloc = len(em.locs) // 2 - loc0
        if nloc > 1024:
            raise CompileError("noise instruction with more than 1024 "
                               "locations is not supported")
        qmask = 0
        for q in targets:
            qmask |= 1 << q
        words = []
        acts = tab.actions_1q(qmask)
        for q in _iter_bits(qmask):
            for lx in (1, 0):
                beta, delta, xis, msig = acts[(q, lx)]
                # sign flips still pending at this point are absorbed into the
                # static phase: par((sigma^P) & M) = par(sigma&M) ^ par(P&M)
                xis = (xis + 2 * ((pending & msig).bit_count() & 1)) & 3
                m_lo, m_hi = lohi(msig)
                words += [beta, delta, m_lo, m_hi,
                          xis | (span.dots(delta) << 8)]
        off = em.table(words)
        # not an op-stream record: the device visits a noise instruction only
        # if one of its locations fired; it is applied right before the op at
        # `insert_pc` (the next op emitted)
        noise_ops.append((len(em.ops), nloc, loc0, qmask, off, instr))

    flat = list(prog.flat())
    # Philox-mode fire schedule constants over the WHOLE program (a
    # truncated compile must draw the same schedule): p_max and the number
    # of noise locations fix the geometric gap table
    loc_ps = []
    for ins in flat:
        if ins.name in NOISE_OPS:
            cnt_ = len(ins.targets) // 2 if ins.name == "DEPOLARIZE2" else len(ins.targets)
            loc_ps += [float(ins.args[0])] * cnt_
    p_max = max(loc_ps) if loc_ps else 0.0
    for i, ins in enumerate(flat):
        name = ins.name
        if name in ("TICK", "QUBIT_COORDS", "SHIFT_COORDS"):
            pass
        elif name in NOISE_OPS:
            emit_noise(name, tuple(ins.targets), float(ins.args[0]), i)
        elif name in ("T", "T_DAG"):
            ok = True
            for q in ins.targets:
                if not emit_t(q, name == "T_DAG", i):
                    ok = False
                    break
            if not ok:
                break
        elif name in GATES_2Q:
            tg = ins.targets
            for a, b in zip(tg[0::2], tg[1::2]):
                if isinstance(a, Rec):
                    fb = "X" if name == "CX" else "Z"
                    # conditional Pauli: sign flips only, applied on device
                    f_lo, f_hi = lohi(tab.gate(fb, (b,)))
                    em.op(OP_FEEDBACK, len(span.vecs), 0, i,
                          [meas + a.offset, f_lo, f_hi, sign_bytes])
                else:
                    clifford(name, (a, b))
        elif name in ("X", "Z") and any(isinstance(t, Rec) for t in ins.targets):
            tg = ins.targets
            for r, q in zip(tg[0::2], tg[1::2]):
                f_lo, f_hi = lohi(tab.gate(name, (q,)))
                em.op(OP_FEEDBACK, len(span.vecs), 0, i,
                      [meas + r.offset, f_lo, f_hi, sign_bytes])
        elif name in GATES_1Q:
            for q in ins.targets:
                clifford(name, (q,))
        elif name in ("M", "MR", "R"):
            for q in ins.targets:
                emit_meas(0, 1 << q, i, record=name != "R", flip_p=0.0,
                          reset=(q,) if name != "M" else None)
        elif name == "MPP":
            fp = float(ins.args[0]) if ins.args else 0.0
            for prod in ins.targets:
                px = pz = 0
                for q, letter in prod.terms:
                    bx, bz = _LETTER_XZ[letter]
                    px |= bx << q
                    pz |= bz << q
                emit_meas(px, pz, i, record=True, flip_p=fp, reset=None)
        elif name == "DETECTOR":
            idx = [meas + t.offset for t in ins.targets]
            off = em.table(idx)
            em.op(OP_DETECTOR, len(span.vecs), 0, i,
                  [det_ordinal | (len(idx) << 32), off])
            det_ordinal += 1
        elif name == "OBSERVABLE_INCLUDE":
            key = int(ins.args[0]) if ins.args else 0
            if key not in obs_keys:
                obs_keys.append(key)
            kid = obs_keys.index(key)
            if kid >= 64:
                raise CompileError("at most 64 distinct observable keys")
            idx = [meas + t.offset for t in ins.targets]
            off = em.table(idx)
            em.op(OP_OBSERVABLE, len(span.vecs), 0, i,
                  [kid | (len(idx) << 32), off])
        else:
            raise CompileError("unexecutable instruction %s" % name)
        if keep_frames:
            basis_after[i] = list(span.vecs)
            xz_after[i] = (tab.x.copy(), tab.z.copy())
        if stop_after is not None and i >= stop_after:
            break
    pre_lo, pre_hi, cnt = flush_words()
    em.op(OP_END, len(span.vecs), 0, 0xFFFFFFFF,
          [pre_lo, pre_hi, cnt * sign_bytes])
    _mark_fused_t_pairs(em.ops, {r[0] for r in noise_ops})
    # noise instruction table (4 words each) and, per 32-location word of the
    # fire bitset, the insertion pc of the instruction owning its first
    # location (the device scans a word only once execution reaches it)
    nloc_total = len(em.locs) // 2
    noise_off = len(em.tables)
    word_owner = []
    for rec_ in noise_ops:
        ipc, nl, l0, qm, off, ins_i = rec_
        em.tables += [ipc | (nl << 32), l0, qm, off]
    wordpc_off = len(em.tables)
    m = 0
    for w in range((nloc_total + 31) // 32):
        l = 32 * w
        while noise_ops[m][2] + noise_ops[m][1] <= l:
            m += 1
        em.tables.append(noise_ops[m][0])
    # geometric gap table for p_max (Philox mode) and, when the locations'
    # probabilities differ, per-location thinning thresholds p / p_max
    geo_off = len(em.tables)
    geo = geo_table(p_max, len(loc_ps)) if p_max > 0.0 else [1 << 53]
    em.tables += geo
    noise_uniform = int(all(q == p_max for q in loc_ps))
    acc_off = 0
    if not noise_uniform:
        acc_off = len(em.tables)
        em.tables += [_threshold(q / p_max) for q in loc_ps[:nloc_total]]
    return DeviceProgram(
        num_qubits=n, num_measurements=meas, num_detectors=det_ordinal,
        obs_keys=obs_keys, max_dim=max_k, num_locations=len(em.locs) // 2,
        num_draws=draws,
        ops=np.array(em.ops, dtype=np.uint64),
        tables=np.array(em.tables if em.tables else [0], dtype=np.uint64),
        locs=np.array(em.locs if em.locs else [0, 0], dtype=np.uint64),
        op_instr=em.op_instr, basis_after=basis_after, xz_after=xz_after,
        truncated_at=truncated, static_sign_bytes=total_static_sign,
        noise_off=noise_off, num_noise=len(noise_ops), wordpc_off=wordpc_off,
        num_words=(nloc_total + 31) // 32, geo_off=geo_off, geo_len=len(geo),
        noise_uniform=noise_uniform, acc_off=acc_off, p_max=p_max)


def _mark_fused_t_pairs(ops, noise_pcs):
    """Set TF_FUSE on a T BUTTERFLY op whose successor is a T BUTTERFLY of
    the same dimension with a different partner vector, no noise inserted
    between them and the same TF_RED form: the device applies both gates in
    one pass over 4-element groups (same arithmetic and pruning order as two
    passes).  With noise inserted before the successor the flag is TF_FUSEQ:
    the device fuses only when none of that noise fires for the shot (the
    Philox schedule or the scanned SplitMix fire bits say so), else runs the
    two gates separately.  Pairs
    are taken greedily left to right."""
    pc = 0
    prev = None
    while True:
        kind, ln, k, fl, _ = decode_header(ops[pc])
        if kind == OP_END:
            break
        if prev is not None and kind == OP_T and (fl & 3) == T_BUTTERFLY:
            ppc, pk, pcb, pred = prev
            cb = ops[pc + 6] & 0xFFFFFFFF
            if pk == k and pcb != cb and k >= 2 and pred == (fl & TF_RED):
                ops[ppc] |= (TF_FUSEQ if pc in noise_pcs else TF_FUSE) << 24
                prev = None
                pc += ln
                continue
        prev = (pc, k, ops[pc + 6] & 0xFFFFFFFF, fl & TF_RED) if (
            kind == OP_T and (fl & 3) == T_BUTTERFLY) else None
        pc += ln


def decode_header(w: int):
    return (w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, (w >> 24) & 0xFF,
            (w >> 32) & 0xFFFFFFFF)
