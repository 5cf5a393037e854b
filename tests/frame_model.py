"""CPU model of the device interpreter (test infrastructure).

Interprets the encoded op stream of ``compiler.compile_program`` exactly as
``csrc/gs_kernels.cu`` does, one shot at a time, so the compiler's static
frame (sign masks, basis bookkeeping, draw offsets) can be checked against
the oracle on CPU before any GPU time is spent.  Not used by the product.
"""

from __future__ import annotations

import math

import numpy as np

from oracle.gstab_oracle import M64, philox4x32_10, philox_u64, sha1_seed, splitmix_u64
from paper_2512_23037_b200 import compiler as C

I_POW = (1.0 + 0.0j, 1.0j, -1.0 + 0.0j, -1.0j)
RUNNING, PRESERVED, DISCARDED, OVERFLOW, CORRUPT, UNSUPPORTED = range(6)
STATUS_NAME = {PRESERVED: "preserved", DISCARDED: "discarded",
               OVERFLOW: "overflow", CORRUPT: "corrupt",
               UNSUPPORTED: "unsupported"}


def par(x: int) -> int:
    return x.bit_count() & 1


def _insert(jp: int, pos: int, bit: int) -> int:
    low = jp & ((1 << pos) - 1)
    return ((jp >> pos) << (pos + 1)) | (bit << pos) | low


def _abs2(v: complex) -> float:
    h = math.hypot(v.real, v.imag)
    return h * h


def _prune(v: complex) -> complex:
    return v if math.hypot(v.real, v.imag) > 1e-12 else 0j


def _f64(w: int) -> float:
    return float(np.array([w], dtype=np.uint64).view(np.float64)[0])


class Draws:
    def __init__(self, mode, master, shot, seed=None, dp=None):
        self.mode = mode
        self.master = master & M64
        self.shot = shot & M64
        self.seed = sha1_seed(master, shot) if seed is None else seed
        self.geo = None
        if mode == "philox" and dp is not None:
            self.geo = _Geo(dp, self.master, self.shot)

    def m53(self, k: int) -> int:
        if self.mode == "philox":
            return philox_u64(self.master, self.shot, k) >> 11
        return splitmix_u64(self.seed, k) >> 11

    def uniform(self, k: int) -> float:
        return self.m53(k) * (2.0 ** -53)


class _Geo:
    """Philox-mode fire schedule read from the compiled tables (gap table
    at geo_off, thinning thresholds at acc_off) -- the device's algorithm."""

    def __init__(self, dp, master, shot):
        t = dp.tables
        self.T = [int(w) for w in t[dp.geo_off: dp.geo_off + dp.geo_len]]
        self.acc = None if dp.noise_uniform else [int(w) for w in t[dp.acc_off: dp.acc_off + dp.num_locations]]
        self.key = (master & 0xFFFFFFFF, master >> 32)
        self.shot = shot
        self.j = 0
        self.pos = -1
        self.on = dp.p_max > 0.0
        self._adv(-1)

    def _blk(self, j, s):
        return philox4x32_10((j & 0xFFFFFFFF, s, self.shot & 0xFFFFFFFF, self.shot >> 32), self.key)

    def _adv(self, prev):
        if not self.on:
            self.pos = 1 << 62
            return
        x = self._blk(self.j, 1)
        m = (x[0] | (x[1] << 32)) >> 11
        self.pick = (x[2] | (x[3] << 32)) >> 11
        lo, hi = 0, len(self.T) - 1
        while lo < hi:
            mid = (lo + hi + 1) >> 1
            if m < self.T[mid]:
                lo = mid
            else:
                hi = mid - 1
        self.cand = self.j
        self.j += 1
        self.pos = prev + 1 + lo

    def at(self, loc):
        if self.pos != loc:
            return False, 0
        j, pick = self.cand, self.pick
        self._adv(loc)
        if self.acc is not None:
            x = self._blk(j, 2)
            if ((x[0] | (x[1] << 32)) >> 11) >= self.acc[loc]:
                return False, 0
        return True, pick


def run_shot(dp, mode, master, shot, capacity, postselect, seed=None,
             want_state=False):
    ops = [int(w) for w in dp.ops]
    tables = [int(w) for w in dp.tables]
    locs = [int(w) for w in dp.locs]
    n = dp.num_qubits
    nm = (1 << n) - 1
    rng = Draws(mode, master, shot, seed, dp)
    noise_at = {}
    for m in range(dp.num_noise):
        w = tables[dp.noise_off + 4 * m: dp.noise_off + 4 * m + 4]
        noise_at.setdefault(w[0] & 0xFFFFFFFF, []).append(
            (w[1], w[0] >> 32, w[2], w[3]))
    sig = 0                                   # bit j = row j
    c = 0
    A = np.zeros(1 << max(dp.max_dim, 0), dtype=np.complex128)
    A[0] = 1.0
    cnt = 1
    rec = [0] * max(dp.num_measurements, 1)
    obs = 0
    nrec = 0
    status = RUNNING
    aux = -1
    model_bytes = 0
    k_final = 0
    pc = 0

    def sig_xor(lo, hi):
        nonlocal sig
        sig ^= lo | (hi << n)

    def bit(j):
        return (sig >> j) & 1

    while status == RUNNING:
        hdr = ops[pc]
        kind, ln, k, flags, instr = C.decode_header(hdr)
        for loc0, nloc, qmask, off in noise_at.get(pc, ()):
            c, cnt_b = _apply_noise(A, 1 << k, rng, locs, tables, n, sig, c,
                                    loc0, nloc, qmask, off, cnt)
            model_bytes += cnt_b
        pay = ops[pc + 1: pc + ln]
        pc += ln
        size = 1 << k
        k_final = k
        if kind == C.OP_END:
            sig_xor(pay[0], pay[1])
            model_bytes += pay[2]
            status = PRESERVED
            break
        if kind in (C.OP_T, C.OP_GROW_LIMIT):
            sig_xor(pay[0], pay[1])
            M = pay[2] | (pay[3] << n)
            delta = pay[4]
            cb = pay[5] & 0xFFFFFFFF
            dmask = pay[5] >> 32
            a = complex(_f64(pay[6]), _f64(pay[7]))
            bxs = complex(_f64(pay[8]), _f64(pay[9]))     # b * i^{xi_s}
            model_bytes += pay[10]
            case = flags & 3
            flip = par(sig & M)
            bx0 = -bxs if flip else bxs
            bx = (bx0, -bx0)
            dc = par(delta & c)

            def s(j):
                return dc ^ par(j & dmask)

            if case == C.T_DIAG:
                f = (a + bx[0], a + bx[1])
                for j in range(size):
                    A[j] = A[j] * f[s(j)]
                model_bytes += 32 * cnt
                continue
            cin = cnt
            if kind == C.OP_GROW_LIMIT:
                tot = 0
                for j in range(size):
                    tot += _prune(a * A[j]) != 0
                    tot += _prune(bx[s(j)] * A[j]) != 0
                status = OVERFLOW if tot > capacity else UNSUPPORTED
                aux = instr
                break
            if case == C.T_BUTTERFLY:
                h = cb.bit_length() - 1
                for j in range(size):
                    if (j >> h) & 1:
                        continue
                    j1 = j ^ cb
                    v0, v1 = A[j], A[j1]
                    A[j] = _prune(a * v0 + bx[s(j1)] * v1)
                    A[j1] = _prune(a * v1 + bx[s(j)] * v0)
            else:
                for j in range(size):
                    v = A[j]
                    A[j] = _prune(a * v)
                    A[size + (j ^ cb)] = _prune(bx[s(j)] * v)
                size *= 2
            cnt = int(np.count_nonzero(A[:size]))
            model_bytes += C.CHI_ENTRY_BYTES * (cin + cnt)
            if cnt > capacity:
                status, aux = OVERFLOW, instr
                break
            if cnt == 0:
                status, aux = CORRUPT, instr
                break
            continue
        if kind == C.OP_MEAS:
            sig_xor(pay[0], pay[1])
            M = pay[2] | (pay[3] << n)
            delta = pay[4]
            dmask = pay[5] & 0xFFFFFFFF
            tmask = pay[5] >> 32
            cb = pay[6] & 0xFFFFFFFF
            t = (pay[6] >> 32) & 0xFF
            isq = (pay[6] >> 40) & 0xFF
            vec = pay[7]
            sel = pay[8] | (pay[9] << n)
            kb = pay[10] | (pay[11] << n)
            slot = pay[12] & 0xFFFFFFFF
            udraw = pay[12] >> 32
            flip_thr = pay[13]
            rst = pay[14] | (pay[15] << n)
            model_bytes += pay[16]
            case = flags & 3
            xi0 = ((flags >> 2 & 3) + 2 * par(sig & M)) & 3
            dc = par(delta & c)
            u = rng.uniform(udraw)
            cin = cnt
            if case == C.M_DET:
                neg0 = (xi0 >> 1) ^ dc
                sp = sm = 0.0
                for j in range(size):
                    if neg0 ^ par(j & dmask):
                        sm += _abs2(A[j])
                    else:
                        sp += _abs2(A[j])
                plus = u < sp
                chosen = sp if plus else 1.0 - sp
                if chosen < 1e-12:
                    status, aux = CORRUPT, instr
                    break
                want_neg = 0 if plus else 1
                r = 1.0 / math.sqrt(sp if plus else sm)
                if flags & C.MF_COMPACT:
                    tau = want_neg ^ neg0
                    newA = np.zeros_like(A)
                    for jp in range(size // 2):
                        base = _insert(jp, isq, 0)
                        x = tau ^ par(base & dmask)
                        newA[jp] = A[base | (x << isq)] * r
                    A = newA
                    c ^= vec if tau else 0
                    size //= 2
                else:
                    for j in range(size):
                        A[j] = A[j] * r if (neg0 ^ par(j & dmask)) == want_neg else 0j
                cnt = int(np.count_nonzero(A[:size]))
            else:
                I = I_POW[xi0]
                ct = (c >> t) & 1
                if case == C.M_PIVOT_SPAN:
                    half = size // 2
                    wp = np.zeros(half, dtype=np.complex128)
                    wm = np.zeros(half, dtype=np.complex128)
                    for jp in range(half):
                        base = _insert(jp, isq, 0)
                        x = ct ^ par(base & tmask)
                        rep = base | (x << isq)
                        part = rep ^ cb
                        xp = I * (-1.0 if dc ^ par(part & dmask) else 1.0)
                        pr = xp * A[part]
                        wp[jp] = A[rep] + pr
                        wm[jp] = A[rep] - pr
                    nsize = half
                else:
                    wp = np.zeros(size, dtype=np.complex128)
                    wm = np.zeros(size, dtype=np.complex128)
                    for j in range(size):
                        if ct ^ par(j & tmask):
                            xp = I * (-1.0 if dc ^ par(j & dmask) else 1.0)
                            pr = xp * A[j]
                            wp[j] = 0j + pr
                            wm[j] = 0j - pr
                        else:
                            wp[j] = A[j]
                            wm[j] = A[j]
                    nsize = size
                sp = 0.0
                for v in wp:
                    sp += _abs2(v)
                pp = 0.5 * sp
                plus = u < pp
                chosen = pp if plus else 1.0 - pp
                if chosen < 1e-12:
                    status, aux = CORRUPT, instr
                    break
                w = wp if plus else wm
                w = np.array([_prune(v) for v in w], dtype=np.complex128)
                sk = 0.0
                for v in w:
                    sk += _abs2(v)
                if sk == 0.0:
                    status, aux = CORRUPT, instr
                    break
                r = 1.0 / math.sqrt(sk)
                A = np.zeros_like(A)
                A[:nsize] = w * r
                c ^= vec if ct else 0
                size = nsize
                cnt = int(np.count_nonzero(A[:size]))
                # tableau sign update (pivot)
                v = bit(n + t)
                if v:
                    sig ^= sel
                sig ^= kb
                sig = (sig & ~(1 << t)) | (v << t)
                sig = (sig & ~(1 << (n + t))) | ((0 if plus else 1) << (n + t))
            model_bytes += C.CHI_ENTRY_BYTES * (cin + cnt)
            b_out = 0 if plus else 1
            rb = b_out
            if flags & C.MF_FLIP:
                if rng.m53(udraw + 1) < flip_thr:
                    rb ^= 1
            if flags & C.MF_RECORD:
                rec[slot] = rb
                nrec = slot + 1
            if (flags & C.MF_RESET) and b_out:
                sig ^= rst
            continue
        if kind == C.OP_FEEDBACK:
            if rec[pay[0]]:
                sig_xor(pay[1], pay[2])
                model_bytes += pay[3]
            continue
        if kind == C.OP_DETECTOR:
            ordinal = pay[0] & 0xFFFFFFFF
            cntx = pay[0] >> 32
            p = 0
            for w in tables[pay[1]: pay[1] + cntx]:
                p ^= rec[w]
            if postselect and p:
                status, aux = DISCARDED, ordinal
                break
            continue
        if kind == C.OP_OBSERVABLE:
            kid = pay[0] & 0xFFFFFFFF
            cntx = pay[0] >> 32
            p = 0
            for w in tables[pay[1]: pay[1] + cntx]:
                p ^= rec[w]
            obs ^= p << kid
            continue
        raise AssertionError("bad op kind %d" % kind)
    out = {"status": status, "aux": aux, "record": rec[:nrec],
           "obs": obs, "model_bytes": model_bytes}
    if want_state:
        out["sig"] = sig
        out["c"] = c
        out["A"] = A[: 1 << k_final].copy()
    return out


def _apply_noise(A, size, rng, locs, tables, n, sig, c, loc0, nloc, qmask,
                 off, cnt):
    """Sample one noise instruction's error and apply it (returns the new
    coset offset and the model bytes)."""
    ex = ez = 0
    for l in range(loc0, loc0 + nloc):
        w0, thr = locs[2 * l], locs[2 * l + 1]
        d = w0 & 0xFFFFFFFF
        qa = (w0 >> 32) & 0xFF
        qb = (w0 >> 40) & 0xFF
        nk = (w0 >> 48) & 3
        if rng.geo is not None:
            fired, pick53 = rng.geo.at(l)
            if not fired:
                continue
            u2 = pick53 * (2.0 ** -53)
        else:
            if rng.m53(d) >= thr:
                continue
            u2 = rng.uniform(d + 1) if nk in (C.NK_DEP1, C.NK_DEP2) else 0.0
        if nk == C.NK_DEP1:
            code = min(1 + int(u2 * 3), 3)
            ex |= (code in (1, 2)) << qa
            ez |= (code in (2, 3)) << qa
        elif nk == C.NK_DEP2:
            pick = min(1 + int(u2 * 15), 15)
            for qq, code in ((qa, pick & 3), (qb, pick >> 2)):
                ex |= (code in (1, 2)) << qq
                ez |= (code in (2, 3)) << qq
        elif nk == C.NK_XERR:
            ex |= 1 << qa
        else:
            ez |= 1 << qa
    if not (ex | ez):
        return c, 0
    beta = delt = xi = dm = 0
    for q in C._iter_bits(ex | ez):
        slot = ((qmask & ((1 << q) - 1))).bit_count()
        lets = []
        for li in range(2):
            base = off + 10 * slot + 5 * li
            lb, ld, mlo, mhi, xd = tables[base: base + 5]
            lx = ((xd & 3) + 2 * par(sig & (mlo | (mhi << n)))) & 3
            lets.append((lb, ld, lx, xd >> 8))
        X, Z = lets
        xb, zb = (ex >> q) & 1, (ez >> q) & 1
        if xb and zb:
            L = (X[0] ^ Z[0], X[1] ^ Z[1],
                 (1 + X[2] + Z[2] + 2 * par(X[1] & Z[0])) & 3, X[3] ^ Z[3])
        elif xb:
            L = X
        else:
            L = Z
        xi = (xi + L[2] + 2 * par(delt & L[0])) & 3
        beta ^= L[0]
        delt ^= L[1]
        dm ^= L[3]
    I = I_POW[xi]
    dc = par(delt & c)
    for j in range(size):
        A[j] = A[j] * (I * (-1.0 if dc ^ par(j & dm) else 1.0))
    return c ^ beta, 2 * C.CHI_ENTRY_BYTES * cnt + 2 * ((2 * n + 7) // 8)


def as_shot_result(dp, res):
    """Convert to the golden ShotResult dict layout."""
    st = res["status"]
    obs = {}
    if st == PRESERVED:
        obs = {str(k): (res["obs"] >> i) & 1 for i, k in enumerate(dp.obs_keys)}
        obs = dict(sorted(obs.items()))
    return {"status": STATUS_NAME[st],
            "observables": obs,
            "discarded_detector": res["aux"] if st == DISCARDED else None,
            "overflow_instruction": res["aux"] if st == OVERFLOW else None,
            "record": res["record"]}
