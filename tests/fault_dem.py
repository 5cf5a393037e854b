"""Fault analysis of noisy circuits on the Clifford proxy (T -> S, T_DAG ->
S_DAG; Gidney et al.'s proxy for cultivation): the
detector / observable signature of every elementary fault, by Pauli-frame
propagation of all faults at once (one bit column per single-qubit X or Z
fault inserted by a noise instruction).

Test / design infrastructure for the MSC workload generator (``msc.py``):
  * ``FaultModel(prog)``: signatures of the noise instructions of a noisy
    program (``apply_noise_model`` output);
  * ``.undetected_logical(order)``: fault sets of size <= order (1 or 2)
    that flip an observable without firing any detector (fault distance);
  * ``.sample(shots, rng)``: Monte Carlo discard / logical-error rates of the
    proxy under the program's channels (DEPOLARIZE1: X/Y/Z at p/3 each,
    DEPOLARIZE2: 15 Paulis at p/15, X_ERROR / Z_ERROR).

The proxy's detectors and observables are deterministic exactly when the T
circuit's are for stabilizer-state checks; discard rates of the T circuit
are measured with the sampler itself (tests/test_msc.py, GPU tests).
"""

from __future__ import annotations

import numpy as np

from paper_2512_23037_b200.circuit import PauliProduct, Rec

_PROXY = {"T": "S", "T_DAG": "S_DAG"}


class FaultModel:
    def __init__(self, prog):
        flat = list(prog.flat())
        n = prog.num_qubits
        # columns: (noise instruction index, kind, qubits, p) per location;
        # per target qubit two columns (X fault, Z fault)
        locs = []
        ncol = 0
        for i, ins in enumerate(flat):
            if ins.name in ("DEPOLARIZE1", "X_ERROR", "Z_ERROR"):
                for q in ins.targets:
                    locs.append((i, ins.name, (q,), float(ins.args[0]), (ncol,)))
                    ncol += 2
            elif ins.name == "DEPOLARIZE2":
                t = ins.targets
                for a, b in zip(t[0::2], t[1::2]):
                    locs.append((i, ins.name, (a, b), float(ins.args[0]), (ncol, ncol + 2)))
                    ncol += 4
        self.locs = locs
        self.ncol = ncol
        X = np.zeros((n, ncol), dtype=bool)
        Z = np.zeros((n, ncol), dtype=bool)
        by_instr = {}
        for li, (i, kind, qs, p, cols) in enumerate(locs):
            by_instr.setdefault(i, []).append((qs, cols))
        rec = []
        dets = []
        obs = {}
        for i, ins in enumerate(flat):
            name = _PROXY.get(ins.name, ins.name)
            tg = ins.targets
            if i in by_instr:
                for qs, cols in by_instr[i]:
                    for q, c in zip(qs, cols):
                        X[q, c] ^= True
                        Z[q, c + 1] ^= True
                continue
            if name not in ("DETECTOR", "OBSERVABLE_INCLUDE") and \
                    any(isinstance(t, Rec) for t in tg):      # feedback Pauli
                r, q = tg[0], tg[1]
                flip = rec[len(rec) + r.offset]
                if name in ("X", "CX"):
                    X[q] ^= flip
                elif name in ("Z", "CZ", "SWAP"):
                    Z[q] ^= flip
                else:
                    raise ValueError("feedback %s" % name)
                continue
            if name in ("H",):
                for q in tg:
                    X[q], Z[q] = Z[q].copy(), X[q].copy()
            elif name in ("S", "S_DAG", "H_XY", "H_NXY"):
                for q in tg:
                    Z[q] ^= X[q]
            elif name in ("I", "X", "Y", "Z", "TICK", "QUBIT_COORDS", "SHIFT_COORDS"):
                pass
            elif name == "CX":
                for c, t in zip(tg[0::2], tg[1::2]):
                    X[t] ^= X[c]
                    Z[c] ^= Z[t]
            elif name == "CZ":
                for a, b in zip(tg[0::2], tg[1::2]):
                    Z[a] ^= X[b]
                    Z[b] ^= X[a]
            elif name == "SWAP":
                for a, b in zip(tg[0::2], tg[1::2]):
                    X[[a, b]] = X[[b, a]]
                    Z[[a, b]] = Z[[b, a]]
            elif name in ("M", "MR"):
                for q in tg:
                    rec.append(X[q].copy())
                    if name == "MR":
                        X[q] = False
                        Z[q] = False
            elif name == "R":
                for q in tg:
                    X[q] = False
                    Z[q] = False
            elif name == "MPP":
                for pp in tg:
                    f = np.zeros(ncol, dtype=bool)
                    for q, letter in pp.terms:
                        if letter == "X":
                            f ^= Z[q]
                        elif letter == "Z":
                            f ^= X[q]
                        else:
                            f ^= X[q] ^ Z[q]
                    rec.append(f)
            elif name == "DETECTOR":
                d = np.zeros(ncol, dtype=bool)
                for r in tg:
                    d ^= rec[len(rec) + r.offset]
                dets.append(d)
            elif name == "OBSERVABLE_INCLUDE":
                k = int(ins.args[0]) if ins.args else 0
                o = obs.setdefault(k, np.zeros(ncol, dtype=bool))
                for r in tg:
                    o ^= rec[len(rec) + r.offset]
            else:
                raise ValueError("unsupported %s" % ins.name)
        self.num_detectors = len(dets)
        self.det = np.array(dets, dtype=bool).reshape(len(dets), ncol)   # (D, ncol)
        self.obs_keys = sorted(obs)
        self.obs = np.array([obs[k] for k in self.obs_keys], dtype=bool).reshape(-1, ncol)
        # packed column signatures: detectors as bytes, observables as int
        self._dpack = np.packbits(self.det, axis=0)                       # (Db, ncol)
        self._opack = np.zeros(ncol, dtype=np.int64)
        for j in range(self.obs.shape[0]):
            self._opack |= self.obs[j].astype(np.int64) << j

    # -- elementary faults ---------------------------------------------

    def faults(self):
        """Every elementary fault: (location index, Pauli label, column
        tuple whose XOR is its signature, probability)."""
        out = []
        for li, (i, kind, qs, p, cols) in enumerate(self.locs):
            c = cols[0]
            if kind == "X_ERROR":
                out.append((li, "X", (c,), p))
            elif kind == "Z_ERROR":
                out.append((li, "Z", (c + 1,), p))
            elif kind == "DEPOLARIZE1":
                out += [(li, "X", (c,), p / 3), (li, "Z", (c + 1,), p / 3),
                        (li, "Y", (c, c + 1), p / 3)]
            else:
                ca, cb = cols
                for k in range(1, 16):
                    la, lb = k & 3, k >> 2
                    cs = []
                    for l_, cc in ((la, ca), (lb, cb)):
                        if l_ in (1, 2):
                            cs.append(cc)
                        if l_ in (2, 3):
                            cs.append(cc + 1)
                    out.append((li, "IXYZ"[la] + "IXYZ"[lb], tuple(cs), p / 15))
        return out

    def signature(self, cols):
        d = np.zeros(self._dpack.shape[0], dtype=np.uint8)
        o = 0
        for c in cols:
            d ^= self._dpack[:, c]
            o ^= int(self._opack[c])
        return d.tobytes(), o

    def undetected_logical(self, order: int = 1, limit: int = 20):
        """Fault sets of size <= order that flip an observable and fire no
        detector (order 1 or 2); at most `limit` examples."""
        fl = self.faults()
        sigs = [self.signature(f[2]) for f in fl]
        zero = bytes(self._dpack.shape[0])
        bad = [(fl[i],) for i, (d, o) in enumerate(sigs) if o and d == zero][:limit]
        if order >= 2 and len(bad) < limit:
            groups = {}
            for i, (d, o) in enumerate(sigs):
                if d != zero:
                    groups.setdefault(d, {}).setdefault(o, i)
            for d, g in groups.items():
                if len(g) > 1:
                    ks = sorted(g)
                    bad.append((fl[g[ks[0]]], fl[g[ks[1]]]))
                    if len(bad) >= limit:
                        break
        return bad

    def sample(self, shots: int, seed: int = 0, batch: int = 200_000):
        """Monte Carlo (discard rate, logical error rate among preserved,
        preserved count, error count) of the proxy."""
        rng = np.random.default_rng(seed)
        fl = self.faults()
        # group elementary faults by location: fire location w.p. p, then pick
        loc_p = np.array([l[3] for l in self.locs])
        loc_faults = [[] for _ in self.locs]
        for f in fl:
            loc_faults[f[0]].append(f[2])
        dsig = []
        osig = []
        for fs in loc_faults:
            ds, os_ = [], []
            for cols in fs:
                d, o = self.signature(cols)
                ds.append(np.frombuffer(d, dtype=np.uint8))
                os_.append(o)
            dsig.append(np.array(ds))
            osig.append(np.array(os_, dtype=np.int64))
        nb = self._dpack.shape[0]
        disc = pres = err = 0
        done = 0
        while done < shots:
            b = min(batch, shots - done)
            D = np.zeros((b, nb), dtype=np.uint8)
            O = np.zeros(b, dtype=np.int64)
            for li, p in enumerate(loc_p):
                hit = np.nonzero(rng.random(b) < p)[0]
                if hit.size == 0:
                    continue
                pick = rng.integers(0, len(dsig[li]), size=hit.size)
                D[hit] ^= dsig[li][pick]
                O[hit] ^= osig[li][pick]
            fired = D.any(axis=1)
            disc += int(fired.sum())
            pres += int((~fired).sum())
            err += int(((O != 0) & ~fired).sum())
            done += b
        return {"discard_rate": disc / shots, "preserved": pres, "errors": err,
                "logical_error_rate": err / max(pres, 1)}
