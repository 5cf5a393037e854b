"""Rebuild reference-layout state snapshots from device dumps.

A device dump of one shot is (sigma, c, dense amplitudes over 2^k
coordinates).  Together with the compiler's shot-invariant frame (x/z
tableau and coordinate basis B after the dumped instruction) it expands to
exactly the reference ``GenStabState`` layout: tableau rows ``xs``/``zs``
with phases ``ph = 2*sigma`` (ref tableau.py:45-56) and sorted unique
``idx``/``amp`` arrays of the nonzero amplitudes (ref state.py:52-58).
"""

from __future__ import annotations

import numpy as np


def coordinate_indices(basis, c: int, k: int) -> np.ndarray:
    """alpha(j) = c XOR (XOR_{i: bit i of j} B[i]) for j in [0, 2^k)."""
    idx = np.full(1 << k, c, dtype=np.uint64)
    js = np.arange(1 << k, dtype=np.uint64)
    for i, b in enumerate(basis[:k]):
        hit = ((js >> np.uint64(i)) & np.uint64(1)).astype(bool)
        idx[hit] ^= np.uint64(b)
    return idx


def reconstruct_state(dp, instr: int, sig: int, c: int, amps) -> dict:
    """Reference-layout snapshot after flat instruction ``instr``.

    ``dp`` must be compiled with ``keep_frames=True``; ``sig`` packs row
    signs with bit j = row j; ``amps`` holds the 2^k dense amplitudes.
    """
    n = dp.num_qubits
    xs, zs = dp.xz_after[instr]
    basis = dp.basis_after[instr]
    k = len(basis)
    amps = np.asarray(amps, dtype=np.complex128)[: 1 << k]
    idx = coordinate_indices(basis, c, k)
    nz = amps != 0
    idx, amps = idx[nz], amps[nz]
    order = np.argsort(idx, kind="stable")
    idx, amps = idx[order], amps[order]
    return {"xs": [int(v) for v in xs], "zs": [int(v) for v in zs],
            "ph": [2 * ((sig >> j) & 1) for j in range(2 * n)],
            "idx": [int(v) for v in idx],
            "amp": [[float(a.real), float(a.imag)] for a in amps]}
