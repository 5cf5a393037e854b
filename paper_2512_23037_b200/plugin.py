"""Kernel plugin module with the reference backend interface.

``gstab.backend`` (ref backend.py:13-53) selects a module exposing
``BACKEND_NAME``, ``anticommute_mask``, ``conj_gate_rows``, ``mul_rows`` and
``parity_pm`` (ref _kernels_py.py:20-110, _kernels.pyx:12-139).  This module
implements that interface on the B200 through the batched C-ABI kernels
(``gs_anticommute_mask`` ...), so a maintainer can register it next to the
reference's ``python``/``compiled`` backends.

These per-row calls are a unit-parity target: the production path
(``sampler.run_batch``) never calls them, because one shot-op per launch is
far below the launch-latency floor.  Batched variants (``*_batch``) take a
leading batch axis for callers that can amortise the launch.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .engine import get_engine

BACKEND_NAME = "b200"


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def anticommute_mask_batch(xs, zs, qx, qz, device: int = 0):
    """xs, zs: (batch, rows) u64 with rows <= 128; qx, qz: (batch,) ->
    list of Python int masks (bit j = row j anticommutes)."""
    xs = np.atleast_2d(_u64(xs))
    zs = np.atleast_2d(_u64(zs))
    b, rows = xs.shape
    out = np.zeros((b, 2), dtype=np.uint64)
    qx, qz = _u64(qx), _u64(qz)          # keep the buffers alive across the call
    _lib.check(_lib.load().gs_anticommute_mask(
        get_engine(device).handle, xs.ctypes.data, zs.ctypes.data, rows, b,
        qx.ctypes.data, qz.ctypes.data, out.ctypes.data))
    return [int(lo) | (int(hi) << 64) for lo, hi in out]


def anticommute_mask(xs, zs, qx: int, qz: int) -> int:
    """Packed bitmask of rows anticommuting with (qx, qz)
    (ref _kernels_py.py:20-27)."""
    if len(xs) == 0:
        return 0
    return anticommute_mask_batch(np.asarray(xs)[None], np.asarray(zs)[None],
                                  [qx], [qz])[0]


def conj_gate_rows_batch(xs, zs, ph, code, m1, m2, device: int = 0):
    """In-place batched Clifford conjugation; arrays shaped (batch, rows)."""
    b, rows = xs.shape
    code = np.ascontiguousarray(code, dtype=np.uint32)
    m1, m2 = _u64(m1), _u64(m2)
    _lib.check(_lib.load().gs_conj_gate_rows(
        get_engine(device).handle, xs.ctypes.data, zs.ctypes.data,
        ph.ctypes.data, rows, b, code.ctypes.data, m1.ctypes.data,
        m2.ctypes.data))


def conj_gate_rows(xs, zs, ph, code: int, m1: int, m2: int) -> None:
    """Conjugate every row by gate ``code`` (ref _kernels_py.py:30-86)."""
    if code not in range(12):
        raise ValueError("unknown gate code %r" % (code,))
    if len(xs) == 0:
        return
    x2, z2, p2 = xs[None].copy(), zs[None].copy(), ph[None].copy()
    conj_gate_rows_batch(x2, z2, p2, [code], [m1], [m2])
    xs[:], zs[:], ph[:] = x2[0], z2[0], p2[0]


def mul_rows_batch(xs, zs, ph, sel, px, pz, pe, device: int = 0):
    b, rows = xs.shape
    sel = np.ascontiguousarray(sel, dtype=np.uint8)
    px, pz = _u64(px), _u64(pz)
    pe = np.ascontiguousarray(pe, dtype=np.uint32)
    _lib.check(_lib.load().gs_mul_rows(
        get_engine(device).handle, xs.ctypes.data, zs.ctypes.data,
        ph.ctypes.data, rows, b, sel.ctypes.data, px.ctypes.data,
        pz.ctypes.data, pe.ctypes.data))


def mul_rows(xs, zs, ph, sel, px: int, pz: int, pe: int) -> None:
    """Right-multiply the selected rows by (px, pz, pe)
    (ref _kernels_py.py:89-105)."""
    if len(xs) == 0:
        return
    x2, z2, p2 = xs[None].copy(), zs[None].copy(), ph[None].copy()
    mul_rows_batch(x2, z2, p2, np.asarray(sel, dtype=np.uint8)[None],
                   [px], [pz], [pe & 3])
    xs[:], zs[:], ph[:] = x2[0], z2[0], p2[0]


def parity_pm(idx, mask: int, device: int = 0) -> np.ndarray:
    """(-1)^popcount(idx & mask) as float64 (ref _kernels_py.py:108-110)."""
    idx = _u64(idx)
    out = np.empty(idx.size, dtype=np.float64)
    _lib.check(_lib.load().gs_parity_pm(get_engine(device).handle,
                                        idx.ctypes.data, idx.size,
                                        int(mask) & 0xFFFFFFFFFFFFFFFF,
                                        out.ctypes.data))
    return out
