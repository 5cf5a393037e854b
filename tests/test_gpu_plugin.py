"""GPU: the reference kernel-plugin interface (plugin.py over the batched
C-ABI kernels) against a numpy restatement of ref _kernels_py.py, mirroring
the reference's own kernel-parity tests (ref tests/test_kernels.py:29-95)."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2512_23037_b200 import plugin


def _rows(rng, count):
    xs = np.array([rng.getrandbits(64) for _ in range(count)], dtype=np.uint64)
    zs = np.array([rng.getrandbits(64) for _ in range(count)], dtype=np.uint64)
    ph = np.array([rng.choice((0, 2)) for _ in range(count)], dtype=np.uint8)
    return xs, zs, ph


def _anti(xs, zs, qx, qz):
    par = (np.bitwise_count(xs & np.uint64(qz)) + np.bitwise_count(zs & np.uint64(qx))) & 1
    return sum(1 << int(j) for j in np.flatnonzero(par))


def _conj(xs, zs, ph, code, m1, m2):
    # restatement of ref _kernels_py.py:30-86 (test oracle)
    m1 = np.uint64(m1)
    x1 = (xs & m1) != 0
    z1 = (zs & m1) != 0
    if code == 0:
        return
    if code == 1: flip = z1
    elif code == 2: flip = x1 ^ z1
    elif code == 3: flip = x1
    elif code == 4:
        flip = x1 & z1; t = (xs ^ zs) & m1; xs ^= t; zs ^= t
    elif code in (5, 6, 7, 8):
        flip = {5: x1 & z1, 6: x1 & ~z1, 7: z1 & ~x1, 8: x1 | z1}[code]
        zs ^= xs & m1
    else:
        m2 = np.uint64(m2)
        x2 = (xs & m2) != 0
        z2 = (zs & m2) != 0
        if code == 9:
            flip = x1 & z2 & ~(x2 ^ z1); xs[x1] ^= m2; zs[z2] ^= m1
        elif code == 10:
            flip = x1 & x2 & (z1 ^ z2); zs[x1] ^= m2; zs[x2] ^= m1
        else:
            for arr in (xs, zs):
                a1 = (arr & m1) != 0; a2 = (arr & m2) != 0
                arr[a1 ^ a2] ^= (m1 | m2)
            return
    ph[flip] ^= 2


def test_anticommute_mask():
    rng = random.Random(0)
    for _ in range(50):
        xs, zs, _ = _rows(rng, rng.randint(1, 128))
        qx, qz = rng.getrandbits(64), rng.getrandbits(64)
        assert plugin.anticommute_mask(xs, zs, qx, qz) == _anti(xs, zs, qx, qz)


@pytest.mark.parametrize("code", range(12))
def test_conj_gate_rows(code):
    rng = random.Random(code)
    for _ in range(20):
        xs, zs, ph = _rows(rng, rng.randint(1, 30))
        q1, q2 = rng.sample(range(64), 2)
        a = (xs.copy(), zs.copy(), ph.copy())
        b = (xs.copy(), zs.copy(), ph.copy())
        plugin.conj_gate_rows(*a, code, 1 << q1, 1 << q2)
        _conj(*b, code, 1 << q1, 1 << q2)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_mul_rows():
    rng = random.Random(5)
    for _ in range(50):
        n = rng.randint(1, 30)
        xs, zs, ph = _rows(rng, n)
        sel = np.array([rng.random() < 0.5 for _ in range(n)])
        px, pz, pe = rng.getrandbits(64), rng.getrandbits(64), rng.randrange(4)
        a = (xs.copy(), zs.copy(), ph.copy())
        plugin.mul_rows(*a, sel, px, pz, pe)
        xj, zj = xs[sel], zs[sel]
        x3, z3 = xj ^ np.uint64(px), zj ^ np.uint64(pz)
        e = (ph[sel].astype(np.int64) + pe + (px & pz).bit_count()
             + 2 * np.bitwise_count(zj & np.uint64(px)).astype(np.int64)
             + np.bitwise_count(xj & zj).astype(np.int64)
             - np.bitwise_count(x3 & z3).astype(np.int64))
        want_x, want_z, want_p = xs.copy(), zs.copy(), ph.copy()
        want_x[sel], want_z[sel], want_p[sel] = x3, z3, (e & 3).astype(np.uint8)
        assert np.array_equal(a[0], want_x) and np.array_equal(a[1], want_z)
        assert np.array_equal(a[2], want_p)


def test_parity_pm():
    rng = random.Random(6)
    for _ in range(30):
        idx = np.array([rng.getrandbits(64) for _ in range(rng.randint(1, 64))],
                       dtype=np.uint64)
        mask = rng.getrandbits(64)
        want = 1.0 - 2.0 * (np.bitwise_count(idx & np.uint64(mask)) & np.uint64(1)).astype(np.float64)
        assert np.array_equal(plugin.parity_pm(idx, mask), want)
