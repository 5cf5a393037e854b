"""The north star's amplitude bar: every chi coefficient within 1e-10
RELATIVE error (fp64) of the reference's, entry by entry."""

import numpy as np

CHI_RTOL = 1e-10


def _as_complex(a):
    """complex128 vector from complex data or [re, im] pairs (fixtures)."""
    a = np.asarray(a)
    if not np.iscomplexobj(a) and a.ndim == 2 and a.shape[1] == 2:
        return a[:, 0].astype(np.float64) + 1j * a[:, 1].astype(np.float64)
    return a.astype(np.complex128).reshape(-1)


def assert_chi_close(got, want, rtol=CHI_RTOL, context=None):
    """max_i |got_i - want_i| / |want_i| <= rtol over the (identical) support.

    Entries kept by the reference are nonzero (pruned at |v| <= 1e-12, ref
    state.py:294-306), so the per-entry ratio is defined; no absolute floor,
    so entries near the prune threshold are held to the same relative bar."""
    g, w = _as_complex(got), _as_complex(want)
    assert g.shape == w.shape, (context, g.shape, w.shape)
    if w.size == 0:
        return
    assert np.all(np.abs(w) > 0), context
    rel = np.abs(g - w) / np.abs(w)
    i = int(np.argmax(rel))
    assert rel[i] <= rtol, (context, "entry %d: got %r want %r rel %.3e" %
                            (i, g[i], w[i], rel[i]))
