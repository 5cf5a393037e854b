"""Golden records for the MSC workloads, produced by the REAL reference in
the build container: the noiseless circuit text is parsed and noised by the
reference itself (gstab.circuit.parse_circuit + gstab.noise.apply_noise_model,
ref noise.py:104-194) and sampled by its run_shot (oracle/_ref build, Cython
backend, bit-identical to the numpy one by ref tests/test_kernels.py):

* ``msc_d5_table2_records.npz``: msc_d5_circuit() (Table 2 d=5 shape),
  p=1e-3, post-selection, 20,000 shots;
* ``msc_d3_table2_records.npz``: msc_d3_circuit() (Table 2 d=3), p=1e-3;
* ``msc_d5_records.npz``: the d=3 -> d=5 grown proxy (msc_grown_circuit(5));
* ``msc_d3_records.npz``: the d=3 proxy (msc_circuit(3)).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_msc.py [names]

Each file holds the circuit text, master seed, statuses (1 preserved /
2 discarded / 3 overflow), the discarding detector index and the packed
record bits of every shot (bits after an early discard are 0).
"""

import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))   # oracle/build_ref.py
sys.path.insert(0, ROOT)

SHOTS = 20_000
MASTER = 20261017
_TEXT = None


def _init(text):
    global _TEXT
    _TEXT = text


def _chunk(bounds):
    from gstab.circuit import parse_circuit
    from gstab.sampler import ShotContext, derive_seed, run_shot
    prog = parse_circuit(_TEXT)
    ctx = ShotContext(prog.num_qubits, 4096)
    lo, hi = bounds
    st = np.zeros(hi - lo, dtype=np.uint8)
    det = np.full(hi - lo, -1, dtype=np.int32)
    obs = np.zeros(hi - lo, dtype=np.uint8)
    rec = np.zeros((hi - lo, prog.num_measurements), dtype=np.uint8)
    code = {"preserved": 1, "discarded": 2, "overflow": 3}
    for i, shot in enumerate(range(lo, hi)):
        ctx.reset(derive_seed(MASTER, shot))
        r = run_shot(prog, ctx, postselect=True, keep_record=True)
        st[i] = code[r.status.value]
        if r.discarded_detector is not None:
            det[i] = r.discarded_detector
        obs[i] = int(bool(r.observables.get(0, 0))) if r.observables else 0
        rec[i, :len(r.record)] = r.record
    return st, det, obs, rec


def make(name, text):
    step = 250
    bounds = [(a, min(a + step, SHOTS)) for a in range(0, SHOTS, step)]
    with mp.get_context("fork").Pool(os.cpu_count(), initializer=_init,
                                     initargs=(text,)) as pool:
        parts = pool.map(_chunk, bounds)
    st = np.concatenate([p[0] for p in parts])
    det = np.concatenate([p[1] for p in parts])
    obs = np.concatenate([p[2] for p in parts])
    rec = np.concatenate([p[3] for p in parts])
    np.savez_compressed(os.path.join(HERE, name), text=text, master=MASTER,
                        status=st, detector=det, observable=obs,
                        records=np.packbits(rec, axis=1, bitorder="little"),
                        num_measurements=rec.shape[1])
    print(name, "statuses:", np.bincount(st), "errors:", int(obs[st == 1].sum()))


def ref_noisy(prog, p):
    """The reference's own parse + uniform noise transform of the text."""
    from gstab.circuit import parse_circuit
    from gstab.noise import apply_noise_model
    return apply_noise_model(parse_circuit(prog.serialize()), p).serialize()


def main():
    from paper_2512_23037_b200 import msc
    jobs = {"d5t": ("msc_d5_table2_records.npz", msc.msc_d5_circuit),
            "d3t": ("msc_d3_table2_records.npz", msc.msc_d3_circuit),
            "d5": ("msc_d5_records.npz", lambda: msc.msc_grown_circuit(5)),
            "d3": ("msc_d3_records.npz", lambda: msc.msc_circuit(3))}
    for key in sys.argv[1:] or list(jobs):
        name, build = jobs[key]
        make(name, ref_noisy(build(), 1e-3))


if __name__ == "__main__":
    main()
