"""Golden records for the headline MSC workloads, produced by the REAL
reference (/root/reference/pkg/src/gstab, numpy backend) in the build
container:

* ``msc_d5_records.npz``: the d=3 -> d=5 grown cultivation proxy
  (``msc_grown_circuit(5)``: 42 qubits, 72 T/T_DAG) under uniform
  depolarizing noise p=1e-3, post-selection on, 20,000 shots;
* ``msc_d3_records.npz``: the d=3 proxy (``msc_circuit(3)``), p=1e-3,
  20,000 shots.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_msc.py

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
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
os.environ.setdefault("GSTAB_BACKEND", "python")

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


def main():
    from paper_2512_23037_b200.msc import msc_circuit, msc_grown_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    which = sys.argv[1:] or ["d5", "d3"]
    if "d5" in which:
        make("msc_d5_records.npz",
             apply_noise_model(msc_grown_circuit(5), 1e-3).serialize())
    if "d3" in which:
        make("msc_d3_records.npz",
             apply_noise_model(msc_circuit(3), 1e-3).serialize())


if __name__ == "__main__":
    main()
