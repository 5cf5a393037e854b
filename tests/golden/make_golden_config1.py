"""Golden records for BASELINE config 1 at full size: all 10^5 shots of the
8-qubit random Clifford+T circuit (4 T, 2 mid-circuit M) under uniform
depolarizing noise p=1e-3, produced by the REAL reference
(/root/reference/pkg/src/gstab, numpy backend) in the build container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_config1.py

Writes tests/golden/config1_records.npz: circuit text, master seed,
statuses (1 preserved / 2 discarded / 3 overflow) and packed record bits.
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

SHOTS = 100_000
MASTER = 20260825
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
    rec = np.zeros((hi - lo, prog.num_measurements), dtype=np.uint8)
    code = {"preserved": 1, "discarded": 2, "overflow": 3}
    for i, shot in enumerate(range(lo, hi)):
        ctx.reset(derive_seed(MASTER, shot))
        r = run_shot(prog, ctx, postselect=True, keep_record=True)
        st[i] = code[r.status.value]
        rec[i, :len(r.record)] = r.record
    return st, rec


def main():
    from paper_2512_23037_b200.msc import config1_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    text = apply_noise_model(config1_circuit(1), 1e-3).serialize()
    step = 2500
    bounds = [(a, min(a + step, SHOTS)) for a in range(0, SHOTS, step)]
    with mp.get_context("fork").Pool(os.cpu_count(), initializer=_init,
                                     initargs=(text,)) as pool:
        parts = pool.map(_chunk, bounds)
    st = np.concatenate([p[0] for p in parts])
    rec = np.concatenate([p[1] for p in parts])
    np.savez_compressed(os.path.join(HERE, "config1_records.npz"), text=text,
                        master=MASTER, status=st,
                        records=np.packbits(rec, axis=1, bitorder="little"),
                        num_measurements=rec.shape[1])
    print("statuses:", np.bincount(st))


if __name__ == "__main__":
    main()
