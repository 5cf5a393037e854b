"""The built reference (oracle/_ref, ``oracle/build_ref.py``) used as the timed
CPU baseline: it imports with its Cython backend and its counters equal the
oracle restatement's on the same workload and seeds (CPU only)."""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import build_ref  # noqa: E402
from oracle import gstab_oracle as orc  # noqa: E402
from paper_2512_23037_b200 import msc  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402

needs_ref = pytest.mark.skipif(not build_ref.available(),
                               reason="oracle/_ref not built")


@needs_ref
def test_reference_imports_with_compiled_backend():
    gstab = build_ref.import_reference()
    assert gstab.backend.name() == "compiled"


@needs_ref
@pytest.mark.parametrize("make,p,shots", [
    (lambda: msc.config1_circuit(1), 1e-3, 300),
    (lambda: msc.msc_circuit(3), 2e-3, 120),
])
def test_reference_counters_equal_oracle(make, p, shots):
    gstab = build_ref.import_reference()
    base = make()
    ref_prog = gstab.noise.apply_noise_model(
        gstab.circuit.parse_circuit(base.serialize()), p)
    cfg = gstab.sampler.SamplerConfig(shots=shots, master_seed=5, postselect=True,
                                      batch_size=64)
    st = gstab.sampler.run_batch(ref_prog, cfg)
    ours = orc.run_counters(apply_noise_model(base, p), shots, 5, postselect=True)
    assert (st.total_shots, st.preserved_shots, st.discarded_shots,
            st.overflow_count, st.logical_error_shots) == (
        ours["total"], ours["preserved"], ours["discarded"], ours["overflow"],
        ours["error_shots"])
    assert dict(st.logical_errors) == ours["per_observable"]
