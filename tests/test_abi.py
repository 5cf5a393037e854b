"""CPU-side checks of the C-ABI library: it loads here (no GPU needed) and
exports every symbol include/gstab_sm100.h declares; engine creation fails
loudly without a B200."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gstab_sm100.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2512_23037_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    return _lib.load()


def test_header_declares_core_entry_points():
    names = _declared()
    for want in ("gs_program_create", "gs_engine_create", "gs_run_counters",
                 "gs_run_records", "gs_dump_shots", "gs_anticommute_mask",
                 "gs_conj_gate_rows", "gs_mul_rows", "gs_parity_pm",
                 "gs_last_error"):
        assert want in names


def test_library_exports_every_declared_symbol(lib):
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.gs_abi_version() == 3


def test_python_binding_lists_match_header():
    from paper_2512_23037_b200 import _lib
    assert sorted(_lib.EXPORTED) == _declared()


def test_engine_creation_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_23037_b200 import _lib
    from paper_2512_23037_b200.engine import Engine
    with pytest.raises(_lib.EngineUnavailable):
        Engine(0)


def test_sampling_without_gpu_raises(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_23037_b200 import SamplerConfig, parse_circuit, run_batch
    from paper_2512_23037_b200._lib import EngineUnavailable
    with pytest.raises(EngineUnavailable):
        run_batch(parse_circuit("H 0\nM 0\n"), SamplerConfig(shots=4))
