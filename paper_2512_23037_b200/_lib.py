"""ctypes binding of ``libgstab_sm100a.so`` (C ABI: include/gstab_sm100.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing or no sm_100 device is present, every sampling call
raises ``EngineUnavailable``.
"""

from __future__ import annotations

import ctypes as ct
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libgstab_sm100a.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)

GS_POSTSELECT = 1
GS_RNG_PHILOX = 2
GS_CHI_GLOBAL = 4
GS_CHI_SMEM = 16
GS_CHI_BLOCK = 64
GS_WIDE_ONLY = 32
GS_SECTION_STATS = 128
GS_NARROW_K5 = 256
GS_BLOCK8 = 512
GS_SPARSE = 1024

# gs_engine_section_stats fields
GS_SEC_SHOTS_IN = 0
GS_SEC_SHOTS_OUT = 1
GS_SEC_MODEL_BYTES = 2
GS_SEC_DEVICE_NS = 3
GS_SEC_LAUNCHES = 4
GS_SEC_WIDE = 5
GS_SEC_PC0 = 6
GS_SEC_FIELDS = 7

GS_C_TOTAL = 0
GS_C_PRESERVED = 1
GS_C_DISCARDED = 2
GS_C_OVERFLOW = 3
GS_C_CORRUPT = 4
GS_C_UNSUPPORTED = 5
GS_C_ERROR_SHOTS = 6
GS_C_MODEL_BYTES = 7
GS_C_PER_OBS = 8

EXPORTED = (
    "gs_program_create", "gs_program_destroy", "gs_program_sections", "gs_engine_create",
    "gs_engine_destroy", "gs_run_counters", "gs_run_counters_witness",
    "gs_run_counters_async",
    "gs_run_records", "gs_dump_shots", "gs_anticommute_mask",
    "gs_conj_gate_rows", "gs_mul_rows", "gs_parity_pm", "gs_last_error",
    "gs_abi_version", "gs_engine_launches", "gs_engine_last_kernel_ms",
    "gs_engine_section_stats", "gs_engine_set_queue_budget", "gs_engine_trim",
)
ABI_VERSION = 3


class EngineUnavailable(RuntimeError):
    """The CUDA library or a B200 device is not available."""


class GsProgramInfo(ct.Structure):
    _fields_ = [("num_qubits", ct.c_uint32), ("num_measurements", ct.c_uint32),
                ("num_detectors", ct.c_uint32), ("num_obs", ct.c_uint32),
                ("max_dim", ct.c_uint32), ("num_locations", ct.c_uint32),
                ("num_noise", ct.c_uint32), ("num_words", ct.c_uint32),
                ("noise_off", ct.c_uint64), ("wordpc_off", ct.c_uint64),
                ("geo_off", ct.c_uint64), ("geo_len", ct.c_uint32),
                ("noise_uniform", ct.c_uint32), ("acc_off", ct.c_uint64)]


class GsRunParams(ct.Structure):
    _fields_ = [("master_seed", ct.c_uint64), ("shot_begin", ct.c_uint64),
                ("shot_count", ct.c_uint64), ("capacity", ct.c_uint64),
                ("flags", ct.c_uint32), ("warps_per_block", ct.c_uint32),
                ("blocks", ct.c_uint32), ("chunk_shots", ct.c_uint32),
                ("seeds", ct.POINTER(ct.c_uint64))]


_lib = None


def load(path: str | None = None):
    """Load and prototype the library (cached)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("GSTAB_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise EngineUnavailable(
            "%s not built; run __graft_entry__.build() (nvcc sm_100a)" % p)
    lib = ct.CDLL(p)
    vp = ct.c_void_p
    u64p = ct.POINTER(ct.c_uint64)
    lib.gs_last_error.restype = ct.c_char_p
    lib.gs_abi_version.restype = ct.c_int
    lib.gs_program_create.argtypes = [ct.POINTER(GsProgramInfo), u64p, ct.c_size_t,
                                      u64p, ct.c_size_t, u64p, ct.c_size_t,
                                      ct.POINTER(vp)]
    lib.gs_program_destroy.argtypes = [vp]
    lib.gs_program_sections.argtypes = [vp, ct.c_uint32]
    lib.gs_program_sections.restype = ct.c_int
    lib.gs_engine_create.argtypes = [ct.c_int, ct.POINTER(vp)]
    lib.gs_engine_destroy.argtypes = [vp]
    lib.gs_run_counters.argtypes = [vp, vp, ct.POINTER(GsRunParams),
                                    ct.POINTER(ct.c_int64)]
    lib.gs_run_counters_witness.argtypes = [vp, vp, ct.POINTER(GsRunParams),
                                            ct.POINTER(ct.c_int64), vp, ct.c_uint32,
                                            ct.POINTER(ct.c_uint32)]
    lib.gs_run_counters_async.argtypes = [vp, vp, ct.POINTER(GsRunParams),
                                          vp, vp]
    lib.gs_run_records.argtypes = [vp, vp, ct.POINTER(GsRunParams), vp, vp,
                                   vp, vp]
    lib.gs_dump_shots.argtypes = [vp, vp, ct.POINTER(GsRunParams), vp, vp, vp,
                                  vp, vp, vp, vp, vp]
    lib.gs_anticommute_mask.argtypes = [vp, vp, vp, ct.c_uint32, ct.c_uint32,
                                        vp, vp, vp]
    lib.gs_conj_gate_rows.argtypes = [vp, vp, vp, vp, ct.c_uint32, ct.c_uint32,
                                      vp, vp, vp]
    lib.gs_mul_rows.argtypes = [vp, vp, vp, vp, ct.c_uint32, ct.c_uint32, vp,
                                vp, vp, vp]
    lib.gs_parity_pm.argtypes = [vp, vp, ct.c_size_t, ct.c_uint64, vp]
    lib.gs_engine_launches.argtypes = [vp]
    lib.gs_engine_launches.restype = ct.c_uint64
    lib.gs_engine_last_kernel_ms.argtypes = [vp]
    lib.gs_engine_last_kernel_ms.restype = ct.c_double
    lib.gs_engine_section_stats.argtypes = [vp, vp, ct.c_uint32, ct.POINTER(ct.c_uint32),
                                            ct.c_int]
    lib.gs_engine_set_queue_budget.argtypes = [vp, ct.c_uint64]
    lib.gs_engine_trim.argtypes = [vp]
    if lib.gs_abi_version() != ABI_VERSION:
        raise EngineUnavailable("%s has ABI %d, expected %d (rebuild)"
                                % (p, lib.gs_abi_version(), ABI_VERSION))
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().gs_last_error().decode(errors="replace")
        raise EngineUnavailable("libgstab_sm100a error %d: %s" % (rc, msg)) \
            if rc in (-2, -4) else RuntimeError("libgstab_sm100a error %d: %s"
                                                % (rc, msg))
