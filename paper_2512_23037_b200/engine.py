"""Thin owner objects over the C ABI: ``Engine`` (one per device) and
``Program`` (a compiled op stream bound to the library).

All sampling goes through ``libgstab_sm100a.so``; there is no CPU path.
"""

from __future__ import annotations

import ctypes as ct
import threading

import numpy as np

from . import _lib
from .compiler import DeviceProgram, compile_program


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(ct.POINTER(ct.c_uint64))


class Program:
    """A ``DeviceProgram`` registered with the library (host copy; uploaded
    to an engine's device on first use)."""

    def __init__(self, dp: DeviceProgram):
        self.dp = dp
        lib = _lib.load()
        info = _lib.GsProgramInfo(dp.num_qubits, dp.num_measurements,
                                  dp.num_detectors, len(dp.obs_keys),
                                  dp.max_dim, dp.num_locations,
                                  dp.num_noise, dp.num_words, dp.noise_off,
                                  dp.wordpc_off, dp.geo_off, dp.geo_len,
                                  dp.noise_uniform, dp.acc_off)
        self._ops = np.ascontiguousarray(dp.ops, dtype=np.uint64)
        self._tables = np.ascontiguousarray(dp.tables, dtype=np.uint64)
        self._locs = np.ascontiguousarray(dp.locs, dtype=np.uint64)
        self._narrow = {}            # (device, flags) -> tuned narrow flag
        self._chi_form = {}          # (device, flags, capacity) -> 0 dense / 1 sparse (sampler)
        self.narrow_tuning = None    # probe times of the last tuning
        h = ct.c_void_p()
        _lib.check(lib.gs_program_create(ct.byref(info), _u64p(self._ops),
                                         self._ops.size, _u64p(self._tables),
                                         self._tables.size, _u64p(self._locs),
                                         self._locs.size, ct.byref(h)))
        self.handle = h

    # probe size of the narrow-limit tuning (narrow_flag)
    TUNE_SHOTS = 1 << 19

    def narrow_flag(self, engine: "Engine", flags: int, capacity: int) -> int:
        """``GS_NARROW_K5`` or 0: the narrow (lane-per-shot) chi dimension
        limit that ran this program faster on a probe of ``TUNE_SHOTS``
        shots (each setting warmed up, then timed on the device), cached per
        device and run flags.  Only the section split changes -- records
        and counters are identical either way (tests/test_gpu_parity.py) --
        so the choice is a pure performance decision: 5 moves the k = 5 ops
        of the MSC d=5 window into lane-per-shot sections (+10 % there) but
        costs narrow occupancy elsewhere (d=3: 4 is 30 % faster)."""
        if flags & _lib.GS_WIDE_ONLY:
            return 0
        cache = self._narrow
        key = self.tuning_key(engine, flags)
        if key in cache:
            return cache[key]
        if self.dp.max_dim < 5:
            cache[key] = 0          # every op is narrow at either limit
            return 0
        times = {}
        with engine.lock:
            for extra in (0, _lib.GS_NARROW_K5):
                par = Engine.params(0x7E57, 1 << 40, self.TUNE_SHOTS, capacity, flags | extra)
                engine.run_counters(self, par)            # warm-up (queues, occupancy)
                engine.run_counters(self, par)
                times[extra] = engine.last_kernel_ms
        best = min(times, key=times.get)
        cache[key] = best
        self.narrow_tuning = {"k4_ms": times[0], "k5_ms": times[_lib.GS_NARROW_K5],
                              "probe_shots": self.TUNE_SHOTS}
        return best

    @staticmethod
    def tuning_key(engine: "Engine", flags: int):
        return (engine.device, flags & (_lib.GS_RNG_PHILOX | _lib.GS_POSTSELECT |
                                        _lib.GS_CHI_GLOBAL | _lib.GS_CHI_SMEM |
                                        _lib.GS_CHI_BLOCK))

    def sections(self, flags: int = 0) -> int:
        """Narrow/wide sections (= sampling launches per chunk of shots)."""
        n = _lib.load().gs_program_sections(self.handle, flags)
        if n < 0:
            _lib.check(n)
        return n

    @classmethod
    def compile(cls, prog, **kw) -> "Program":
        return cls(compile_program(prog, **kw))

    @property
    def num_counters(self) -> int:
        return _lib.GS_C_PER_OBS + len(self.dp.obs_keys)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().gs_program_destroy(h)
            except Exception:
                pass
            self.handle = None


class Engine:
    """A device context of the sampler (streams, scratch, counters).

    The C engine's scratch is shared by its runs and the C ABI does not
    support concurrent calls on one engine (include/gstab_sm100.h); ctypes
    releases the GIL during a call, so every entry point here holds the
    engine's lock -- ``get_engine``'s process-wide engines are safe to use
    from several Python threads (their runs are serialised)."""

    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = ct.c_void_p()
        _lib.check(lib.gs_engine_create(int(device), ct.byref(h)))
        self.handle = h
        self.device = device
        self.lock = threading.RLock()

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.load().gs_engine_destroy(h)
            except Exception:
                pass
            self.handle = None

    @staticmethod
    def params(master_seed=0, shot_begin=0, shot_count=0, capacity=4096,
               flags=0, warps_per_block=0, blocks=0, seeds=None, chunk_shots=0):
        p = _lib.GsRunParams()
        p.master_seed = master_seed & 0xFFFFFFFFFFFFFFFF
        p.shot_begin = shot_begin
        p.shot_count = shot_count
        p.capacity = capacity
        p.flags = flags
        p.warps_per_block = warps_per_block
        p.blocks = blocks
        p.chunk_shots = chunk_shots
        p._seeds_keep = None
        if seeds is not None:
            s = np.ascontiguousarray(seeds, dtype=np.uint64)
            p._seeds_keep = s
            p.seeds = _u64p(s)
        return p

    # -- sampling -----------------------------------------------------

    def run_counters(self, prog: Program, params) -> np.ndarray:
        out = np.zeros(prog.num_counters, dtype=np.int64)
        with self.lock:
            _lib.check(_lib.load().gs_run_counters(
                self.handle, prog.handle, ct.byref(params),
                out.ctypes.data_as(ct.POINTER(ct.c_int64))))
        return out

    def run_counters_witness(self, prog: Program, params, cap: int):
        """Counters plus the global indices of (up to ``cap``) preserved
        shots with a flipped observable, sorted."""
        out = np.zeros(prog.num_counters, dtype=np.int64)
        wit = np.zeros(max(cap, 1), dtype=np.uint64)
        found = ct.c_uint32(0)
        with self.lock:
            _lib.check(_lib.load().gs_run_counters_witness(
                self.handle, prog.handle, ct.byref(params),
                out.ctypes.data_as(ct.POINTER(ct.c_int64)), wit.ctypes.data, cap,
                ct.byref(found)))
        return out, np.sort(wit[:min(cap, found.value)]), int(found.value)

    def run_counters_async(self, prog: Program, params, counters_dev_ptr: int,
                           stream_ptr: int) -> None:
        with self.lock:
            _lib.check(_lib.load().gs_run_counters_async(
                self.handle, prog.handle, ct.byref(params),
                ct.c_void_p(counters_dev_ptr), ct.c_void_p(stream_ptr)))

    def run_records(self, prog: Program, params):
        S = params.shot_count
        rw = (prog.dp.num_measurements + 63) // 64
        status = np.zeros(max(S, 1), dtype=np.uint8)
        aux = np.zeros(max(S, 1), dtype=np.int32)
        rec = np.zeros((max(S, 1), max(rw, 1)), dtype=np.uint64)
        obs = np.zeros(max(S, 1), dtype=np.uint64)
        with self.lock:
            _lib.check(_lib.load().gs_run_records(
                self.handle, prog.handle, ct.byref(params), status.ctypes.data,
                aux.ctypes.data, rec.ctypes.data, obs.ctypes.data))
        return status[:S], aux[:S], rec[:S, :rw], obs[:S]

    def dump(self, prog: Program, params):
        S = params.shot_count
        rw = (prog.dp.num_measurements + 63) // 64
        if prog.dp.max_dim > 24:
            raise ValueError("dumps hold 2^max_dim amplitudes per shot: compile with max_dim <= 24")
        stride = 1 << prog.dp.max_dim
        status = np.zeros(max(S, 1), dtype=np.uint8)
        aux = np.zeros(max(S, 1), dtype=np.int32)
        rec = np.zeros((max(S, 1), max(rw, 1)), dtype=np.uint64)
        obs = np.zeros(max(S, 1), dtype=np.uint64)
        sig = np.zeros((max(S, 1), 2), dtype=np.uint64)
        cv = np.zeros(max(S, 1), dtype=np.uint64)
        amps = np.zeros((max(S, 1), stride, 2), dtype=np.float64)
        dim = np.zeros(max(S, 1), dtype=np.uint32)
        with self.lock:
            _lib.check(_lib.load().gs_dump_shots(
                self.handle, prog.handle, ct.byref(params), status.ctypes.data,
                aux.ctypes.data, rec.ctypes.data, obs.ctypes.data, sig.ctypes.data,
                cv.ctypes.data, amps.ctypes.data, dim.ctypes.data))
        return {"status": status[:S], "aux": aux[:S], "rec": rec[:S, :rw],
                "obs": obs[:S], "sig": sig[:S], "c": cv[:S],
                "amps": amps[:S, :, 0] + 1j * amps[:S, :, 1], "dim": dim[:S]}

    # -- scratch ------------------------------------------------------

    def set_queue_budget(self, bytes_per_queue: int) -> None:
        """Inter-section queue budget per queue (0 = auto: min(8 GiB, 1/16
        of free device memory)); larger runs are chunked, same results."""
        with self.lock:
            _lib.check(_lib.load().gs_engine_set_queue_budget(self.handle, int(bytes_per_queue)))

    def trim(self) -> None:
        """Free the engine's scratch buffers (re-allocated on demand)."""
        with self.lock:
            _lib.check(_lib.load().gs_engine_trim(self.handle))

    # -- diagnostics --------------------------------------------------

    def section_stats(self, reset: bool = True) -> list:
        """Per-section statistics of the GS_SECTION_STATS runs since the last
        reset: shots in/out, SURVEY §8(d) model bytes, summed device time
        (CUDA events), launches, kind and first op."""
        cap = 256
        out = np.zeros(cap * _lib.GS_SEC_FIELDS, dtype=np.uint64)
        n = ct.c_uint32(0)
        with self.lock:
            _lib.check(_lib.load().gs_engine_section_stats(
                self.handle, out.ctypes.data, cap, ct.byref(n), int(reset)))
        rows = out[:min(n.value, cap) * _lib.GS_SEC_FIELDS].reshape(-1, _lib.GS_SEC_FIELDS)
        return [{"shots_in": int(r[_lib.GS_SEC_SHOTS_IN]),
                 "shots_out": int(r[_lib.GS_SEC_SHOTS_OUT]),
                 "model_bytes": int(r[_lib.GS_SEC_MODEL_BYTES]),
                 "device_ms": int(r[_lib.GS_SEC_DEVICE_NS]) * 1e-6,
                 "launches": int(r[_lib.GS_SEC_LAUNCHES]),
                 "kernel": "wide" if r[_lib.GS_SEC_WIDE] else "narrow",
                 "pc0": int(r[_lib.GS_SEC_PC0])} for r in rows]

    @property
    def launches(self) -> int:
        return int(_lib.load().gs_engine_launches(self.handle))

    @property
    def last_kernel_ms(self) -> float:
        return float(_lib.load().gs_engine_last_kernel_ms(self.handle))


_engines: dict[int, Engine] = {}
_engines_lock = threading.Lock()


def get_engine(device: int = 0) -> Engine:
    """Process-wide engine per device (created on first use)."""
    with _engines_lock:
        eng = _engines.get(device)
        if eng is None:
            eng = Engine(device)
            _engines[device] = eng
        return eng
