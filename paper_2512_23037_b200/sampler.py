"""Drop-in shot-engine API (mirrors ``gstab.sampler``,
``/root/reference/pkg/src/gstab/sampler.py``) executed on the B200.

* ``SamplerConfig`` (ref sampler.py:80-99) + ``rng`` / ``device`` /
  ``max_dim`` fields.  ``threads`` is accepted for compatibility and
  ignored: parallelism is the GPU's shot-per-warp grid.
* ``run_batch(prog, cfg) -> RunStats`` (ref sampler.py:348-382): all
  ``cfg.shots`` shots in persistent-kernel launches; counters only.  The
  overflow rerun loop with capacity doubling (ref sampler.py:306-316) is one
  pass at the final capacity: a rerun replays identical draws, so the
  outcome equals a single run at ``entry_capacity * 2**doublings``.
* ``sample(prog, cfg) -> ShotBatch``: per-shot statuses, records and
  observables (the vectorised ``run_shot(..., keep_record=True)``).
* ``run_shot(prog, ctx, ...)`` with ``ShotContext`` (ref sampler.py:152-255)
  for single-trajectory callers.
* ``derive_seed``, ``ShotStatus``, ``ShotResult``, ``RunStats.as_dict``
  schema, ``bayes_interval`` and ``throughput_bench`` as in the reference.

RNG: ``rng="splitmix"`` (default) reproduces the reference's SHA-1 seeds and
SplitMix64 stream bit-for-bit; ``rng="philox"`` uses counter-based
Philox4x32-10 streams (production mode, statistically equivalent).
"""

from __future__ import annotations

import enum
import hashlib
import math
import struct
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .engine import Engine, Program, get_engine

_M64 = (1 << 64) - 1
_WAVE = 1 << 22         # default shots resident per launch (batch_size=None)


class CorruptStateError(RuntimeError):
    """A shot hit a ~zero-weight measurement branch (ref state.py:40-41)."""


class UnsupportedCircuitError(RuntimeError):
    """A shot reached an op whose static chi dimension exceeds the program's
    dimension limit while its support still fit the entry capacity.  The
    static frame keeps every T coordinate of the
    shot-invariant span until a measurement removes it, so a circuit whose T
    gates cancel back to a small support (e.g. many ``H q; T q; T_DAG q; H q``
    blocks on distinct qubits) needs a dense chi over the whole span where
    the reference's sparse map holds one entry (ref state.py:294-306).  With
    ``chi="auto"`` (default) such runs switch to the sparse form (GS_SPARSE,
    up to 30 span dimensions, effective capacity <= 2^16), so this is raised
    only with ``chi="dense"``, beyond those limits, or with an explicit
    ``max_dim`` -- never silently."""

    def __init__(self, shots: int, instruction: int | None, limit: int | None):
        self.shots = shots
        self.instruction = instruction
        self.limit = limit
        at = "" if instruction is None else " at flat instruction %d" % instruction
        lim = "" if limit is None else " %d" % limit
        super().__init__(
            "%d shot(s) reached a chi dimension above the limit%s%s while within the entry "
            "capacity (the static frame keeps cancelled T coordinates until a measurement "
            "drops them; use SamplerConfig(chi='sparse') or raise max_dim)" % (shots, lim, at))


class CapacityError(RuntimeError):
    """Raised by ``run_shot`` callers expecting the reference exception type;
    batch APIs report overflow as a per-shot status instead."""


def derive_seed(master_seed: int, shot_index: int) -> int:
    """LE64 of the first 8 bytes of SHA-1(LE64 master || LE64 shot)
    (ref sampler.py:37-42).  The device computes the same on the fly."""
    d = hashlib.sha1(struct.pack("<QQ", master_seed & _M64,
                                 shot_index & _M64)).digest()
    return struct.unpack("<Q", d[:8])[0]


class ShotStatus(enum.Enum):
    RUNNING = "running"
    PRESERVED = "preserved"
    DISCARDED = "discarded"
    OVERFLOW = "overflow"


_STATUS = {1: ShotStatus.PRESERVED, 2: ShotStatus.DISCARDED,
           3: ShotStatus.OVERFLOW}


@dataclass
class ShotResult:
    status: ShotStatus
    observables: dict = field(default_factory=dict)
    discarded_detector: int | None = None
    overflow_instruction: int | None = None
    record: list | None = None


@dataclass
class SamplerConfig:
    shots: int
    master_seed: int = 0
    # shots resident per launch (one wave = one gs_run_counters call, the
    # GPU analogue of the reference's waves, ref sampler.py:348-382);
    # None = 2^22: saturates a B200 (Fig. 4 analogue, profiles/
    # fig4_batch_size_r02u.csv: 36.6 M shots/s at 2^20, 37.0 M at 2^22 on the
    # d=5 workload) with 1/4 of the section-queue memory of 2^24
    batch_size: int | None = None
    entry_capacity: int = 4096
    threads: int = 1
    postselect: bool = False
    rerun_on_overflow: bool = True
    max_capacity_doublings: int = 3
    rng: str = "splitmix"
    device: int = 0
    max_dim: int | None = None   # chi dimension limit (auto from capacity)
    # chi form: "dense" (lane / warp / block per shot over 2^k coordinates),
    # "sparse" (warp per shot over the nonzero entries, GS_SPARSE), "auto"
    # (dense; sparse when the dense program would hit its dimension limit)
    chi: str = "auto"

    def __post_init__(self):
        if self.shots < 0:
            raise ValueError("shots must be >= 0")
        if self.batch_size is not None and self.batch_size < 1:
            raise ValueError("batch_size must be >= 1")
        if self.entry_capacity < 2:
            raise ValueError("entry_capacity must be >= 2")
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.rng not in ("splitmix", "philox"):
            raise ValueError("rng must be 'splitmix' or 'philox'")
        if self.chi not in ("auto", "dense", "sparse"):
            raise ValueError("chi must be 'auto', 'dense' or 'sparse'")

    @property
    def dim_limit(self) -> int:
        """Largest chi dimension the device buffers hold: a shot whose
        support needs more coordinates than 2^limit while staying within the
        entry capacity reports UNSUPPORTED (never silently wrong)."""
        if self.max_dim is not None:
            return self.max_dim
        return min(24, max(1, (self.effective_capacity - 1).bit_length() + 5))

    @property
    def wave_shots(self) -> int:
        return _WAVE if self.batch_size is None else int(self.batch_size)

    @property
    def effective_capacity(self) -> int:
        d = self.max_capacity_doublings if self.rerun_on_overflow else 0
        return self.entry_capacity << max(d, 0)

    def run_flags(self) -> int:
        f = 0
        if self.postselect:
            f |= _lib.GS_POSTSELECT
        if self.rng == "philox":
            f |= _lib.GS_RNG_PHILOX
        return f


@dataclass
class RunStats:
    total_shots: int
    preserved_shots: int
    discarded_shots: int
    overflow_count: int
    logical_errors: dict
    logical_error_shots: int
    wall_time_s: float
    bayes_factor: float = 1000.0
    # B200 extras (not in as_dict, which keeps the reference schema)
    device_time_s: float = 0.0
    model_bytes: int = 0
    witnesses: list = field(default_factory=list)   # shot indices (see run_batch)

    @property
    def discard_rate(self) -> float:
        return self.discarded_shots / self.total_shots if self.total_shots else 0.0

    @property
    def logical_error_rate(self) -> float:
        return (self.logical_error_shots / self.preserved_shots
                if self.preserved_shots else 0.0)

    @property
    def bayes_interval(self):
        if self.preserved_shots == 0:
            return (0.0, 1.0)
        return bayes_interval(self.logical_error_shots, self.preserved_shots,
                              self.bayes_factor)

    @property
    def throughput(self) -> float:
        return self.total_shots / self.wall_time_s if self.wall_time_s > 0 else 0.0

    def as_dict(self) -> dict:
        lo, hi = self.bayes_interval
        return {
            "total_shots": self.total_shots,
            "preserved_shots": self.preserved_shots,
            "discarded_shots": self.discarded_shots,
            "overflow_count": self.overflow_count,
            "discard_rate": self.discard_rate,
            "logical_errors": {str(k): v for k, v in
                               sorted(self.logical_errors.items())},
            "logical_error_shots": self.logical_error_shots,
            "logical_error_rate": self.logical_error_rate,
            "bayes_lo": lo,
            "bayes_hi": hi,
            "wall_time_s": self.wall_time_s,
            "throughput": self.throughput,
        }

    def device_dict(self) -> dict:
        return {"device_time_s": self.device_time_s,
                "model_bytes": self.model_bytes,
                "device_shots_per_s": (self.total_shots / self.device_time_s
                                       if self.device_time_s > 0 else 0.0)}


# ----------------------------------------------------------------------
# program cache
# ----------------------------------------------------------------------

_PROGRAMS: dict = {}


def _program_for(prog, max_dim: int) -> Program:
    key = (id(prog), max_dim)
    hit = _PROGRAMS.get(key)
    if hit is not None and hit[0] is prog:
        return hit[1]
    p = Program.compile(prog, max_dim=max_dim)
    if len(_PROGRAMS) > 64:
        _PROGRAMS.clear()
    _PROGRAMS[key] = (prog, p)
    return p


# the sparse form's limits (gs_sparse.cuh): u32 coordinates of a <= 30-dim
# span, list indices in 16 bits
SPARSE_MAX_DIM = 30
SPARSE_MAX_CAPACITY = 1 << 16


def _plan(prog, cfg: SamplerConfig):
    """(program, chi-form run flag, fallback) for ``cfg.chi``.  "auto" runs
    the dense forms; when the program compiled at ``cfg.dim_limit`` is
    truncated (a shot can reach a dimension the dense buffers cannot hold
    while within the capacity -- the advisor's cancelling-T case) the
    fallback is the same program on the sparse form (max_dim 30), like the
    reference's map (ref state.py:294-306).  Callers run a wave dense and
    switch to the fallback -- rerunning that wave -- once a wave reports an
    UNSUPPORTED shot: the forms give identical per-shot results, so the
    counters stay exact.  ``_choose_form`` decides up front on a probe."""
    if cfg.chi == "dense":
        return _program_for(prog, cfg.dim_limit), 0, None
    sparse_ok = cfg.effective_capacity <= SPARSE_MAX_CAPACITY
    if cfg.chi == "sparse":
        if not sparse_ok:
            raise ValueError("chi='sparse' needs an effective capacity <= %d" % SPARSE_MAX_CAPACITY)
        lim = SPARSE_MAX_DIM if cfg.max_dim is None else min(cfg.max_dim, SPARSE_MAX_DIM)
        return _program_for(prog, lim), _lib.GS_SPARSE, None
    p = _program_for(prog, cfg.dim_limit)
    if p.dp.truncated_at is not None and sparse_ok and cfg.max_dim is None:
        return p, 0, (_program_for(prog, SPARSE_MAX_DIM), _lib.GS_SPARSE)
    return p, 0, None


PROBE_SHOTS = 4096


def _choose_form(p, eng, cfg, fallback, shot_begin):
    """For a truncated program (``_plan``'s fallback): run a probe of the
    run's first <= PROBE_SHOTS shots dense; an UNSUPPORTED shot there picks
    the sparse form (a dense wave would stall on 2^limit-entry passes for
    shots the sparse form runs on a few entries: 34 K vs 30 M shots/s on
    24 cancelled T blocks, profiles/sparse_r02.jsonl); otherwise the faster
    of the two on the same probe (config-4 n=64, T=32: sparse 1.6x; the
    results are identical either way).  Cached per program and run flags."""
    key = (eng.device, cfg.run_flags(), cfg.effective_capacity)
    hit = p._chi_form.get(key)
    if hit is not None:
        return (p, 0) if hit == 0 else fallback
    n = max(1, min(PROBE_SHOTS, cfg.shots))
    par = Engine.params(cfg.master_seed, shot_begin, n, cfg.effective_capacity, cfg.run_flags())
    c = eng.run_counters(p, par)
    t_dense = eng.last_kernel_ms
    choice = 1
    if not c[_lib.GS_C_UNSUPPORTED]:
        ps, fs = fallback
        par = Engine.params(cfg.master_seed, shot_begin, n, cfg.effective_capacity,
                            cfg.run_flags() | fs)
        eng.run_counters(ps, par)
        choice = 1 if eng.last_kernel_ms < t_dense else 0
    p._chi_form[key] = choice
    return (p, 0) if choice == 0 else fallback


# runs at least this long (shots) tune the narrow limit first (the probe
# costs 4 x Program.TUNE_SHOTS shots, once per program)
TUNE_MIN_SHOTS = 1 << 23


def tuned_flags(p: Program, eng: Engine, cfg: SamplerConfig) -> int:
    """Performance-only run flags measured for this program (the narrow chi
    limit, ``Program.narrow_flag``); 0 for short runs."""
    if cfg.shots < TUNE_MIN_SHOTS:   # reuse an earlier tuning, never probe
        return p._narrow.get(Program.tuning_key(eng, cfg.run_flags()), 0)
    return p.narrow_flag(eng, cfg.run_flags(), cfg.effective_capacity)


def counters_to_stats(c: np.ndarray, obs_keys, wall: float,
                      device_s: float = 0.0, dp=None) -> RunStats:
    """Host counter vector -> RunStats; corrupt shots raise like the
    reference (ref state.py:170-171 propagates out of run_batch)."""
    if c[_lib.GS_C_CORRUPT]:
        raise CorruptStateError("%d shot(s) selected a ~zero-weight measurement "
                                "branch" % int(c[_lib.GS_C_CORRUPT]))
    if c[_lib.GS_C_UNSUPPORTED]:
        raise UnsupportedCircuitError(int(c[_lib.GS_C_UNSUPPORTED]),
                                      getattr(dp, "truncated_at", None),
                                      getattr(dp, "max_dim", None))
    per = {}
    for i, k in enumerate(obs_keys):
        v = int(c[_lib.GS_C_PER_OBS + i])
        if v:
            per[k] = v
    return RunStats(
        total_shots=int(c[_lib.GS_C_TOTAL]),
        preserved_shots=int(c[_lib.GS_C_PRESERVED]),
        discarded_shots=int(c[_lib.GS_C_DISCARDED]),
        overflow_count=int(c[_lib.GS_C_OVERFLOW]),
        logical_errors=dict(sorted(per.items())),
        logical_error_shots=int(c[_lib.GS_C_ERROR_SHOTS]),
        wall_time_s=wall, device_time_s=device_s,
        model_bytes=int(c[_lib.GS_C_MODEL_BYTES]))


def run_batch(prog, cfg: SamplerConfig, *, shot_begin: int = 0,
              engine: Engine | None = None, witnesses: int = 0) -> RunStats:
    """Counters of shots [shot_begin, shot_begin + cfg.shots) (global shot
    indices, so shards of one run combine exactly), issued in waves of
    ``cfg.batch_size`` shots -- one synchronous gs_run_counters call per wave,
    as the reference issues waves of batch_size (ref sampler.py:348-382).
    Counters do not depend on the wave size.

    ``witnesses > 0`` also collects the global indices of up to that many
    preserved shots whose observables flipped ("rare-failure witnesses",
    paper §V-B); replay one with ``run_shot`` and
    ``ShotContext.reset(derive_seed(master_seed, index))``.
    """
    t0 = time.perf_counter()
    p, form, fallback = _plan(prog, cfg)
    eng = engine or get_engine(cfg.device)
    with eng.lock:   # the waves and their device times, not interleaved with other threads
        if fallback is not None and cfg.shots:
            p, form = _choose_form(p, eng, cfg, fallback, shot_begin)
            if form:
                fallback = None
        return _run_batch_locked(p, eng, cfg, shot_begin, witnesses, t0, form, fallback)


def _run_batch_locked(p, eng, cfg, shot_begin, witnesses, t0, form=0, fallback=None):
    flags = cfg.run_flags() | (form or tuned_flags(p, eng, cfg))
    total = np.zeros(p.num_counters, dtype=np.int64)
    wit: list = []
    dev_s = 0.0
    done = 0
    while done < cfg.shots:
        cnt = min(cfg.wave_shots, cfg.shots - done)
        par = Engine.params(cfg.master_seed, shot_begin + done, cnt,
                            cfg.effective_capacity, flags)
        if witnesses > len(wit):
            c, w, _ = eng.run_counters_witness(p, par, witnesses - len(wit))
        else:
            c, w = eng.run_counters(p, par), []
        dev_s += eng.last_kernel_ms * 1e-3
        if fallback is not None and c[_lib.GS_C_UNSUPPORTED]:
            # past the dense dimension limit: this wave and the rest sparse
            p, form = fallback
            fallback = None
            flags = cfg.run_flags() | form
            continue
        total += c
        wit.extend(int(x) for x in w)
        done += cnt
    st = counters_to_stats(total, p.dp.obs_keys, time.perf_counter() - t0,
                           dev_s, dp=p.dp)
    st.witnesses = sorted(wit)
    return st


@dataclass
class ShotBatch:
    """Per-shot results of ``sample``: status codes (1 preserved, 2
    discarded, 3 overflow), aux (discarded detector / overflow instruction /
    -1), packed records (bit m of word m//64 = measurement m), observable
    bits (bit i = ``obs_keys[i]``)."""
    status: np.ndarray
    aux: np.ndarray
    records: np.ndarray
    obs_bits: np.ndarray
    obs_keys: list
    num_measurements: int

    def record_bits(self) -> np.ndarray:
        """Unpacked records, shape (shots, num_measurements), uint8."""
        if self.num_measurements == 0:
            return np.zeros((len(self.status), 0), dtype=np.uint8)
        b = np.unpackbits(self.records.view(np.uint8), axis=1, bitorder="little")
        return b[:, : self.num_measurements]

    def result(self, i: int, *, measured: int | None = None) -> ShotResult:
        st = _STATUS.get(int(self.status[i]))
        if st is None:
            raise CorruptStateError("shot %d ended in status %d" % (i, self.status[i]))
        if self.num_measurements:
            bits = np.unpackbits(np.ascontiguousarray(self.records[i]).view(np.uint8),
                                 bitorder="little")[: self.num_measurements]
        else:
            bits = np.zeros(0, dtype=np.uint8)
        nrec = len(bits) if measured is None else measured
        obs = {}
        if st is ShotStatus.PRESERVED:
            ob = int(self.obs_bits[i])
            obs = {k: (ob >> j) & 1 for j, k in enumerate(self.obs_keys)}
        return ShotResult(
            status=st, observables=obs,
            discarded_detector=int(self.aux[i]) if st is ShotStatus.DISCARDED else None,
            overflow_instruction=int(self.aux[i]) if st is ShotStatus.OVERFLOW else None,
            record=[int(b) for b in bits[:nrec]])


def sample(prog, cfg: SamplerConfig, *, shot_begin: int = 0, seeds=None,
           engine: Engine | None = None, extra_flags: int = 0) -> ShotBatch:
    """Per-shot statuses, measurement records and observables.
    ``extra_flags``: performance-only run flags (e.g. ``GS_NARROW_K5``)."""
    p, form, fallback = _plan(prog, cfg)
    eng = engine or get_engine(cfg.device)
    if fallback is not None and cfg.shots:
        with eng.lock:
            p, form = _choose_form(p, eng, cfg, fallback, shot_begin)
        if form:
            fallback = None
    par = Engine.params(cfg.master_seed, shot_begin, cfg.shots,
                        cfg.effective_capacity, cfg.run_flags() | form | extra_flags, seeds=seeds)
    status, aux, rec, obs = eng.run_records(p, par)
    if fallback is not None and np.any(status == 5):   # (see _plan)
        p, form = fallback
        par = Engine.params(cfg.master_seed, shot_begin, cfg.shots, cfg.effective_capacity,
                            cfg.run_flags() | form | extra_flags, seeds=seeds)
        status, aux, rec, obs = eng.run_records(p, par)
    if np.any(status == 4):
        raise CorruptStateError("a shot selected a ~zero-weight branch")
    if np.any(status == 5):
        raise UnsupportedCircuitError(int(np.sum(status == 5)), int(aux[status == 5][0]),
                                      p.dp.max_dim)
    return ShotBatch(status, aux, rec, obs, list(p.dp.obs_keys),
                     p.dp.num_measurements)


class ShotContext:
    """Per-trajectory context (ref sampler.py:152-166): a seed and a
    capacity; the state itself lives on the device."""

    def __init__(self, num_qubits: int, entry_capacity: int):
        self.num_qubits = num_qubits
        self.entry_capacity = entry_capacity
        self.seed = None
        self.capacity = entry_capacity

    def reset(self, seed: int, capacity: int | None = None) -> None:
        self.seed = seed & _M64
        self.capacity = capacity if capacity is not None else self.entry_capacity


def run_shot(prog, ctx: ShotContext, *, postselect: bool = False,
             observer=None, keep_record: bool = False) -> ShotResult:
    """One trajectory with an explicit SplitMix seed (ref sampler.py:169).
    The lockstep ``observer`` hook of the CPU reference is not supported on
    the device path."""
    if observer is not None:
        raise NotImplementedError("observer callbacks need the CPU oracle")
    if ctx.seed is None:
        raise ValueError("ShotContext.reset(seed) was not called")
    cfg = SamplerConfig(shots=1, entry_capacity=max(ctx.capacity, 2),
                        postselect=postselect, rerun_on_overflow=False)
    batch = sample(prog, cfg, seeds=np.array([ctx.seed], dtype=np.uint64))
    measured = _records_before(prog, batch, 0)
    res = batch.result(0, measured=measured)
    if not keep_record:
        res.record = None
    return res


_PREFIX: dict = {}


def _measure_prefix(prog):
    """(measurements before flat instruction j, measurements before the
    d-th executed DETECTOR), computed once per program."""
    hit = _PREFIX.get(id(prog))
    if hit is not None and hit[0] is prog:
        return hit[1], hit[2]
    by_instr, by_det = [], []
    m = 0
    for ins in prog.flat():
        by_instr.append(m)
        if ins.name in ("M", "MR", "MPP"):
            m += len(ins.targets)
        elif ins.name == "DETECTOR":
            by_det.append(m)
    by_instr.append(m)
    if len(_PREFIX) > 64:
        _PREFIX.clear()
    _PREFIX[id(prog)] = (prog, by_instr, by_det)
    return by_instr, by_det


def _records_before(prog, batch: ShotBatch, i: int) -> int:
    """Number of measurements made before a shot stopped (the reference
    returns the partial record of discarded / overflowed shots)."""
    st = int(batch.status[i])
    if st == 1:
        return batch.num_measurements
    stop = int(batch.aux[i])
    by_instr, by_det = _measure_prefix(prog)
    if st == 3:
        return by_instr[min(max(stop, 0), len(by_instr) - 1)]
    if st == 2 and 0 <= stop < len(by_det):
        return by_det[stop]
    return by_instr[-1]


# ----------------------------------------------------------------------
# statistics (ref sampler.py:389-429)
# ----------------------------------------------------------------------

def bayes_interval(k: int, n: int, factor: float = 1000.0):
    """All binomial rates whose likelihood is within ``factor`` of the
    maximum; closed forms at k == 0 and k == n, bisection otherwise."""
    if n < 1:
        raise ValueError("need at least one trial")
    if not 0 <= k <= n:
        raise ValueError("k out of range")
    if k == 0:
        return 0.0, 1.0 - factor ** (-1.0 / n)
    if k == n:
        return factor ** (-1.0 / n), 1.0
    phat = k / n
    top = k * math.log(phat) + (n - k) * math.log1p(-phat)
    lf = math.log(factor)

    def inside(p: float) -> bool:
        if p <= 0.0 or p >= 1.0:
            return False
        return k * math.log(p) + (n - k) * math.log1p(-p) - top + lf >= 0.0

    def edge(a: float, b: float, a_inside: bool) -> float:
        # invariant: inside(a) == a_inside, inside(b) != a_inside
        for _ in range(2000):
            mid = 0.5 * (a + b)
            if mid in (a, b):
                break
            if inside(mid) == a_inside:
                a = mid
            else:
                b = mid
        return 0.5 * (a + b)

    return edge(phat, 0.0, True), edge(phat, 1.0, True)


def throughput_bench(prog, cfg: SamplerConfig, sweep: str, values):
    """Rows (swept value, shots/s, discard rate) (ref sampler.py:436-452)."""
    from .noise import apply_noise_model
    rows = []
    for v in values:
        if sweep == "batch-size":
            st = run_batch(prog, replace(cfg, batch_size=int(v)))
        elif sweep == "noise":
            st = run_batch(apply_noise_model(prog, float(v)), cfg)
        else:
            raise ValueError("unknown sweep kind %r" % (sweep,))
        rows.append((float(v), st.throughput, st.discard_rate))
    return rows
