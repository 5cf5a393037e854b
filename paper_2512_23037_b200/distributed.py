"""Multi-GPU sampling: one process per GPU, shots sharded by global index,
one all-reduce of the int64 counter vector at the end.

Shots are independent and seeded by (master_seed, global shot index) (ref
sampler.py:37-42, 348-382), so rank r of R simply runs the contiguous global
range ``shard_range(shots, r, R)`` and the summed counters equal a
single-process run exactly, for any R (the reference's worker-count
determinism, ref tests/test_sampler.py:164-178).  The only collective is one
``all_reduce(SUM)`` of ``GS_C_PER_OBS + num_obs`` int64 counters issued on
the device buffer the kernel accumulated into (NCCL over NVLink on B200).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import _lib
from .sampler import SamplerConfig, counters_to_stats, _plan, tuned_flags


def shard_range(total: int, rank: int, world: int):
    """Contiguous, balanced global shot range [begin, begin+count) of a rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def rank_device(cfg: SamplerConfig) -> int:
    """CUDA ordinal of this rank: LOCAL_RANK (one process per GPU, torchrun)
    modulo the visible devices, else ``cfg.device``."""
    import torch
    n = max(torch.cuda.device_count(), 1)
    lr = os.environ.get("LOCAL_RANK")
    return int(lr) % n if lr is not None else cfg.device


def _gpu_shard_counters(prog, cfg: SamplerConfig, begin: int, count: int):
    """Run one rank's shard on its GPU (set explicitly, not inherited from
    the caller's current device); counters stay on that device."""
    import torch
    from .engine import Engine, get_engine
    p, form, fallback = _plan(prog, cfg)
    if fallback is not None:   # (counters stay on the device here: no dense probe)
        p, form = fallback
    dev = rank_device(cfg)
    with torch.cuda.device(dev):
        eng = get_engine(dev)
        counters = torch.zeros(p.num_counters, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev)
        chunk = cfg.wave_shots
        flags = cfg.run_flags() | (form or tuned_flags(p, eng, cfg))
        done = 0
        while done < count:
            n = min(chunk, count - done)
            par = Engine.params(cfg.master_seed, begin + done, n,
                                cfg.effective_capacity, flags)
            eng.run_counters_async(p, par, counters.data_ptr(), stream.cuda_stream)
            done += n
    return counters, p.dp.obs_keys


def run_batch_distributed(prog, cfg: SamplerConfig, *, group=None,
                          shard_runner=None):
    """``run_batch`` across all ranks of the default (or given) process
    group.  Every rank returns the same global ``RunStats``.

    ``shard_runner(prog, cfg, begin, count) -> (counter tensor, obs_keys)``
    defaults to the GPU engine; tests substitute a CPU runner to exercise
    the sharding and reduction over gloo.
    """
    import torch
    import torch.distributed as dist
    t0 = time.perf_counter()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    begin, count = shard_range(cfg.shots, rank, world)
    runner = shard_runner or _gpu_shard_counters
    counters, obs_keys = runner(prog, cfg, begin, count)
    if world > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    c = counters.cpu().numpy().astype(np.int64)
    return counters_to_stats(c, obs_keys, time.perf_counter() - t0)
