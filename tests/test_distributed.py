"""Multi-process path on CPU (gloo, world_size 2): global-index sharding +
the single counter all-reduce must reproduce a one-process run exactly.
The shard runner here is the CPU oracle (test infrastructure), standing in
for the GPU engine that the same code path drives on B200s."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_23037_b200 import SamplerConfig, parse_circuit
from paper_2512_23037_b200.distributed import run_batch_distributed, shard_range
from paper_2512_23037_b200 import _lib

PROG = ("H 0\nCX 0 1\nDEPOLARIZE1(0.1) 0 1\nT 0\nM 0\nM 1\n"
        "DETECTOR rec[-1] rec[-2]\nOBSERVABLE_INCLUDE(0) rec[-1]\n"
        "OBSERVABLE_INCLUDE(2) rec[-2]\n")


def _oracle_runner(prog, cfg, begin, count):
    from oracle import gstab_oracle as orc
    c = orc.run_counters(prog, count, cfg.master_seed, shot_begin=begin,
                         mode=cfg.rng, postselect=cfg.postselect)
    keys = [0, 2]
    vec = np.zeros(_lib.GS_C_PER_OBS + len(keys), dtype=np.int64)
    vec[_lib.GS_C_TOTAL] = c["total"]
    vec[_lib.GS_C_PRESERVED] = c["preserved"]
    vec[_lib.GS_C_DISCARDED] = c["discarded"]
    vec[_lib.GS_C_OVERFLOW] = c["overflow"]
    vec[_lib.GS_C_ERROR_SHOTS] = c["error_shots"]
    for i, k in enumerate(keys):
        vec[_lib.GS_C_PER_OBS + i] = c["per_observable"].get(k, 0)
    return torch.from_numpy(vec), keys


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = SamplerConfig(shots=301, master_seed=5, postselect=True, rng="philox")
        st = run_batch_distributed(parse_circuit(PROG), cfg,
                                   shard_runner=_oracle_runner)
        out[rank] = (st.total_shots, st.preserved_shots, st.discarded_shots,
                     st.logical_error_shots, tuple(sorted(st.logical_errors.items())))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions_exactly():
    for total in (0, 1, 7, 100, 10**9 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (b0, c0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + c0 == b1
            assert sum(c for _, c in spans) == total
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def test_gloo_world2_matches_single_process():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = SamplerConfig(shots=301, master_seed=5, postselect=True, rng="philox")
    whole, keys = _oracle_runner(parse_circuit(PROG), cfg, 0, 301)
    w = whole.numpy()
    want = (int(w[0]), int(w[1]), int(w[2]), int(w[6]),
            tuple((k, int(w[8 + i])) for i, k in enumerate(keys) if w[8 + i]))
    assert out[0] == out[1] == want
