"""Multi-process GPU path on one B200: two ranks (gloo for the collective,
both on cuda:0) shard a run by global shot index through the real engine
(`run_batch_distributed`, device counters reduced in place); the reduced
counters equal a one-process run exactly."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cancelled_t(nq):
    from paper_2512_23037_b200 import parse_circuit
    body = "".join("H %d\nT %d\nDEPOLARIZE1(0.01) %d\nT_DAG %d\nH %d\n" % (q, q, q, q, q)
                   for q in range(nq))
    return parse_circuit(body + "M " + " ".join(map(str, range(nq))) + "\nDETECTOR rec[-1]\n")


def _worker(rank, world, port, out, which="grown"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_23037_b200 import SamplerConfig
        from paper_2512_23037_b200.distributed import run_batch_distributed
        from paper_2512_23037_b200.msc import msc_grown_circuit
        from paper_2512_23037_b200.noise import apply_noise_model
        if which == "grown":
            prog = apply_noise_model(msc_grown_circuit(5), 1e-3)
        else:   # past the dense dimension limit: the shards run the sparse form
            prog = _cancelled_t(22)
        cfg = SamplerConfig(shots=200_001, master_seed=5, postselect=True, rng="philox")
        st = run_batch_distributed(prog, cfg)
        out[rank] = st.as_dict()
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_process():
    from paper_2512_23037_b200 import SamplerConfig, run_batch
    from paper_2512_23037_b200.msc import msc_grown_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    prog = apply_noise_model(msc_grown_circuit(5), 1e-3)
    one = run_batch(prog, SamplerConfig(shots=200_001, master_seed=5, postselect=True,
                                        rng="philox")).as_dict()
    keys = ("total_shots", "preserved_shots", "discarded_shots", "logical_error_shots",
            "overflow_count")
    for r in (0, 1):
        for k in keys:
            assert out[r][k] == one[k], (r, k)


def test_two_ranks_on_the_sparse_form():
    """A program past the dense dimension limit (22 cancelled T blocks):
    the shards take the sparse form; the reduced counters equal a
    one-process run_batch (which probes, then runs sparse)."""
    from paper_2512_23037_b200 import SamplerConfig, run_batch
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.start_processes(_worker, args=(2, _free_port(), out, "sparse"), nprocs=2, join=True,
                       start_method="spawn")
    one = run_batch(_cancelled_t(22), SamplerConfig(shots=200_001, master_seed=5,
                                                    postselect=True, rng="philox")).as_dict()
    for r in (0, 1):
        for k in ("total_shots", "preserved_shots", "discarded_shots", "overflow_count"):
            assert out[r][k] == one[k], (r, k)
