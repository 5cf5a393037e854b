"""GPU runtime plumbing of the engine (through the C ABI): per-section
statistics (GS_SECTION_STATS), cross-stream ordering of sync and async runs
on one engine, the queue budget / trim, wave sizes, and the NCCL code path of
run_batch_distributed at world size 1."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2512_23037_b200 import SamplerConfig, run_batch
from paper_2512_23037_b200 import _lib
from paper_2512_23037_b200.engine import Engine, Program
from paper_2512_23037_b200.msc import msc_grown_circuit
from paper_2512_23037_b200.noise import apply_noise_model
from paper_2512_23037_b200.sampler import _program_for


@pytest.fixture(scope="module")
def d5():
    return apply_noise_model(msc_grown_circuit(5), 1e-3)


def _flags(stats=False):
    f = _lib.GS_POSTSELECT | _lib.GS_RNG_PHILOX
    return f | (_lib.GS_SECTION_STATS if stats else 0)


def test_section_stats_partition_the_run(d5):
    p = _program_for(d5, 13)
    eng = Engine(0)
    S = 1 << 18
    c0 = eng.run_counters(p, Engine.params(4, 0, S, 4096, _flags()))
    eng.section_stats(reset=True)
    c1 = eng.run_counters(p, Engine.params(4, 0, S, 4096, _flags(True)))
    secs = eng.section_stats(reset=True)
    assert np.array_equal(c0, c1)          # measurement does not change results
    assert len(secs) == p.sections(0) > 1
    assert secs[0]["shots_in"] == S
    for a, b in zip(secs, secs[1:]):
        assert a["shots_out"] == b["shots_in"]
    assert secs[-1]["shots_out"] == 0
    # the sections' device-counted model bytes add up to the run's counter
    assert sum(s["model_bytes"] for s in secs) == int(c1[_lib.GS_C_MODEL_BYTES])
    assert all(s["device_ms"] > 0 and s["launches"] == 1 for s in secs)
    assert {s["kernel"] for s in secs} == {"narrow", "wide"}
    # reset cleared everything
    assert all(s["launches"] == 0 and s["model_bytes"] == 0
               for s in eng.section_stats(reset=True))


def test_section_stats_of_the_sparse_form(d5):
    """GS_SPARSE runs one section (the whole program): its stats hold every
    shot and the run's model bytes, and the counters equal the dense run's."""
    p = _program_for(d5, 13)
    eng = Engine(0)
    S = 1 << 15
    c0 = eng.run_counters(p, Engine.params(4, 0, S, 4096, _flags()))
    eng.section_stats(reset=True)
    c1 = eng.run_counters(p, Engine.params(4, 0, S, 4096, _flags(True) | _lib.GS_SPARSE))
    secs = eng.section_stats(reset=True)
    assert np.array_equal(c0, c1)
    assert len(secs) == 1 and p.sections(_lib.GS_SPARSE) == 1
    assert secs[0]["shots_in"] == S and secs[0]["shots_out"] == 0
    assert secs[0]["model_bytes"] == int(c1[_lib.GS_C_MODEL_BYTES])
    assert secs[0]["kernel"] == "wide" and secs[0]["launches"] == 1


def test_section_stats_accumulate_over_chunks_and_async(d5):
    import torch
    p = _program_for(d5, 13)
    eng = Engine(0)
    eng.section_stats(reset=True)
    dev = torch.zeros(p.num_counters, dtype=torch.int64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(3):
            eng.run_counters_async(p, Engine.params(5, k << 16, 1 << 16, 4096, _flags(True),
                                                    chunk_shots=1 << 14),
                                   dev.data_ptr(), st.cuda_stream)
    secs = eng.section_stats(reset=True)
    assert secs[0]["shots_in"] == 3 << 16
    assert all(s["launches"] == 12 for s in secs)
    assert sum(s["model_bytes"] for s in secs) == int(dev[_lib.GS_C_MODEL_BYTES].item())


def test_async_then_sync_on_one_engine_is_ordered(d5):
    """An async run on a side stream followed at once by synchronous runs on
    the engine's own stream: shared scratch must not race (the engine orders
    the streams), so every counter vector equals a clean run's."""
    import torch
    p = _program_for(d5, 13)
    eng = Engine(0)
    ref = eng.run_counters(p, Engine.params(7, 0, 1 << 19, 4096, _flags()))
    st = torch.cuda.Stream()
    for _ in range(3):
        dev = torch.zeros(p.num_counters, dtype=torch.int64, device="cuda")
        eng.run_counters_async(p, Engine.params(7, 0, 1 << 19, 4096, _flags()),
                               dev.data_ptr(), st.cuda_stream)
        again = eng.run_counters(p, Engine.params(7, 0, 1 << 19, 4096, _flags()))
        st.synchronize()
        assert np.array_equal(dev.cpu().numpy(), ref)
        assert np.array_equal(again, ref)


def test_queue_budget_and_trim_keep_results(d5):
    p = _program_for(d5, 13)
    eng = Engine(0)
    ref = eng.run_counters(p, Engine.params(8, 0, 1 << 18, 4096, _flags()))
    eng.trim()
    eng.set_queue_budget(3 << 20)           # ~8k slots: many chunks
    small = eng.run_counters(p, Engine.params(8, 0, 1 << 18, 4096, _flags()))
    eng.set_queue_budget(0)
    eng.trim()
    auto = eng.run_counters(p, Engine.params(8, 0, 1 << 18, 4096, _flags()))
    assert np.array_equal(small, ref) and np.array_equal(auto, ref)


def test_wave_size_does_not_change_counters(d5):
    base = None
    for bs in (None, 1 << 12, 100_000):
        st = run_batch(d5, SamplerConfig(shots=300_000, master_seed=3, postselect=True,
                                         rng="philox", batch_size=bs))
        key = (st.total_shots, st.preserved_shots, st.discarded_shots,
               st.logical_error_shots, st.model_bytes)
        base = base or key
        assert key == base


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_run_batch_distributed_over_nccl_world_size_1(d5):
    """The multi-GPU code path as torchrun runs it, at world size 1 on one
    B200: NCCL process group bound to the device, shard, async launches on
    the rank's device, the counter all-reduce over NCCL."""
    import torch
    import torch.distributed as dist
    from paper_2512_23037_b200.distributed import run_batch_distributed
    env = {"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(_free_port()),
           "RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        dist.init_process_group("nccl", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
        assert dist.get_backend() == "nccl"
        cfg = SamplerConfig(shots=1 << 20, master_seed=11, postselect=True, rng="philox")
        got = run_batch_distributed(d5, cfg)
        # the collective really ran on NCCL
        t = torch.ones(4, dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        assert t.sum().item() == 4
        dist.destroy_process_group()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    want = run_batch(d5, cfg)
    assert (got.total_shots, got.preserved_shots, got.discarded_shots,
            got.logical_error_shots) == (want.total_shots, want.preserved_shots,
                                         want.discarded_shots, want.logical_error_shots)


def test_narrow_limit_tuning_is_cached_and_result_neutral():
    """Program.narrow_flag times both narrow chi limits on a probe and keeps
    the faster; the counters of a run are identical under either limit."""
    from paper_2512_23037_b200 import SamplerConfig, _lib, run_batch
    from paper_2512_23037_b200.engine import Engine, get_engine
    from paper_2512_23037_b200.msc import msc_d5_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    from paper_2512_23037_b200.sampler import _program_for
    prog = apply_noise_model(msc_d5_circuit(), 1e-3)
    cfg = SamplerConfig(shots=1 << 21, master_seed=4, postselect=True, rng="philox")
    p = _program_for(prog, cfg.dim_limit)
    eng = get_engine(0)
    f = p.narrow_flag(eng, cfg.run_flags(), cfg.effective_capacity)
    assert f in (0, _lib.GS_NARROW_K5)
    assert set(p.narrow_tuning) == {"k4_ms", "k5_ms", "probe_shots"}
    assert p.narrow_flag(eng, cfg.run_flags(), cfg.effective_capacity) == f   # cached
    assert p.sections(cfg.run_flags()) != p.sections(cfg.run_flags() | _lib.GS_NARROW_K5)
    got = [eng.run_counters(p, Engine.params(4, 0, cfg.shots, cfg.effective_capacity,
                                             cfg.run_flags() | x))
           for x in (0, _lib.GS_NARROW_K5)]
    assert (got[0] == got[1]).all()
    st = run_batch(prog, cfg)
    assert st.total_shots == cfg.shots and st.preserved_shots == int(got[0][_lib.GS_C_PRESERVED])


def test_shared_engine_is_safe_across_python_threads():
    """get_engine's process-wide engine is shared: runs from several Python
    threads are serialised by its lock (ctypes releases the GIL) and every
    thread gets the counters a lone run gives."""
    import threading
    from paper_2512_23037_b200 import SamplerConfig, parse_circuit, run_batch
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(parse_circuit("H 0 1 2\nT 0 1\nCX 0 2\nT_DAG 2\nM 0 1 2\n"
                                           "DETECTOR rec[-1] rec[-3]\n"), 0.01)
    cfg = SamplerConfig(shots=300_000, master_seed=8, postselect=True, rng="philox")
    want = run_batch(prog, cfg).as_dict()
    got = [None] * 6

    def work(i):
        got[i] = run_batch(prog, cfg).as_dict()

    ts = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for g in got:
        for k in ("total_shots", "preserved_shots", "discarded_shots", "logical_error_shots"):
            assert g[k] == want[k], (k, g[k], want[k])
