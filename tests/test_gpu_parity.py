"""GPU parity: the CUDA sampler (through the C ABI) against the reference's
golden fixtures and the CPU oracle.

Bars (north star): records / statuses / counters bit-exact; tableau x/z/sign
bits and amplitude indices exact; every amplitude within 1e-10 RELATIVE
error of the reference's (fp64; ``chi_check.assert_chi_close``).
"""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import gstab_oracle as orc
from paper_2512_23037_b200 import (SamplerConfig, ShotContext, compile_program,
                                   derive_seed, parse_circuit, run_batch,
                                   run_shot, sample)
from paper_2512_23037_b200 import _lib
from paper_2512_23037_b200.engine import Engine, Program, get_engine
from paper_2512_23037_b200.frames import reconstruct_state
from paper_2512_23037_b200.sampler import _records_before

from chi_check import assert_chi_close


def _gpu_results(prog, master, shots, capacity, postselect, rng="splitmix",
                 shot_begin=0, flags_extra=0):
    dp = compile_program(prog)
    p = Program(dp)
    eng = get_engine(0)
    flags = (_lib.GS_POSTSELECT if postselect else 0) | flags_extra
    if rng == "philox":
        flags |= _lib.GS_RNG_PHILOX
    par = Engine.params(master, shot_begin, shots, capacity, flags)
    status, aux, rec, obs = eng.run_records(p, par)
    from paper_2512_23037_b200.sampler import ShotBatch
    b = ShotBatch(status, aux, rec, obs, list(dp.obs_keys), dp.num_measurements)
    out = []
    for i in range(shots):
        r = b.result(i, measured=_records_before(prog, b, i))
        out.append({"status": r.status.value,
                    "observables": {str(k): v for k, v in sorted(r.observables.items())},
                    "discarded_detector": r.discarded_detector,
                    "overflow_instruction": r.overflow_instruction,
                    "record": r.record})
    return out


def _oracle_results(prog, master, shots, capacity, postselect, mode="splitmix",
                    shot_begin=0):
    flat = list(prog.flat())
    out = []
    for s in range(shot_begin, shot_begin + shots):
        r = orc.run_one_shot(flat, prog.num_qubits,
                             orc.DrawStream(mode, master, s), capacity, postselect)
        out.append({"status": r["status"],
                    "observables": {str(k): v for k, v in sorted(r["observables"].items())},
                    "discarded_detector": r["discarded_detector"],
                    "overflow_instruction": r["overflow_instruction"],
                    "record": r["record"]})
    return out


def test_golden_shot_results_bit_exact(golden_shots):
    for fx in golden_shots:
        prog = parse_circuit(fx["text"])
        got = _gpu_results(prog, fx["master"], len(fx["shots"]), fx["capacity"],
                           fx["postselect"])
        assert got == fx["shots"], fx["name"]


@pytest.mark.parametrize("flag", [_lib.GS_CHI_GLOBAL, _lib.GS_CHI_SMEM,
                                  _lib.GS_WIDE_ONLY,
                                  _lib.GS_WIDE_ONLY | _lib.GS_CHI_SMEM,
                                  _lib.GS_WIDE_ONLY | _lib.GS_CHI_BLOCK,
                                  _lib.GS_SPARSE])
def test_golden_shot_results_storage_variants(golden_shots, flag):
    for fx in golden_shots[::3]:
        prog = parse_circuit(fx["text"])
        got = _gpu_results(prog, fx["master"], len(fx["shots"]), fx["capacity"],
                           fx["postselect"], flags_extra=flag)
        assert got == fx["shots"], fx["name"]


@pytest.mark.parametrize("flag", [0, _lib.GS_SPARSE])
def test_golden_state_snapshots(golden_states, flag):
    eng = get_engine(0)
    for fx in golden_states:
        prog = parse_circuit(fx["text"])
        for snap in fx["snaps"]:
            dp = compile_program(prog, stop_after=snap["i"], keep_frames=True)
            p = Program(dp)
            seeds = np.array([derive_seed(fx["master"], fx["shot"])], dtype=np.uint64)
            d = eng.dump(p, Engine.params(fx["master"], 0, 1, 4096, flag, seeds=seeds))
            assert int(d["status"][0]) == 1
            st = reconstruct_state(dp, snap["i"], int(d["sig"][0][0]) |
                                   (int(d["sig"][0][1]) << prog.num_qubits),
                                   int(d["c"][0]), d["amps"][0])
            assert st["xs"] == snap["xs"] and st["zs"] == snap["zs"]
            assert st["ph"] == snap["ph"], (fx["text"], snap["i"])
            assert st["idx"] == snap["idx"], (fx["text"], snap["i"])
            assert_chi_close(st["amp"], snap["amp"], context=(fx["text"], snap["i"]))


def test_golden_counters(golden_counters):
    for fx in golden_counters:
        kw = dict(fx["config"])
        cfg = SamplerConfig(**kw)
        st = run_batch(parse_circuit(fx["text"]), cfg)
        want = fx["counters"]
        assert st.total_shots == want["total"]
        assert st.preserved_shots == want["preserved"]
        assert st.discarded_shots == want["discarded"]
        assert st.overflow_count == want["overflow"]
        assert st.logical_error_shots == want["error_shots"]
        assert {str(k): v for k, v in st.logical_errors.items()} == want["per_observable"]


def _random_program(rng, n, gates, tcount, noise_p, mpp=True):
    lines = ["H %d" % rng.randrange(n)]
    meas = 0
    one = ("I", "X", "Y", "Z", "H", "S", "S_DAG", "H_XY", "H_NXY")
    for _ in range(gates):
        r = rng.random()
        if r < 0.12 and tcount > 0:
            tcount -= 1
            lines.append("%s %d" % (rng.choice(("T", "T_DAG")), rng.randrange(n)))
        elif r < 0.40:
            lines.append("%s %d" % (rng.choice(one), rng.randrange(n)))
        elif r < 0.62 and n >= 2:
            a, b = rng.sample(range(n), 2)
            lines.append("%s %d %d" % (rng.choice(("CX", "CZ", "SWAP")), a, b))
        elif r < 0.70:
            lines.append("%s %d" % (rng.choice(("M", "MR", "R")), rng.randrange(n)))
            meas += lines[-1][0] == "M"
        elif r < 0.75 and mpp:
            qs = rng.sample(range(n), min(n, rng.randint(1, 3)))
            prod = "*".join("%s%d" % (rng.choice("XYZ"), q) for q in qs)
            arg = "(%g)" % noise_p if rng.random() < 0.3 else ""
            lines.append("MPP%s %s" % (arg, prod))
            meas += 1
        elif r < 0.84:
            kind = rng.choice(("X_ERROR", "Z_ERROR", "DEPOLARIZE1", "DEPOLARIZE2"))
            if kind == "DEPOLARIZE2" and n >= 2:
                a, b = rng.sample(range(n), 2)
                lines.append("DEPOLARIZE2(%g) %d %d" % (noise_p, a, b))
            else:
                kind = "DEPOLARIZE1" if kind == "DEPOLARIZE2" else kind
                qs = [rng.randrange(n) for _ in range(rng.randint(1, 3))]
                lines.append("%s(%g) %s" % (kind, noise_p, " ".join(map(str, qs))))
        elif r < 0.90 and meas:
            g = rng.choice(("X", "Z", "CX", "CZ"))
            lines.append("%s rec[-%d] %d" % (g, rng.randint(1, meas), rng.randrange(n)))
        elif r < 0.95 and meas:
            lines.append("DETECTOR rec[-%d]" % rng.randint(1, meas))
        else:
            lines.append("TICK")
    lines.append("M %d" % rng.randrange(n))
    lines.append("OBSERVABLE_INCLUDE(%d) rec[-1]" % rng.randrange(3))
    return parse_circuit("\n".join(lines) + "\n")


@pytest.mark.parametrize("mode", ["splitmix", "philox"])
def test_random_programs_match_oracle(mode):
    rng = random.Random(1234 if mode == "splitmix" else 99)
    for it in range(60):
        n = rng.choice((2, 5, 9, 17, 33, 64))
        prog = _random_program(rng, n, rng.choice((30, 80)), rng.choice((4, 10, 16)),
                               rng.choice((0.02, 0.2)))
        post = it % 2 == 0
        cap = rng.choice((4, 64, 4096))
        got = _gpu_results(prog, 5 + it, 24, cap, post, rng=mode, shot_begin=1000)
        ref = _oracle_results(prog, 5 + it, 24, cap, post, mode=mode, shot_begin=1000)
        assert got == ref, (it, prog.serialize())


@pytest.mark.parametrize("mode", ["splitmix", "philox"])
def test_shot_indices_beyond_32_bits(mode):
    # BASELINE config 5 runs >= 1e10 shots: global indices past 2^32 (and a
    # master seed with its high word set) must key the same streams as the
    # oracle (SHA-1 of <QQ, Philox counter words 2-3 / key words 0-1)
    rng = random.Random(77)
    prog = _random_program(rng, 9, 60, 10, 0.05)
    for begin in ((1 << 32) - 8, 12_345_678_901, (1 << 62) + 5):
        master = (0xDEADBEEF << 32) | 17
        got = _gpu_results(prog, master, 16, 4096, True, rng=mode, shot_begin=begin)
        ref = _oracle_results(prog, master, 16, 4096, True, mode=mode, shot_begin=begin)
        assert got == ref, (mode, begin)


@pytest.mark.parametrize("n,t", [(56, 16), (48, 24)])
def test_large_chi_block_per_shot_matches_oracle(n, t):
    """Config-4 programs with chi beyond 32 KB run one block of warps per
    shot by default (k = 13: 8 warps, 2 blocks per SM; k = 15: 16 warps; both
    on global ping-pong buffers); records, statuses and overflow points must
    equal the oracle's and those of every other large-chi form (warp per
    shot on a global buffer, 16- and 8-warp blocks on shared or global chi)."""
    from paper_2512_23037_b200.msc import config4_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(config4_circuit(n, t, seed=n + t), 1e-3)
    dp = compile_program(prog, max_dim=16)
    assert dp.max_dim > 11
    shots = 6
    for mode in ("splitmix", "philox"):
        flags = _lib.GS_RNG_PHILOX if mode == "philox" else 0
        p = Program(dp)
        eng = get_engine(0)
        outs = []
        for extra in (0, _lib.GS_CHI_GLOBAL, _lib.GS_CHI_BLOCK,
                      _lib.GS_CHI_BLOCK | _lib.GS_BLOCK8,
                      _lib.GS_CHI_BLOCK | _lib.GS_BLOCK8 | _lib.GS_CHI_GLOBAL, _lib.GS_SPARSE):
            par = Engine.params(9, 0, shots, 32768, flags | extra)
            outs.append(eng.run_records(p, par))
        for other in outs[1:]:
            for x, y in zip(outs[0], other):
                assert np.array_equal(x, y), mode
        ref = _oracle_results(prog, 9, shots, 32768, False, mode=mode)
        got = _gpu_results(prog, 9, shots, 32768, False, rng=mode)
        assert got == ref, mode


def test_run_shot_api_matches_reference_examples():
    prog = parse_circuit("H 0\nH 1\nT 0\nT 1\n")
    ctx = ShotContext(prog.num_qubits, 2)
    ctx.reset(derive_seed(0, 0))
    res = run_shot(prog, ctx)
    assert res.status.value == "overflow" and res.overflow_instruction == 3
    for shot in range(20):
        ctx = ShotContext(2, 4096)
        ctx.reset(derive_seed(0, shot))
        res = run_shot(parse_circuit("H 0\nM 0\nX rec[-1] 0\nM 0\n"), ctx,
                       keep_record=True)
        assert res.record[1] == 0


def test_shard_and_launch_shape_invariance():
    from paper_2512_23037_b200.msc import msc_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(msc_circuit(3), 2e-3)
    p = Program(compile_program(prog))
    eng = get_engine(0)
    flags = _lib.GS_POSTSELECT | _lib.GS_RNG_PHILOX
    whole = eng.run_counters(p, Engine.params(7, 0, 20000, 32768, flags))
    parts = sum(eng.run_counters(p, Engine.params(7, a, 5000, 32768, flags))
                for a in range(0, 20000, 5000))
    odd = eng.run_counters(p, Engine.params(7, 0, 20000, 32768, flags,
                                            warps_per_block=3, blocks=17))
    assert np.array_equal(whole, parts)
    assert np.array_equal(whole, odd)


@pytest.mark.parametrize("d", [3, 5])
def test_msc_noiseless_is_deterministic(d):
    from paper_2512_23037_b200.msc import msc_circuit
    prog = msc_circuit(d)
    st = run_batch(prog, SamplerConfig(shots=4096, postselect=True, rng="philox"))
    assert st.discarded_shots == 0 and st.logical_error_shots == 0
    assert st.preserved_shots == 4096


@pytest.mark.parametrize("mode", ["splitmix", "philox"])
@pytest.mark.parametrize("variant", ["default", "wide_only", "chi_global",
                                     "chi_smem", "wide_only_chi_smem", "chi_block",
                                     "chi_block_global", "wide_only_chi_block", "narrow_k5",
                                     "chi_block8", "chi_block8_global", "sparse"])
def test_chi_storage_modes_match_oracle(variant, mode):
    """Lane-per-shot / warp-per-shot / block-per-shot execution and shared- /
    global-memory chi buffers must all give the oracle's results, in both
    random streams (Philox also exercises the conditional T-pair fusion,
    TF_FUSEQ, which depends on the shot's noise schedule)."""
    rng = random.Random(7)
    flags_extra = {"default": 0, "wide_only": _lib.GS_WIDE_ONLY,
                   "chi_global": _lib.GS_CHI_GLOBAL, "chi_smem": _lib.GS_CHI_SMEM,
                   "wide_only_chi_smem": _lib.GS_WIDE_ONLY | _lib.GS_CHI_SMEM,
                   "chi_block": _lib.GS_CHI_BLOCK,
                   "chi_block_global": _lib.GS_CHI_BLOCK | _lib.GS_CHI_GLOBAL,
                   "wide_only_chi_block": _lib.GS_WIDE_ONLY | _lib.GS_CHI_BLOCK,
                   "narrow_k5": _lib.GS_NARROW_K5,
                   "chi_block8": _lib.GS_CHI_BLOCK | _lib.GS_BLOCK8,
                   "chi_block8_global": _lib.GS_CHI_BLOCK | _lib.GS_BLOCK8 | _lib.GS_CHI_GLOBAL,
                   "sparse": _lib.GS_SPARSE}[variant]
    eng = get_engine(0)
    for it in range(25):
        n = rng.choice((4, 9, 20))
        prog = _random_program(rng, n, 70, rng.choice((8, 14)), 0.1)
        dp = compile_program(prog)
        p = Program(dp)
        flags = _lib.GS_POSTSELECT * (it % 2) | flags_extra
        if mode == "philox":
            flags |= _lib.GS_RNG_PHILOX
        par = Engine.params(3 + it, 0, 16, 4096, flags)
        status, aux, rec, obs = eng.run_records(p, par)
        from paper_2512_23037_b200.sampler import ShotBatch
        b = ShotBatch(status, aux, rec, obs, list(dp.obs_keys), dp.num_measurements)
        ref = _oracle_results(prog, 3 + it, 16, 4096, bool(it % 2), mode=mode)
        for i in range(16):
            r = b.result(i, measured=_records_before(prog, b, i))
            assert r.status.value == ref[i]["status"], (variant, it, i)
            assert r.record == ref[i]["record"], (variant, it, i)


@pytest.mark.parametrize("flag", [0, _lib.GS_CHI_BLOCK, _lib.GS_SPARSE])
def test_msc_d5_dumps_match_oracle_through_t_layer(flag):
    """Full-size state check: the d=5 proxy with chi peaking at 1024
    entries, dumped after the first T layer and after the undo layer
    (warp per shot, and one block of warps per shot)."""
    from paper_2512_23037_b200.msc import msc_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(msc_circuit(5), 2e-3)
    flat = list(prog.flat())
    t_idx = [i for i, ins in enumerate(flat) if ins.name in ("T", "T_DAG")]
    eng = get_engine(0)
    for stop in (t_idx[1], t_idx[2], t_idx[3] + 3, t_idx[5]):
        dp = compile_program(prog, stop_after=stop, keep_frames=True)
        p = Program(dp)
        for shot in range(3):
            seeds = np.array([derive_seed(4, shot)], dtype=np.uint64)
            cap = 1 << 16 if flag & _lib.GS_SPARSE else 1 << 20   # (sparse: <= 2^16)
            d = eng.dump(p, Engine.params(4, 0, 1, cap, flag, seeds=seeds))
            ref = orc.run_one_shot(flat, prog.num_qubits,
                                   orc.DrawStream("splitmix", 4, shot), cap,
                                   False, stop_after=stop, snapshot=True)
            assert int(d["status"][0]) == 1
            st = reconstruct_state(dp, stop, int(d["sig"][0][0]) |
                                   (int(d["sig"][0][1]) << prog.num_qubits),
                                   int(d["c"][0]), d["amps"][0])
            rs = ref["state"]
            assert st["ph"] == rs["ph"] and st["idx"] == rs["idx"]
            assert_chi_close(st["amp"], rs["amp"], context=(stop, shot))


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
def test_lane_per_shot_matches_warp_per_shot(rng):
    """The batched lane-per-shot (narrow) interpreter and the warp-per-shot
    (wide) interpreter give identical records, statuses and counters on
    random programs (chi dims crossing the narrow limit back and forth), the
    d=3 and the grown d=5 MSC workloads."""
    from paper_2512_23037_b200.msc import msc_circuit, msc_grown_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    rnd = random.Random(21)
    progs = [apply_noise_model(msc_circuit(3), 3e-3),
             apply_noise_model(msc_grown_circuit(5), 3e-3)]
    for _ in range(12):
        n = rnd.choice((5, 9, 16))
        progs.append(_random_program(rnd, n, 90, rnd.choice((6, 12, 20)), 0.1))
    eng = get_engine(0)
    for i, prog in enumerate(progs):
        p = Program(compile_program(prog))
        flags = _lib.GS_POSTSELECT * (i % 2) | (_lib.GS_RNG_PHILOX if rng == "philox" else 0)
        shots = 3000 if i < 2 else 200
        a = eng.run_records(p, Engine.params(5 + i, 0, shots, 4096, flags))
        b = eng.run_records(p, Engine.params(5 + i, 0, shots, 4096,
                                             flags | _lib.GS_WIDE_ONLY))
        for x, y in zip(a, b):
            assert np.array_equal(x, y), i
        ca = eng.run_counters(p, Engine.params(5 + i, 0, shots, 4096, flags))
        cb = eng.run_counters(p, Engine.params(5 + i, 0, shots, 4096,
                                               flags | _lib.GS_WIDE_ONLY))
        assert np.array_equal(ca, cb), i


@pytest.mark.parametrize("rng", ["splitmix", "philox"])
def test_section_chunking_invariance(rng):
    """Shots pass through the narrow/wide section queues in chunks; records
    and counters do not depend on the chunk size (incl. ragged last
    chunks) or on the launch shape."""
    from paper_2512_23037_b200.msc import msc_grown_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    prog = apply_noise_model(msc_grown_circuit(5), 3e-3)
    p = Program(compile_program(prog))
    eng = get_engine(0)
    flags = _lib.GS_POSTSELECT | (_lib.GS_RNG_PHILOX if rng == "philox" else 0)
    ref = eng.run_records(p, Engine.params(9, 100, 5000, 4096, flags))
    for kw in ({"chunk_shots": 1000}, {"chunk_shots": 333}, {"chunk_shots": 64, "blocks": 7},
               {"warps_per_block": 1}):
        got = eng.run_records(p, Engine.params(9, 100, 5000, 4096, flags, **kw))
        for x, y in zip(ref, got):
            assert np.array_equal(x, y), kw
    c0 = eng.run_counters(p, Engine.params(9, 100, 5000, 4096, flags))
    c1 = eng.run_counters(p, Engine.params(9, 100, 5000, 4096, flags, chunk_shots=777))
    assert np.array_equal(c0, c1)


@pytest.mark.parametrize("flag", [0, _lib.GS_CHI_BLOCK, _lib.GS_SPARSE])
def test_dumps_restore_the_reduced_t_phase(flag):
    """Reduced-form T ops leave their global phase e^{+-i pi/8} out of chi
    and count it; dumps must restore it both inside the wide section that
    ran them (the kernel's count) and in a later narrow section (the static
    entry count of that section)."""
    text = ("H 0 1 2 3 4 5 6\nT 0 1 2 3 4 5\nT_DAG 6\n"   # k grows 0..7, wide from k=4
            "CX 0 1\nM 0 1 2 3\n"                         # back to k=3: narrow
            "H 0\nS 1\nCX 1 2\n")
    prog = parse_circuit(text)
    flat = list(prog.flat())
    eng = get_engine(0)
    t_last = max(i for i, ins in enumerate(flat) if ins.name in ("T", "T_DAG"))
    for stop in (t_last, len(flat) - 1):
        dp = compile_program(prog, stop_after=stop, keep_frames=True)
        p = Program(dp)
        for shot in range(4):
            seeds = np.array([derive_seed(6, shot)], dtype=np.uint64)
            d = eng.dump(p, Engine.params(6, 0, 1, 4096, flag, seeds=seeds))
            ref = orc.run_one_shot(flat, prog.num_qubits, orc.DrawStream("splitmix", 6, shot),
                                   4096, False, stop_after=stop, snapshot=True)
            assert int(d["status"][0]) == 1
            st = reconstruct_state(dp, stop, int(d["sig"][0][0]) |
                                   (int(d["sig"][0][1]) << prog.num_qubits),
                                   int(d["c"][0]), d["amps"][0])
            rs = ref["state"]
            assert st["ph"] == rs["ph"] and st["idx"] == rs["idx"], (stop, shot)
            assert_chi_close(st["amp"], rs["amp"], context=(stop, shot))


@pytest.mark.parametrize("flag", [0, _lib.GS_WIDE_ONLY, _lib.GS_CHI_BLOCK, _lib.GS_SPARSE])
def test_conditional_pair_fusion_matches_oracle(flag):
    """TF_FUSEQ pairs (T gates with a noise insertion between them) are fused
    only for shots whose Philox schedule has no candidate there: with noise
    strong enough that many shots do fire there, every shot's record and
    status must still equal the oracle's (which never fuses)."""
    from paper_2512_23037_b200.msc import msc_grown_circuit
    from paper_2512_23037_b200.noise import apply_noise_model
    from paper_2512_23037_b200.compiler import TF_FUSEQ, decode_header
    prog = apply_noise_model(msc_grown_circuit(5), 4e-3)
    dp = compile_program(prog)
    pc, n_q = 0, 0
    while pc < len(dp.ops):
        kind, ln, _, fl, _ = decode_header(int(dp.ops[pc]))
        n_q += kind == 1 and bool(fl & TF_FUSEQ)
        if kind == 0:
            break
        pc += ln
    assert n_q > 0
    got = _gpu_results(prog, 21, 48, 4096, False, rng="philox", flags_extra=flag)
    ref = _oracle_results(prog, 21, 48, 4096, False, mode="philox")
    assert got == ref
