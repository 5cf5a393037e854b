"""Compiler correctness on CPU: the frame model (a CPU transliteration of the
device interpreter) must reproduce the reference's golden per-shot results
bit-for-bit and its state snapshots to 1e-10 relative per entry."""

from chi_check import assert_chi_close

import numpy as np
import pytest

import frame_model as FM
from paper_2512_23037_b200 import compiler as C
from paper_2512_23037_b200.circuit import parse_circuit
from paper_2512_23037_b200.frames import reconstruct_state


def test_frame_model_matches_golden_shots(golden_shots):
    for fx in golden_shots:
        if fx["name"].startswith("config1"):
            nshots = 40
        else:
            nshots = len(fx["shots"])
        prog = parse_circuit(fx["text"])
        dp = C.compile_program(prog)
        for shot in range(nshots):
            res = FM.run_shot(dp, "splitmix", fx["master"], shot,
                              fx["capacity"], fx["postselect"])
            got = FM.as_shot_result(dp, res)
            assert got == fx["shots"][shot], (fx["name"], shot)


def test_frame_model_states(golden_states):
    for fx in golden_states:
        prog = parse_circuit(fx["text"])
        for snap in fx["snaps"]:
            dp = C.compile_program(prog, stop_after=snap["i"], keep_frames=True)
            res = FM.run_shot(dp, "splitmix", fx["master"], fx["shot"], 4096,
                              False, want_state=True)
            st = reconstruct_state(dp, snap["i"], res["sig"], res["c"], res["A"])
            assert st["xs"] == snap["xs"] and st["zs"] == snap["zs"]
            assert st["ph"] == snap["ph"], (fx["text"], snap["i"])
            assert st["idx"] == snap["idx"], (fx["text"], snap["i"])
            assert_chi_close(st["amp"], snap["amp"])


def test_frame_model_random_programs_vs_oracle():
    """Compiler check on programs with MPP flips, R/MR, SWAP-controlled
    feedback, repeated noise targets, both RNG modes and tiny capacities."""
    import random
    from oracle import gstab_oracle as orc
    from tests_helpers import random_program
    rng = random.Random(11)
    for it in range(40):
        prog = random_program(rng)
        flat = list(prog.flat())
        dp = C.compile_program(prog)
        mode = "philox" if it % 2 else "splitmix"
        cap = rng.choice((2, 8, 4096))
        for shot in range(4):
            post = shot % 2 == 0
            ref = orc.run_one_shot(flat, prog.num_qubits,
                                   orc.DrawStream(mode, 5, shot), cap, post)
            got = FM.as_shot_result(dp, FM.run_shot(dp, mode, 5, shot, cap, post))
            want = {"status": ref["status"],
                    "observables": {str(k): v for k, v in sorted(ref["observables"].items())},
                    "discarded_detector": ref["discarded_detector"],
                    "overflow_instruction": ref["overflow_instruction"],
                    "record": ref["record"]}
            assert got == want, (it, shot, prog.serialize())
