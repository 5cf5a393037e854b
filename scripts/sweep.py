"""Throughput sweeps on one B200 (paper Fig. 3 / Fig. 4 analogues):
shots/s vs noise strength p (d=3 proxy, grown d=5 proxy) and vs batch
size (grown d=5, p=1e-3).
Device time from CUDA events inside gs_run_counters."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23037_b200 import _lib
from paper_2512_23037_b200.compiler import compile_program
from paper_2512_23037_b200.engine import Engine, Program
from paper_2512_23037_b200.msc import msc_circuit, msc_grown_circuit
from paper_2512_23037_b200.noise import apply_noise_model

eng = Engine(0)
flags = _lib.GS_POSTSELECT | _lib.GS_RNG_PHILOX
rows = []
CIRC = {3: lambda: msc_circuit(3), 5: lambda: msc_grown_circuit(5)}
for d in (3, 5):
    for p in (0.0, 5e-4, 1e-3, 2e-3, 5e-3, 1e-2):
        prog = apply_noise_model(CIRC[d](), p) if p else CIRC[d]()
        P = Program(compile_program(prog))
        shots = 1 << 21
        eng.run_counters(P, Engine.params(1, 0, shots, 32768, flags))
        c = eng.run_counters(P, Engine.params(2, shots, shots, 32768, flags))
        ms = eng.last_kernel_ms
        rows.append({"sweep": "noise", "d": d, "p": p, "shots": shots,
                     "shots_per_s": shots / (ms * 1e-3),
                     "discard_rate": int(c[_lib.GS_C_DISCARDED]) / shots,
                     "model_bytes_per_shot": int(c[_lib.GS_C_MODEL_BYTES]) / shots})
        print(json.dumps(rows[-1]), flush=True)
prog = apply_noise_model(msc_grown_circuit(5), 1e-3)
P = Program(compile_program(prog))
for lg in range(8, 25, 2):
    shots = 1 << lg
    eng.run_counters(P, Engine.params(1, 0, shots, 32768, flags))
    c = eng.run_counters(P, Engine.params(3, 0, shots, 32768, flags))
    ms = eng.last_kernel_ms
    rows.append({"sweep": "batch", "d": 5, "p": 1e-3, "shots": shots,
                 "shots_per_s": shots / (ms * 1e-3)})
    print(json.dumps(rows[-1]), flush=True)
