"""How much of the d=5 time is chi work?  Same circuit with T/T_DAG
replaced by S/S_DAG (Clifford proxy: chi stays one amplitude)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_23037_b200 import _lib, parse_circuit
from paper_2512_23037_b200.compiler import compile_program
from paper_2512_23037_b200.engine import Engine, Program
from paper_2512_23037_b200.msc import msc_circuit
from paper_2512_23037_b200.noise import apply_noise_model

eng = Engine(0)
flags = _lib.GS_POSTSELECT | _lib.GS_RNG_PHILOX
for p in (0.0, 1e-3):
    for variant in ("T", "S"):
        text = msc_circuit(5).serialize()
        if variant == "S":
            text = text.replace("T_DAG", "S_DAG").replace("\nT ", "\nS ")
        prog = parse_circuit(text)
        if p:
            prog = apply_noise_model(prog, p)
        P = Program(compile_program(prog))
        shots = 1 << 21
        eng.run_counters(P, Engine.params(1, 0, shots, 32768, flags))
        c = eng.run_counters(P, Engine.params(2, shots, shots, 32768, flags))
        ms = eng.last_kernel_ms
        print(json.dumps({"p": p, "gates": variant, "shots_per_s": shots / (ms * 1e-3),
                          "discard": int(c[_lib.GS_C_DISCARDED]) / shots}), flush=True)
