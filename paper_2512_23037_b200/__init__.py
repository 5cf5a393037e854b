"""B200-native (sm_100a) shot-parallel generalized-stabilizer sampler.

Drop-in for the shot engine of the reference ``gstab`` package
(arXiv 2512.23037, SOFT): parse a circuit, add uniform depolarizing noise,
and sample shots on the GPU with post-selection and logical-error counters.

    from paper_2512_23037_b200 import parse_circuit, apply_noise_model, \
        SamplerConfig, run_batch
    prog = apply_noise_model(parse_circuit(text), 1e-3)
    stats = run_batch(prog, SamplerConfig(shots=10**7, postselect=True))

The sampling path is ``compiler.compile_program`` (host, once per circuit)
-> ``libgstab_sm100a.so`` (CUDA sections: lane-per-shot for chi dimension
<= 4 or 5, warp-per-shot above, a block of warps per shot for chi >= 2^14).
There is no CPU fallback.
"""

from .circuit import (Block, CircuitProgram, Instruction, ParseError,
                      PauliProduct, Rec, compute_stats, parse_circuit)
from .noise import NoiseModelError, NoiseOp, apply_noise_model
from .compiler import CompileError, DeviceProgram, compile_program
from .sampler import (CorruptStateError, UnsupportedCircuitError, RunStats, SamplerConfig, ShotBatch,
                      ShotContext, ShotResult, ShotStatus, bayes_interval,
                      derive_seed, run_batch, run_shot, sample,
                      throughput_bench)

__version__ = "0.1.0"

__all__ = [
    "Block", "CircuitProgram", "Instruction", "ParseError", "PauliProduct",
    "Rec", "compute_stats", "parse_circuit", "NoiseModelError", "NoiseOp",
    "apply_noise_model", "CompileError", "DeviceProgram", "compile_program",
    "CorruptStateError", "UnsupportedCircuitError", "RunStats", "SamplerConfig", "ShotBatch",
    "ShotContext", "ShotResult", "ShotStatus", "bayes_interval", "derive_seed",
    "run_batch", "run_shot", "sample", "throughput_bench", "__version__",
]
