"""Where the e2e time of the headline goes (parse, host compile, narrow-limit
probe, waves: device vs host), on the GPU:  python scripts/e2e_breakdown.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_23037_b200 import SamplerConfig, parse_circuit, run_batch  # noqa: E402
from paper_2512_23037_b200.engine import Engine, get_engine  # noqa: E402
from paper_2512_23037_b200.msc import msc_d5_circuit  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402
from paper_2512_23037_b200.sampler import _program_for, tuned_flags  # noqa: E402

text = apply_noise_model(msc_d5_circuit(), 1e-3).serialize()
eng = get_engine(0)
warm = parse_circuit(text)
run_batch(warm, SamplerConfig(shots=1 << 23, master_seed=1, postselect=True, rng="philox"))
out = {}
shots = 1 << 28
cfg = SamplerConfig(shots=shots, master_seed=777, postselect=True, rng="philox")
t0 = time.perf_counter()
prog = parse_circuit(text)
t1 = time.perf_counter()
p = _program_for(prog, cfg.dim_limit)
t2 = time.perf_counter()
flags = cfg.run_flags() | tuned_flags(p, eng, cfg)
t3 = time.perf_counter()
dev = 0.0
done = 0
while done < shots:
    n = min(cfg.wave_shots, shots - done)
    eng.run_counters(p, Engine.params(777, (1 << 40) + done, n, cfg.effective_capacity, flags))
    dev += eng.last_kernel_ms * 1e-3
    done += n
t4 = time.perf_counter()
out = {"parse_s": t1 - t0, "compile_s": t2 - t1, "tune_s": t3 - t2, "waves_s": t4 - t3,
       "waves_device_s": dev, "waves": -(-shots // cfg.wave_shots),
       "host_per_wave_ms": 1e3 * ((t4 - t3) - dev) / -(-shots // cfg.wave_shots),
       "e2e_shots_per_s": shots / (t4 - t0), "device_shots_per_s": shots / dev}
print(json.dumps(out))
