"""One BASELINE config-4 point (random Clifford+T, n qubits, t T gates,
p=1e-3, post-selection) through run_batch: warm-up, then `--shots` shots
timed on the device.  For ncu captures of the large-chi forms:
    python scripts/c4_point.py 48 24 --shots 20000"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_23037_b200 import SamplerConfig, run_batch  # noqa: E402
from paper_2512_23037_b200.msc import config4_circuit  # noqa: E402
from paper_2512_23037_b200.noise import apply_noise_model  # noqa: E402
from paper_2512_23037_b200.sampler import _program_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int)
ap.add_argument("t", type=int)
ap.add_argument("--shots", type=int, default=20000)
ap.add_argument("--warm", type=int, default=2048)
ap.add_argument("--flags", default="", help="extra run flags, e.g. CHI_BLOCK,CHI_GLOBAL")
ap.add_argument("--blocks", type=int, default=0, help="resident blocks of the launches (0 = auto)")
args = ap.parse_args()
from paper_2512_23037_b200 import _lib  # noqa: E402
EXTRA = 0
for f in filter(None, args.flags.split(",")):
    EXTRA |= getattr(_lib, "GS_" + f)


class Cfg(SamplerConfig):
    def run_flags(self) -> int:
        return super().run_flags() | EXTRA


SamplerConfig = Cfg  # noqa: F811
if args.blocks:
    from paper_2512_23037_b200.engine import Engine
    _params = Engine.params

    def _with_blocks(*a, **kw):
        kw["blocks"] = args.blocks
        return _params(*a, **kw)

    Engine.params = staticmethod(_with_blocks)
prog = apply_noise_model(config4_circuit(args.n, args.t, seed=args.n + args.t), 1e-3)
if args.warm:
    run_batch(prog, SamplerConfig(shots=args.warm, master_seed=1, rng="philox"))
cfg = SamplerConfig(shots=args.shots, master_seed=args.n * 1000 + args.t, rng="philox",
                    postselect=True)
st = run_batch(prog, cfg)
p = _program_for(prog, cfg.dim_limit)
print(json.dumps({"n": args.n, "t": args.t, "shots": st.total_shots,
                  "device_shots_per_s": st.device_dict()["device_shots_per_s"],
                  "overflow": st.overflow_count, "max_dim": p.dp.max_dim,
                  "sections": p.sections(), "flags": args.flags, "blocks": args.blocks}))
