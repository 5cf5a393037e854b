"""Large-sample statistical parity (opt-in: GS_LONG_STATS=1, ~8 min on one
B200 + 16 host cores): the Table-2 d=5 and d=3 cultivation circuits, the
grown d=5 proxy, the d=3 proxy and BASELINE config 3, post-selected, sampled with billions of
Philox shots on the GPU against reference-stream (SplitMix) shots of the
CPU oracle (GS_LONG_SCALE scales both sample sizes).  Discard rate and
logical-error rate must agree (Bayes-factor-1000 intervals overlap and
z < 4.5, tests/stats_check.py); the summary line
is printed for profiles/.

    GS_LONG_STATS=1 python -m pytest tests/test_gpu_statistics_long.py -m gpu -s
"""

import json
import math
import os
import time

import pytest

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("GS_LONG_STATS") != "1",
                                 reason="opt-in long run (GS_LONG_STATS=1)")]

from oracle import gstab_oracle as orc
from paper_2512_23037_b200 import SamplerConfig, run_batch
from paper_2512_23037_b200.msc import (injection_circuit, msc_circuit, msc_d3_circuit,
                                       msc_d5_circuit, msc_grown_circuit)
from paper_2512_23037_b200.noise import apply_noise_model
from stats_check import assert_rates_agree, z_score as _z


WORKLOADS = {
    # name: (builder, p, default GPU shots, default CPU shots)
    # the round-2 headline (BASELINE config 5) and config 2 with Table 2's shape
    "msc_d5_table2": (msc_d5_circuit, 1e-3, 2 * 10 ** 9, 60000),
    "msc_d3_table2": (msc_d3_circuit, 1e-3, 10 ** 9, 200000),
    "msc_d5_grown_proxy": (lambda: msc_grown_circuit(5), 1e-3, 4 * 10 ** 9, 60000),
    # BASELINE config 2: MSC d=3, 1e8 shots on one B200
    "msc_d3_proxy": (lambda: msc_circuit(3), 1e-3, 10 ** 8, 200000),
    # BASELINE config 3: d=3 injection + 3 rounds, p=5e-4
    "d3_injection_3_rounds": (lambda: injection_circuit(3, 3), 5e-4, 10 ** 9, 100000),
}


@pytest.mark.parametrize("name", sorted(WORKLOADS))
def test_discard_and_logical_error_rates_large_sample(name):
    build, p_noise, gpu_default, cpu_default = WORKLOADS[name]
    scale = float(os.environ.get("GS_LONG_SCALE", "1"))
    gpu_shots = int(gpu_default * scale)
    cpu_shots = int(cpu_default * scale)
    prog = apply_noise_model(build(), p_noise)
    t0 = time.perf_counter()
    gpu = run_batch(prog, SamplerConfig(shots=gpu_shots, master_seed=2026,
                                        postselect=True, rng="philox"))
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    cpu = orc.run_counters_parallel(prog, cpu_shots, os.cpu_count() or 1,
                                    master_seed=7, mode="splitmix", postselect=True)
    t_cpu = time.perf_counter() - t0
    z_disc = _z(gpu.discarded_shots, gpu.total_shots, cpu["discarded"], cpu["total"])
    z_ler = _z(gpu.logical_error_shots, gpu.preserved_shots,
               cpu["error_shots"], max(cpu["preserved"], 1))
    lo, hi = gpu.bayes_interval
    summary = {
        "workload": name, "p": p_noise,
        "gpu": {"shots": gpu.total_shots, "rng": "philox", "wall_s": t_gpu,
                "shots_per_s": gpu.total_shots / t_gpu,
                "discard_rate": gpu.discard_rate,
                "logical_error_rate": gpu.logical_error_rate,
                "bayes_interval": [lo, hi], "overflow": gpu.overflow_count},
        "cpu_oracle": {"shots": cpu["total"], "rng": "splitmix", "wall_s": t_cpu,
                       "shots_per_s": cpu["total"] / t_cpu,
                       "discard_rate": cpu["discarded"] / cpu["total"],
                       "logical_error_rate": cpu["error_shots"] / max(cpu["preserved"], 1),
                       "processes": os.cpu_count()},
        "z_discard": z_disc, "z_logical_error": z_ler,
    }
    print("LONG_STATS " + json.dumps(summary))
    assert gpu.total_shots == gpu_shots and gpu.overflow_count == 0
    assert_rates_agree(gpu.discarded_shots, gpu.total_shots, cpu["discarded"], cpu["total"])
    assert_rates_agree(gpu.logical_error_shots, gpu.preserved_shots,
                       cpu["error_shots"], cpu["preserved"])


def test_philox_production_stream_vs_the_reference_stream_at_scale():
    """The benchmarked Philox stream against the reference's own SplitMix
    stream at scale: the GPU's SplitMix records are bit-identical to the
    reference's (tests/test_gpu_configs.py goldens), so a billion-shot
    SplitMix run on the GPU is a reference-equivalent sample of the same
    law.  Discard and logical-error rates of the two streams on the Table-2
    d=5 circuit must agree (Bayes-factor-1000 intervals, z < 4.5)."""
    from paper_2512_23037_b200.msc import msc_d5_circuit
    scale = float(os.environ.get("GS_LONG_SCALE", "1"))
    shots = int(2 * 10 ** 9 * scale)
    prog = apply_noise_model(msc_d5_circuit(), 1e-3)
    out = {}
    for rng in ("philox", "splitmix"):
        t0 = time.perf_counter()
        st = run_batch(prog, SamplerConfig(shots=shots, master_seed=4242 if rng == "philox" else 99,
                                           postselect=True, rng=rng))
        out[rng] = (st, time.perf_counter() - t0)
    (a, ta), (b, tb) = out["philox"], out["splitmix"]
    summary = {"workload": "msc_d5_table2", "p": 1e-3, "shots_each": shots,
               "philox": {"discard_rate": a.discard_rate, "logical_error_rate": a.logical_error_rate,
                          "logical_error_shots": a.logical_error_shots, "wall_s": ta},
               "splitmix_reference_stream": {"discard_rate": b.discard_rate,
                                             "logical_error_rate": b.logical_error_rate,
                                             "logical_error_shots": b.logical_error_shots, "wall_s": tb},
               "z_discard": _z(a.discarded_shots, a.total_shots, b.discarded_shots, b.total_shots),
               "z_logical_error": _z(a.logical_error_shots, a.preserved_shots,
                                     b.logical_error_shots, b.preserved_shots)}
    print("LONG_STATS " + json.dumps(summary))
    assert_rates_agree(a.discarded_shots, a.total_shots, b.discarded_shots, b.total_shots)
    assert_rates_agree(a.logical_error_shots, a.preserved_shots,
                       b.logical_error_shots, b.preserved_shots)
