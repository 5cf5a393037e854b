"""Benchmark: MSC d=5 (Table 2 shape: 42 q, 741 gates, 72 T) shots/s on 1..8
B200, p=1e-3, post-selection.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step = one persistent-kernel launch that samples ``--shots-per-step`` shots
per GPU (weak scaling: rank r takes global shots [step*N*S + r*S, +S)).
Timing: barrier + synchronize on both sides of the K timed steps; every step
is bracketed by CUDA events on the launching stream; L2 is flushed (256 MiB
write) between steps outside the events; the max over ranks is reported.

Extra keys: ``roofline`` (state-touch model bytes counted on device / kernel
time vs measured HBM copy bandwidth), ``cpu_baseline`` (the reference
itself -- oracle/_ref, built by oracle/build_ref.py with its Cython backend --
through its own run_batch on all host cores, rank 0, bounded sample; the
oracle port when oracle/_ref is absent or with --ref-port), ``e2e`` (the public
C-ABI path with host buffers: program upload + launch + counter readback),
``clocks`` (nvidia-smi sampled during the timed region) and
``gpu_launches``.

``--impl reference``: each step is one reference ``run_batch`` call
(threads = all host cores, batch_size=1024, post-selection) over a bounded
sample of the same workload, parsed and noised by the reference itself.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MSC d=5 shots/sec at 1/2/4/8 B200 (vs CPU ref); achieved HBM GB/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def _ncu_latest(workload: str, shots: int):
    """DRAM traffic + issue utilisation of the section kernels from the
    committed ncu --set full capture (profiles/ncu_latest.json) of this
    workload (per-shot DRAM bytes; `shots` kept for the call signature)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_latest.json")) as fh:
            d = json.load(fh)
    except Exception:
        return None
    if d.get("workload") != workload:
        return None
    return d


def _micro_peaks():
    """Measured SMEM / FP64 / issue ceilings of this B200 (scripts/peaks.cu,
    run on the box; profiles/peaks.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def _ceiling(mp, key, sm_mhz):
    """A measured per-SM-per-clock ceiling at this run's SM clock (GB/s,
    Gflop/s or G warp-inst/s)."""
    per = mp[key]["per_sm_per_clk"] if isinstance(mp.get(key), dict) else None
    if per is None:
        return None
    return per * mp["sms"] * (sm_mhz or mp["sm_clock_max_mhz"]) * 1e-3


def _roofline(secs, ncu, total_shots, value, model_bytes, hbm_peak, hbm_src, sm_mhz=None):
    """Roofline of the dominant section kernel against the resource that
    binds it: chi lives in shared memory, so HBM carries only
    the section queues; the kernels are issue-bound.

    * issue: warp instructions of the dominant launch per shot (ncu capture
      of the same workload, profiles/ncu_latest.json) x the shots it ran /
      its live device time (CUDA events around that launch in this run), vs
      the measured issue ceiling (profiles/peaks.json: warp instructions per
      SM per clock of FP32-FMA / FMA+LOP3 chains x SMs x this run's SM clock);
    * smem: SURVEY §8(d) state-touch bytes the dominant section executed
      (counted on the device, GS_SECTION_STATS) / its live time, vs the
      measured LDS.128+STS.128 ceiling (per SM per clock x SMs x clock) --
      the 24 B/entry model includes the
      8-byte index the dense chi layout keeps implicit, so this overstates
      the shared-memory bytes actually moved (ncu wavefronts: smem_pct);
    * hbm: ncu DRAM bytes per shot x this run's rate, vs the measured copy
      bandwidth (MEASURED_PEAKS.json)."""
    mp = _micro_peaks()
    out = {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
           "traffic": None}
    if not secs:
        return out
    tot_ms = sum(s["device_ms"] for s in secs) or 1.0
    i = max(range(len(secs)), key=lambda j: secs[j]["device_ms"])
    d = secs[i]
    dev_s = d["device_ms"] * 1e-3
    launches = max(d["launches"], 1)
    sec_rows = [{"section": j, "kernel": s["kernel"], "pc0": s["pc0"],
                 "shots_in": s["shots_in"], "device_ms": s["device_ms"],
                 "share": s["device_ms"] / tot_ms,
                 "model_gbs": s["model_bytes"] / max(s["device_ms"] * 1e-3, 1e-12) / 1e9}
                for j, s in enumerate(secs)]
    kern = None
    if ncu and len(ncu.get("kernels", [])) == len(secs):
        kern = ncu["kernels"][i]
    smem_ach = d["model_bytes"] / dev_s / 1e9 if dev_s > 0 else None
    out.update({"kernel": "%s_kernel (section %d of %d)" % (d["kernel"], i, len(secs)),
                "kernel_share": d["device_ms"] / tot_ms,
                "launches": d["launches"],
                "shots_per_launch": d["shots_in"] / launches,
                "model_bytes_per_launch": d["model_bytes"] / launches,
                "device_ms_per_launch": d["device_ms"] / launches,
                "sections": sec_rows})
    smem_peak = _ceiling(mp, "smem_ldst_gbs", sm_mhz) if mp else None
    issue_peak = (mp["issue_ipc_per_sm"] * mp["sms"] * (sm_mhz or mp["sm_clock_max_mhz"]) * 1e-3
                  if mp and "issue_ipc_per_sm" in mp else None)
    if smem_peak and smem_ach is not None:
        out["smem"] = {"achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
                       "frac": smem_ach / smem_peak,
                       "bytes": "SURVEY 8(d) state-touch model, device-counted"}
    if kern:
        scale = total_shots / ncu["shots_in_capture"]    # capture = one chunk
        inst = kern["warp_instructions"] * scale
        out["issue_active_pct_ncu"] = kern["issue_active_pct"]
        out["fp64_pipe_pct_ncu"] = kern["fp64_pipe_pct"]
        out["smem_wavefront_pct_ncu"] = kern.get("smem_wavefront_pct")
        out["ncu_capture"] = ncu["capture"]
        out["traffic"] = kern["dram_bytes"] * scale / launches
        if issue_peak:
            ach = inst / dev_s / 1e9
            out.update({"bound": "issue", "achieved": ach, "peak": issue_peak,
                        "unit": "Gwarp-inst/s", "frac": ach / issue_peak,
                        "peak_source": "measured (profiles/peaks.json: scripts/peaks.cu "
                                       "issue IPC per SM x SMs x this run's SM clock)"})
    if out["bound"] is None and "smem" in out:
        out.update({"bound": "smem", "achieved": out["smem"]["achieved"],
                    "peak": out["smem"]["peak"], "unit": "GB/s", "frac": out["smem"]["frac"],
                    "peak_source": "measured (profiles/peaks.json, LDS.128+STS.128)"})
    if ncu:
        dram = ncu["dram_bytes_per_shot"] * value / 1e9
        out["hbm"] = {"dram_achieved_gbs": dram, "peak": hbm_peak, "frac": dram / hbm_peak,
                      "peak_source": hbm_src}
    out["model_bytes_per_shot"] = model_bytes / max(total_shots, 1)
    return out


def _peaks():
    try:
        with open(PEAKS) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


WORKLOADS = {
    # BASELINE config 5: d=5 cultivation with Table 2's shape (42 q, 741
    # gates, 477 2Q, 93 M, 72 T, support 19, T-depth 6; msc.msc_d5_circuit)
    "msc_d5": ("msc_d5_table2", lambda m: m.msc_d5_circuit()),
    # round-1 headline: d=3 -> d=5 grown proxy (42 q, 72 T, 542 gates)
    "msc_d5_grown": ("msc_d5_grown_proxy", lambda m: m.msc_grown_circuit(5)),
    # all checks at d=5 (42 q, 96 T; more chi work)
    "msc_d5_2check": ("msc_d5_2check_proxy", lambda m: m.msc_circuit(5)),
    # BASELINE config 2: d=3 cultivation with Table 2's shape
    "msc_d3": ("msc_d3_table2", lambda m: m.msc_d3_circuit()),
    "msc_d3_proxy": ("msc_d3_proxy", lambda m: m.msc_circuit(3)),
    # BASELINE config 3 (quoted at p=5e-4: see DEFAULT_P)
    "injection_d3": ("d3_injection_3_rounds", lambda m: m.injection_circuit(3, 3)),
    # BASELINE config 1 and two points of the config-4 sweep
    "config1": ("config1_random_n8_t4", lambda m: m.config1_circuit(1)),
    "config4_n32_t24": ("config4_random_n32_t24", lambda m: m.config4_circuit(32, 24, seed=56)),
    "config4_n64_t32": ("config4_random_n64_t32", lambda m: m.config4_circuit(64, 32, seed=96)),
}
# noise strength each BASELINE config is quoted at (others: 1e-3)
DEFAULT_P = {"injection_d3": 5e-4}


def _workload(key: str, p: float):
    from paper_2512_23037_b200 import msc
    from paper_2512_23037_b200.noise import apply_noise_model
    from paper_2512_23037_b200.circuit import compute_stats
    name, make = WORKLOADS[key]
    base = make(msc)
    return name, apply_noise_model(base, p), compute_stats(base).as_dict(), base.serialize()


def physical_gpu_id(dev: int) -> str:
    """nvidia-smi -i selector of CUDA ordinal `dev`: its UUID (immune to a
    CUDA_VISIBLE_DEVICES remap), else the ordinal."""
    try:
        import torch
        u = str(torch.cuda.get_device_properties(dev).uuid)
        if u and u != "None":
            return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        pass
    return str(dev)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region
    (`index`: an nvidia-smi -i selector, see physical_gpu_id)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = sorted(float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit())
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(self.rows), "reasons": sorted(reasons)}


def cpu_baseline(prog, seconds: float, mode: str, p_noise: float):
    """Time the CPU oracle port on all host cores for a bounded sample.

    Always in the reference's own random stream (SHA-1 seeds + SplitMix,
    ref sampler.py:37-61): the reference has no Philox mode, and the port's
    pure-Python Philox is ~3x slower than its SplitMix path, which would
    understate the CPU.  `mode` is recorded only."""
    mode_run = "splitmix"
    from oracle import gstab_oracle as orc
    cores = os.cpu_count() or 1
    # calibrate on one core after a warm-up call (first-call costs: table
    # builds, numpy dispatch), then size the parallel sample to ~`seconds`
    # so the process-pool start-up is a small part of it
    orc.run_counters(prog, 8, 1, mode=mode_run, postselect=True)
    t0 = time.perf_counter()
    orc.run_counters(prog, 64, 1, mode=mode_run, postselect=True)
    per_shot = max((time.perf_counter() - t0) / 64, 1e-5)
    shots = max(cores * 32, int(seconds * cores / per_shot))
    t0 = time.perf_counter()
    c = orc.run_counters_parallel(prog, shots, cores, master_seed=1, mode=mode_run,
                                  postselect=True)
    dt = time.perf_counter() - t0
    return {"value": c["total"] / dt, "unit": "shots/s", "cores": cores,
            "kind": "port",
            "sample": "%d shots of the same workload (oracle/gstab_oracle.py, "
                      "%d processes, %.1f s, reference SplitMix stream; the GPU "
                      "arm's stream: %s)" % (c["total"], cores, dt, mode),
            "discard_rate": c["discarded"] / max(c["total"], 1)}


def _ref_program(text: str, p: float):
    """The workload parsed and noised by the reference itself (oracle/_ref:
    gstab.circuit.parse_circuit, gstab.noise.apply_noise_model)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from build_ref import import_reference
    gstab = import_reference()
    prog = gstab.circuit.parse_circuit(text)
    return gstab, (gstab.noise.apply_noise_model(prog, p) if p > 0 else prog)


def reference_run(gstab, prog, shots: int, shot_begin: int, cores: int):
    """One bounded sample through the reference's own public API:
    gstab.sampler.run_batch(prog, SamplerConfig(threads=cores,
    batch_size=1024, postselect=True)) (ref sampler.py:348-382), timed by
    the wall clock around the call (its process pool included).  The shot
    range is moved by re-keying the master seed (seeds are per (master,
    shot), ref sampler.py:37-42)."""
    cfg = gstab.sampler.SamplerConfig(shots=shots, master_seed=1 + shot_begin,
                                      threads=cores, batch_size=1024,
                                      postselect=True)
    t0 = time.perf_counter()
    st = gstab.sampler.run_batch(prog, cfg)
    dt = time.perf_counter() - t0
    return st, dt


def reference_baseline(text: str, p: float, seconds: float):
    """The real reference (oracle/_ref, Cython backend) on all host cores
    for a bounded ~`seconds` sample of the workload, in its own SplitMix
    stream."""
    gstab, prog = _ref_program(text, p)
    cores = os.cpu_count() or 1
    # calibrate on one core (first call pays imports / dispatch), then size
    # the parallel sample
    cal = gstab.sampler.SamplerConfig(shots=8, master_seed=99, postselect=True)
    gstab.sampler.run_batch(prog, cal)
    cal = gstab.sampler.SamplerConfig(shots=48, master_seed=98, postselect=True)
    t0 = time.perf_counter()
    gstab.sampler.run_batch(prog, cal)
    per_shot = max((time.perf_counter() - t0) / 48, 1e-5)
    shots = max(cores * 64, int(seconds * cores / per_shot) // 1024 * 1024)
    st, dt = reference_run(gstab, prog, shots, 0, cores)
    return {"value": st.total_shots / dt, "unit": "shots/s", "cores": cores,
            "kind": "reference", "backend": gstab.backend.name(),
            "sample": "%d shots of the same workload through the reference's "
                      "run_batch (oracle/_ref gstab, %s backend, threads=%d, "
                      "batch_size=1024, %.1f s, its SplitMix stream)"
                      % (st.total_shots, gstab.backend.name(), cores, dt),
            "discard_rate": st.discarded_shots / max(st.total_shots, 1)}


def _have_reference() -> bool:
    return os.path.isfile(os.path.join(ROOT, "oracle", "_ref", "gstab", "sampler.py"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--shots-per-step", type=int, default=1 << 24)
    ap.add_argument("--workload", default="msc_d5", choices=sorted(WORKLOADS))
    ap.add_argument("--p", type=float, default=None,
                    help="depolarizing strength (default: the workload's BASELINE p)")
    ap.add_argument("--rng", default="philox", choices=["philox", "splitmix"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-waves", type=int, default=16,
                    help="e2e sample: this many steps' worth of shots per GPU")
    ap.add_argument("--no-section-stats", action="store_true",
                    help="time the steps without per-section events / byte attribution")
    ap.add_argument("--ref-port", action="store_true",
                    help="time the oracle port instead of the reference (oracle/_ref)")
    ap.add_argument("--chi-global", action="store_true")
    ap.add_argument("--chi-smem", action="store_true")
    ap.add_argument("--wpb", type=int, default=0)
    ap.add_argument("--wide-only", action="store_true")
    ap.add_argument("--narrow-k", default="auto", choices=["auto", "4", "5"],
                    help="narrow (lane-per-shot) chi limit; auto = timed per program")
    ap.add_argument("--fixed-batch", action="store_true",
                    help="keep --shots-per-step even when a step is shorter than 0.2 s")
    ap.add_argument("--print-sections", action="store_true",
                    help="print the number of section launches per chunk and exit")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.p is None:
        args.p = DEFAULT_P.get(args.workload, 1e-3)
    workload, prog, stats, text = _workload(args.workload, args.p)
    config = {"workload": workload, "noise_p": args.p, "postselect": True,
              "rng": args.rng, "shots_per_step_per_gpu": args.shots_per_step,
              "circuit": stats, "parallelism": "shot-dp%d" % world,
              "l2": "flushed between steps (256 MiB write, untimed)"}

    if args.impl == "reference":
        if rank != 0:
            return 0
        cores = os.cpu_count() or 1
        if _have_reference() and not args.ref_port:
            # the reference itself: each step is one run_batch call over a
            # bounded sample of the workload on all host cores
            gstab, rprog = _ref_program(text, args.p)
            cal = gstab.sampler.SamplerConfig(shots=48, master_seed=98, postselect=True)
            gstab.sampler.run_batch(rprog, cal)
            t0 = time.perf_counter()
            gstab.sampler.run_batch(rprog, cal)
            per_shot = max((time.perf_counter() - t0) / 48, 1e-5)
            step_s = max(1.0, args.cpu_seconds / 4)
            shots = max(cores * 64, int(step_s * cores / per_shot) // 1024 * 1024)
            tot_shots = tot_s = 0.0
            disc = 0
            for s_ in range(args.warmup + args.steps):
                st, dt = reference_run(gstab, rprog, shots, s_ * shots, cores)
                if s_ >= args.warmup:
                    tot_shots += st.total_shots
                    tot_s += dt
                    disc += st.discarded_shots
            v = tot_shots / tot_s
            cb = {"value": v, "unit": "shots/s", "cores": cores, "kind": "reference",
                  "backend": gstab.backend.name(),
                  "sample": "%d shots per step through the reference's run_batch "
                            "(oracle/_ref gstab, %s backend, threads=%d, "
                            "batch_size=1024, ~%.1f s per step, its SplitMix stream)"
                            % (shots, gstab.backend.name(), cores, tot_s / args.steps),
                  "discard_rate": disc / max(tot_shots, 1)}
            ms = 1000.0 * tot_s / args.steps
        else:
            vals = []
            samples = []
            for _ in range(args.warmup + args.steps):
                cb = cpu_baseline(prog, max(2.0, args.cpu_seconds / 3), args.rng, args.p)
                vals.append(cb["value"])
                samples.append(cb)
            v = sorted(vals[args.warmup:])[len(vals[args.warmup:]) // 2]
            cb = samples[-1]
            cb["value"] = v
            ms = 1000.0 / v if v else None
        line = {"metric": METRIC, "value": v, "unit": "shots/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded SplitMix noise, the reference's own "
                        "stream, on the generated MSC workload)",
                "config": config, "cpu_baseline": cb,
                "e2e": {"value": v, "unit": "shots/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2512_23037_b200 import _lib
    from paper_2512_23037_b200.compiler import compile_program
    from paper_2512_23037_b200.engine import Engine, Program, get_engine

    dev = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("GS_DIST_BACKEND", "nccl")   # gloo: CI on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    dp = compile_program(prog)
    P = Program(dp)
    if args.print_sections:
        print(P.sections((_lib.GS_WIDE_ONLY if args.wide_only else 0) |
                         (_lib.GS_NARROW_K5 if args.narrow_k == "5" else 0)))
        return 0
    eng = get_engine(dev)   # the process-wide engine run_batch (e2e) also uses
    flags = _lib.GS_POSTSELECT | (_lib.GS_RNG_PHILOX if args.rng == "philox" else 0)
    if args.chi_global:
        flags |= _lib.GS_CHI_GLOBAL
    if args.chi_smem:
        flags |= _lib.GS_CHI_SMEM
    if args.wide_only:
        flags |= _lib.GS_WIDE_ONLY
    # narrow chi limit 4 or 5: timed on a probe per program (Program.narrow_flag;
    # results identical either way), rank 0's choice on every rank
    if args.narrow_k == "auto":
        nf = P.narrow_flag(eng, flags, 32768)
        if world > 1:
            t = torch.tensor([nf], dtype=torch.int64, device="cuda")
            dist.broadcast(t, 0)
            nf = int(t.item())
    else:
        nf = _lib.GS_NARROW_K5 if args.narrow_k == "5" else 0
    flags |= nf
    config["narrow_kn"] = 5 if nf else 4
    if getattr(P, "narrow_tuning", None):
        config["narrow_tuning"] = P.narrow_tuning
    S = args.shots_per_step
    nc = P.num_counters
    stream = torch.cuda.current_stream()
    counters = torch.zeros(nc, dtype=torch.int64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def launch(step, fl=None):
        base = step * world * S + rank * S
        par = Engine.params(12345, base, S, 32768, flags if fl is None else fl,
                            warps_per_block=args.wpb)
        eng.run_counters_async(P, par, counters.data_ptr(), stream.cuda_stream)

    for w in range(args.warmup):
        launch(w)
    torch.cuda.synchronize()
    # fast workloads: grow the batch so a step lasts >= ~0.2 s (the clock
    # sampler needs the timed region to span several 100 ms samples); the
    # headline workload (2^24 shots, ~0.27 s per step) is unaffected
    if not args.fixed_batch:
        t0 = time.perf_counter()
        launch(args.warmup)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        while dt * (S / args.shots_per_step) < 0.2 and S < (1 << 31):
            S *= 2
        if world > 1:   # every rank must use the same batch
            t = torch.tensor([S], dtype=torch.int64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            S = int(t.item())
        if S != args.shots_per_step:
            config["shots_per_step_per_gpu"] = S
            launch(args.warmup)
            torch.cuda.synchronize()
    counters.zero_()
    # per-section device time (CUDA events around each section launch, on
    # the launching stream) and device-counted model bytes, over exactly the
    # timed steps
    eng.section_stats(reset=True)
    tflags = flags | (0 if args.no_section_stats else _lib.GS_SECTION_STATS)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(physical_gpu_id(dev))
    clocks.start()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = eng.launches
    t_wall = time.perf_counter()
    for s in range(args.steps):
        flush.zero_()
        ev[s][0].record(stream)
        launch(args.warmup + s, tflags)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall
    ck = clocks.stop()
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    secs = eng.section_stats(reset=True)
    my_ms = sum(kernel_ms)
    launches = eng.launches - launches0
    if world > 1:
        t = torch.tensor([my_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.all_reduce(counters)            # the one data-path collective
    else:
        tot_ms = my_ms
    c = counters.cpu().numpy()
    total_shots = int(c[_lib.GS_C_TOTAL])
    value = total_shots / (tot_ms * 1e-3)
    model_bytes = int(c[_lib.GS_C_MODEL_BYTES])
    peak, peak_src = _peaks()

    # e2e through the public Python API, as a user calls it: a fresh
    # CircuitProgram (so the host compile to device bytecode is inside the
    # timed region, once), then run_batch over this rank's shots in waves of
    # cfg.wave_shots (each wave: gs_run_counters with host buffers -- the op stream
    # uploaded host->device, counters read back device->host); N > 1:
    # run_batch_distributed (the same per rank + one all-reduce of the
    # counters).  Wall time between barriers, max over ranks.
    from paper_2512_23037_b200 import SamplerConfig, parse_circuit, run_batch
    from paper_2512_23037_b200.distributed import run_batch_distributed
    noisy_text = prog.serialize()
    h2d = int(dp.ops.nbytes + dp.tables.nbytes + dp.locs.nbytes)
    d2h = nc * 8
    e2e_shots = S * max(1, args.e2e_waves)
    cfg_e = SamplerConfig(shots=e2e_shots * world, master_seed=777, postselect=True,
                          rng=args.rng, entry_capacity=4096)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    user_prog = parse_circuit(noisy_text)
    if world > 1:
        st_e = run_batch_distributed(user_prog, cfg_e)
    else:
        st_e = run_batch(user_prog, cfg_e, shot_begin=1 << 40)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    waves = -(-e2e_shots // cfg_e.wave_shots)
    e2e = {"value": st_e.total_shots / e2e_s, "unit": "shots/s",
           "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * waves * world,
           "shots": st_e.total_shots, "wall_s": e2e_s,
           "path": ("parse_circuit + run_batch%s (host compile, op-stream upload, "
                    "%d waves of gs_run_counters with host counter readback)"
                    % ("_distributed" if world > 1 else "", waves))}
    cb = None
    if rank == 0:
        ncu = _ncu_latest(workload, S)
        # per GPU: this rank's section launches, shots and rate
        roofline = _roofline(secs, ncu, S * args.steps, value / world,
                             model_bytes // world, peak, peak_src, ck.get("sm_mhz"))
        if not args.no_cpu_baseline:
            if _have_reference() and not args.ref_port:
                cb = reference_baseline(text, args.p, args.cpu_seconds)
            else:
                cb = cpu_baseline(prog, args.cpu_seconds, args.rng, args.p)
        line = {
            "metric": METRIC, "value": value, "unit": "shots/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded %s noise on the generated MSC proxy)" % args.rng,
            "config": config,
            "discard_rate": int(c[_lib.GS_C_DISCARDED]) / max(total_shots, 1),
            "logical_error_shots": int(c[_lib.GS_C_ERROR_SHOTS]),
            "preserved": int(c[_lib.GS_C_PRESERVED]),
            "roofline": roofline,
            "cpu_baseline": cb, "e2e": e2e, "clocks": ck,
            "gpu_launches": int(launches), "kernel_ms": kernel_ms,
            "wall_s": t_wall,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
