"""Summarise an ncu full capture of the sampling kernel (read here, no GPU):
key metrics + instruction histogram by SASS block."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_misc_per_issue_active.ratio"]


def ncu(*args):
    return subprocess.run(["ncu", "-i"] + list(args), capture_output=True,
                          text=True).stdout


def main(rep, shots=None, top=15):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    out = {}
    for w in WANT:
        if w in h:
            i = h.index(w)
            out[w] = (v[i], u[i])
            print("%-80s %s %s" % (w, v[i], u[i]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    hh, body = src[1], src[2:]
    ia = hh.index("Instructions Executed")
    iss = hh.index("Warp Stall Sampling (All Samples)")
    iad = hh.index("Address")
    base = int(body[0][iad], 16)
    blocks, cur = [], None
    for x in body:
        a = int(x[iad], 16) - base
        e = int(x[ia] or 0)
        s = int(x[iss] or 0)
        if cur and cur["e"] == e:
            cur["n"] += 1
            cur["s"] += s
            cur["end"] = a
        else:
            cur = {"start": a, "end": a, "e": e, "n": 1, "s": s}
            blocks.append(cur)
    tot = sum(b["e"] * b["n"] for b in blocks)
    st = sum(b["s"] for b in blocks) or 1
    print("total warp instructions %d%s" % (tot, "" if not shots else
                                             " (%.0f per shot)" % (tot / shots)))
    for b in sorted(blocks, key=lambda b: -b["e"] * b["n"])[:top]:
        print("  %6x-%6x n=%4d exec=%10d inst%%=%5.1f stall%%=%5.1f"
              % (b["start"], b["end"], b["n"], b["e"], 100 * b["e"] * b["n"] / tot,
                 100 * b["s"] / st))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
