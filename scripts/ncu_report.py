"""Text summary of one ncu --set full capture of a chunk's section launches
(scripts/gpu_round.sh / gpu_ncu1.sh): per-launch key metrics in launch
order, then source attribution (scripts/ncu_lines.py) of the first
narrow_kernel and the first wide_kernel launch.

    python scripts/ncu_report.py gpurun_out/prof_TAG.ncu-rep "title" > profiles/TAG_ncu_full_sections.txt
"""
import csv
import io
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    "gpu__time_duration.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def ncu(*args):
    return subprocess.run(["ncu", "-i"] + list(args), capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units = rows[0], rows[1]
    print(title)
    for n, r in enumerate(rows[2:]):
        print("--- launch %d: %s" % (n, r[h.index("Kernel Name")].split("(")[0]))
        for m in METRICS:
            if m in h:
                i = h.index(m)
                print("  %-80s %s %s" % (m, r[i], units[i]))
    # source attribution of the longest launch of each kernel
    it = h.index("gpu__time_duration.sum")
    for kern in ("narrow", "wide"):
        mine = [r for r in rows[2:] if r[h.index("Kernel Name")].startswith("void %s_kernel" % kern)]
        if not mine:
            continue
        dur = [float(r[it]) if r[it] not in ("", "-nan", "nan") else 0.0 for r in mine]
        skip = max(range(len(mine)), key=lambda i: dur[i])
        label = "%s_kernel (its longest launch: #%d of %d, %s %s)" % (
            kern, skip, len(mine), mine[skip][it], units[it])
        src = ncu(rep, "--page", "source", "--csv", "--print-source", "sass",
                  "-k", "regex:%s_kernel" % kern, "--launch-skip", str(skip),
                  "--launch-count", "1")
        if not src.strip():
            continue
        with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
            f.write(src)
        print("\n== " + label)
        sys.stdout.flush()
        subprocess.run([sys.executable, os.path.join(HERE, "ncu_lines.py"), f.name] +
                       sys.argv[3:4])
        os.unlink(f.name)


if __name__ == "__main__":
    main()
