"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py launches <launches.csv> [--last-eval]   # per-kernel share table
    python tools/summarize_ncu.py report <file.ncu-rep>                   # key metrics of a full capture
"""
import csv
import subprocess
import sys

KEY_METRICS = [
    "gpu__time_duration.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]


def launches(path, last_eval):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    k, v = h.index("Kernel Name"), h.index("Metric Value")
    seq = [(r[k], float(r[v].replace(",", ""))) for r in rows[hi + 1:] if len(r) > v]
    if last_eval:
        # the last evaluate starts at the last keys_kernel launch (tree build)
        starts = [i for i, (n, _) in enumerate(seq) if "keys_kernel" in n]
        if len(starts) >= 2:
            seq = seq[starts[-2]:]
    agg = {}
    for n, t in seq:
        short = n.split("(")[0].replace("pkgpu::<unnamed>::", "").replace("void ", "")[:70]
        a = agg.setdefault(short, [0.0, 0])
        a[0] += t
        a[1] += 1
    tot = sum(t for _, t in seq)
    print(f"| kernel | launches | device time (ms) | share |\n|---|---|---|---|")
    for n, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        if t / tot < 0.0005:
            continue
        print(f"| `{n}` | {c} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    print(f"| **total** | {len(seq)} | {tot / 1e6:.3f} | 100% |")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel: {name[:120]}")
        for m in KEY_METRICS:
            if m in h:
                i = h.index(m)
                print(f"  {m} = {r[i]} {units[i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], "--last-eval" in sys.argv)
    else:
        report(sys.argv[2])
