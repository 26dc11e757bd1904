"""Summarise .ncu-rep captures into profiles/ (markdown): key throughput,
memory, pipe and stall metrics per kernel.  python tools/ncu_summary.py out.md rep1 [rep2 ...]"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % (active)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe % (active)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2 -> L1 bytes"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle / issue"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    dst = sys.argv[1]
    lines = ["# ncu summaries (round 1)", "",
             "Captured with `ncu --set full --clock-control none --import-source on` under gpurun on one B200;",
             "per-launch numbers are replayed/serialised, so compare shares, not absolute step times.", ""]
    for rep in sys.argv[2:]:
        h, u, data = raw(rep)
        for v in data:
            name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            lines += [f"## {rep.split('/')[-1]} — `{name[:110]}`", "", "| metric | value | unit |", "|---|---|---|"]
            for key, label in WANT:
                if key in h:
                    i = h.index(key)
                    lines.append(f"| {label} (`{key}`) | {v[i]} | {u[i]} |")
            lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
