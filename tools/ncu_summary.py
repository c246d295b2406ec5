"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv> [--last N]
        per-kernel totals of the last N launches (default: all) -> share of device time
    python tools/ncu_summary.py full <report.ncu-rep>
        key counters of each profiled launch (time, DRAM bytes, L2 hit rate, occupancy ...)
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, last=None):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    rows = [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    if last:
        rows = rows[-last:]
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        tot[name] = tot.get(name, 0.0) + float(r["Metric Value"]) / 1e3
        cnt[name] += 1
    allt = sum(tot.values())
    out = [f"launches: {len(rows)}, device time {allt / 1e3:.3f} ms (ncu, serialised, cold cache)", "",
           "| kernel | launches | total us | avg us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / cnt[k]:.2f} | {100 * v / allt:.1f}% |")
    return "\n".join(out)


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read by SMs"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "stall long scoreboard"),
    ("smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "stall lg throttle"),
    ("smsp__warp_issue_stalled_barrier_per_warp_active.pct", "stall barrier"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"### `{d.get('Kernel Name', '?')[:140]}`")
        out.append("")
        out.append("| counter | value |")
        out.append("|---|---:|")
        for k, label in KEYS:
            if k in hdr:
                out.append(f"| {label} (`{k}`) | {d[k]} {units[hdr.index(k)]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
        print(launches(sys.argv[2], last))
    else:
        print(full(sys.argv[2]))
