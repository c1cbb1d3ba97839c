"""Summarise an ncu launch list (CSV) and one `--set full` capture into a
markdown file under profiles/.

    python tools/ncu_summary.py gpurun_out/launches_X.csv gpurun_out/prof_X.ncu-rep \
        profiles/<round>_<cfg>_<kernel>.md "<title>"
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            d.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")))
    return d


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2]


def main():
    lcsv, rep, dst, title = sys.argv[1:5]
    lines = [f"# {title}", "", "## Launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
             "| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
    d = launches(lcsv)
    tot = sum(sum(v) for v in d.values())
    for k, v in d.items():
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.1%} |")
    h, u, v = raw(rep)
    lines += ["", "## `--set full` capture of the top kernel (one launch)", "",
              "| metric | unit | value |", "|---|---|---|"]
    for i, x in enumerate(h):
        if x in METRICS:
            lines.append(f"| {x} | {u[i]} | {v[i]} |")
    st = [(float(v[i]), x) for i, x in enumerate(h)
          if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued")
          and v[i] not in ("", "0")]
    tot_s = sum(s for s, _ in st) or 1.0
    lines += ["", "## Warp stall sampling (share of samples)", "", "| reason | share |", "|---|---|"]
    for s, x in sorted(st, reverse=True)[:10]:
        lines.append(f"| {x.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {s / tot_s:.1%} |")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
