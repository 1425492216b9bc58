"""Summarize ncu artefacts into markdown for profiles/.

  python tools/ncu_summary.py report.ncu-rep            # --set full capture
  python tools/ncu_summary.py --launches launches.csv   # gpu__time_duration launch list
"""

import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__waves_per_multiprocessor",
    "lts__t_sector_hit_rate.pct",
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full: `{path}`", ""]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:90]
        lines += [f"## {name}", "", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {r[i]} {units[i]} |")
        st = [(h[33:], float(r[i].replace(",", ""))) for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued") and r[i]]
        tot = sum(v for _, v in st) or 1.0
        top = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:5])
        lines += [f"| top stall reasons (pc sampling) | {top} |", ""]
    return "\n".join(lines)


def launches(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr, recs, order = None, {}, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["ID"]
            if k not in recs:
                recs[k] = {"name": d["Kernel Name"][:60]}
                order.append(k)
            recs[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    sel = order[-last:] if last else order
    lines = [f"# launch list: `{path}` (cold-cache, serialised; compare shares)", "",
             "| # | kernel | time (us) | DRAM read (MB) | GB/s |", "|---|---|---|---|---|"]
    tot = 0.0
    for i, k in enumerate(sel):
        o = recs[k]
        t = o.get("gpu__time_duration.sum", 0.0)
        b = o.get("dram__bytes_read.sum", 0.0)
        tot += t
        lines.append(f"| {i} | {o['name']} | {t / 1e3:.1f} | {b / 1e6:.1f} | {b / max(t, 1):.0f} |")
    lines.append(f"| | total | {tot / 1e3:.1f} | | |")
    return "\n".join(lines)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else None))
    else:
        print(full(sys.argv[1]))
