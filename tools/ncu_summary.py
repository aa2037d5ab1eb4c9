#!/usr/bin/env python
"""Summarise ncu captures into committed text under profiles/.

  python tools/ncu_summary.py full  <report.ncu-rep> <out.txt>
  python tools/ncu_summary.py launches <launch_list.csv> <out.txt>
"""
import csv
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {rep.split('/')[-1]}"]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"\n## {d.get('Kernel Name', '?')}  (launch id {d.get('ID', '?')})")
        for key, label in METRICS:
            if key in d:
                lines.append(f"  {label:32s} {d[key]:>18s} {u.get(key, '')}")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", ""))
            wr = float(d["dram__bytes_write.sum"].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = rd * scale.get(u["dram__bytes_read.sum"], 1) + wr * scale.get(u["dram__bytes_write.sum"], 1)
            t = float(d["gpu__time_duration.sum"].replace(",", ""))
            tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
            ts = t * tscale.get(u["gpu__time_duration.sum"], 1e-9)
            lines.append(f"  {'DRAM traffic (read+write)':32s} {tot / 1e9:18.4f} GB   -> {tot / ts / 1e9:.1f} GB/s")
        except Exception:
            pass
        # stall reasons (top 6)
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warp_latency_issue_stalled_"):-6]))
                except ValueError:
                    pass
        if stalls:
            stalls.sort(reverse=True)
            lines.append("  top stall reasons (cycles/instruction): " +
                         ", ".join(f"{n} {v:.1f}" for v, n in stalls[:6]))
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
        agg[d["Kernel Name"]][0] += 1
        agg[d["Kernel Name"]][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list ({path.split('/')[-1]}): {len(data)} launches, {tot:.3f} ms "
             "(cold-cache, serialised: compare shares)", "launches  total_ms  ms/launch  share  kernel"]
    for k, (cnt, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{cnt:8d} {ms:9.3f} {ms / cnt:10.4f} {100 * ms / tot:5.1f}%  {k}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
