#!/usr/bin/env python
"""Summarise gpurun_out/ ncu artefacts into profiles/ (tracked).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/launches_<tag>.md
  python tools/ncu_summary.py full gpurun_out/prof_zgemm.ncu-rep profiles/ncu_<tag>.md [traffic.json]

`launches`: per-kernel share of device time in an `ncu --metrics gpu__time_duration.sum`
launch list (cold-cache, serialised: shares, not absolutes).  `full`: the roofline-relevant
metrics of every captured launch of an `ncu --set full` report; with a 4th argument, also
writes the mean DRAM bytes per launch (bench.py's roofline.traffic).
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_barrier",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]


def launches(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("tcbc::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    out = [f"# ncu launch list summary ({src})", "",
           "gpu__time_duration.sum per launch, --clock-control none; cold-cache and serialised, so compare shares.", "",
           "| share | total ms | launches | kernel |", "|---:|---:|---:|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| {100 * v / tot:.2f}% | {v / 1e6:.3f} | {n} | `{k}` |")
    out.append(f"| 100% | {tot / 1e6:.3f} | {sum(n for n, _ in agg.values())} | all |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(src, dst, traffic=None):
    txt = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = [f"# ncu --set full summary ({src})", ""]
    tb = []
    for r in rows[2:]:
        out.append(f"## {r[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                out.append(f"- {k} = {r[h.index(k)]} {units[h.index(k)]}")
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(r[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
            wr = float(r[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
            tb.append(rd + wr)
        except (ValueError, KeyError):
            pass
        out.append("")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))
    if traffic and tb:
        json.dump({"bytes_per_launch": sum(tb) / len(tb), "launches": len(tb), "source": src}, open(traffic, "w"), indent=1)


def traffic(src, dst_md, dst_json, applies=2):
    """DRAM bytes of every zgemm launch in an ncu --metrics CSV of `applies` bench steps."""
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    idk = h.index("ID")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1}
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        except ValueError:
            continue
        per[r[idk]][r[mi]] = v
        per[r[idk]]["name"] = r[ki].split("(")[0].replace("tcbc::", "").replace("<unnamed>::", "")
    launches = [d for d in per.values() if "dram__bytes_read.sum" in d and "zgemm_grouped" in d["name"]]
    tot_b = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in launches)
    tot_t = sum(d.get("gpu__time_duration.sum", 0.0) for d in launches)
    out = [f"# zgemm DRAM traffic per launch ({src}, {applies} bench steps)", "",
           f"launches: {len(launches)}; mean DRAM bytes per launch: {tot_b / len(launches) / 1e6:.1f} MB; "
           f"mean achieved DRAM bandwidth {tot_b / tot_t / 1e9:.0f} GB/s (cold-cache, serialised replays)", "",
           "| launch | kernel | time us | DRAM read MB | DRAM write MB | DMMA active % |", "|---:|---|---:|---:|---:|---:|"]
    for i, d in enumerate(launches):
        out.append(f"| {i} | `{d['name'].replace('void ', '')}` | {d.get('gpu__time_duration.sum', 0) * 1e6:.1f} | "
                   f"{d['dram__bytes_read.sum'] / 1e6:.1f} | {d['dram__bytes_write.sum'] / 1e6:.1f} | "
                   f"{d.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} |")
    open(dst_md, "w").write("\n".join(out) + "\n")
    json.dump({"bytes_per_step": tot_b / applies, "kernel_launches_per_step": len(launches) / applies,
               "bytes_per_kernel_launch": tot_b / len(launches), "source": src,
               "note": "DRAM read+write of every zgemm_grouped launch of one bench step (ncu --metrics "
                       "dram__bytes_read/write.sum, cold-cache serialised replays)"},
              open(dst_json, "w"), indent=1)
    print("\n".join(out[:4]))


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]) if len(sys.argv) > 5 else 2)
        sys.exit(0)
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
