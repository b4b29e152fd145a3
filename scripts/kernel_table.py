"""Per-kernel table of one whole layer (every launch) against MEASURED_PEAKS.json, from an ncu CSV
with the metrics below (`--page raw --csv` of a report, or `--csv` console output):

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
        sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,\\
        sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_ \\
        --launch-skip 240 --launch-count 40 --csv --log-file out.csv python scripts/few_heads.py --P 1 --no-graph --steps 1
    python scripts/kernel_table.py out.csv [title] > profiles/r02_kernel_table.md

Per kernel (summed over its launches in the layer): time, share, DRAM bytes and achieved GB/s
against the measured HBM copy bandwidth, and tensor-pipe activity (issued tensor work, ~ fraction
of the bf16 peak).  ncu serialises launches and runs them cold-cache: shares and bytes are what
compare with the live bench, not absolute times.
"""
import csv
import io
import json
import os
import re
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else ""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    idi = hdr.index("ID")
    per_launch = OrderedDict()
    for r in rows[1:]:
        key = (r[idi], r[ki])
        d = per_launch.setdefault(key, {})
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:  # "n/a" (metric not collected for this launch)
            continue
        unit = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                  "second": 1e6, "s": 1e6}.get(unit, 1.0)   # -> us
        if r[mi].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1.0)
        d[r[mi]] = v
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6538.3)
    agg = OrderedDict()
    for (_, name), d in per_launch.items():
        short = re.sub(r"\(.*", "", name).replace("void ", "")
        a = agg.setdefault(short, dict(n=0, us=0.0, rd=0.0, wr=0.0, tens=0.0, sm=0.0))
        a["n"] += 1
        t = d.get("gpu__time_duration.sum", 0.0)
        a["us"] += t
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
        a["tens"] += t * d.get("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 0.0)
        a["sm"] += t * d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0.0)
    total = sum(a["us"] for a in agg.values())
    print(f"# Per-kernel table of one layer{(' — ' + title) if title else ''}\n")
    print(f"ncu `--clock-control none`, launches serialised and cold-cache; {sum(a['n'] for a in agg.values())} "
          f"launches, {total:.1f} us.  HBM peak = MEASURED_PEAKS.json hbm_gbs = {hbm:.0f} GB/s; tensor % = "
          f"bf16 tcgen05 ops as % of the tensor peak (`sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off`, time-weighted over the kernel's launches).\n")
    print("| kernel | launches | us | share | DRAM read MB | DRAM write MB | GB/s | % of HBM peak | tensor pipe % | SM throughput % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for k, a in agg.items():
        gbs = (a["rd"] + a["wr"]) / (a["us"] * 1e-6) / 1e9 if a["us"] else 0.0
        print(f"| `{k}` | {a['n']} | {a['us']:.1f} | {100 * a['us'] / total:.1f}% | {a['rd'] / 1e6:.0f} | "
              f"{a['wr'] / 1e6:.0f} | {gbs:.0f} | {100 * gbs / hbm:.0f}% | {a['tens'] / a['us'] if a['us'] else 0:.1f} | "
              f"{a['sm'] / a['us'] if a['us'] else 0:.1f} |")


if __name__ == "__main__":
    main()
