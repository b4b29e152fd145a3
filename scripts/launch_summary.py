"""Summarise an ncu launch list (gpu__time_duration.sum, --clock-control none) of one bench layer.

    python scripts/launch_summary.py gpurun_out/launches.csv <n_launches_per_layer> [title] [k_init_sample occurrence] > profiles/rNN_launches_summary.tsv

Takes the LAST n launches (one whole layer after warm-up) and prints per-kernel totals and shares.
ncu serialises launches and runs them cold-cache, so the shares (not the absolute times) are what
must agree with bench.py's live CUDA-event stage times.
"""
import csv
import io
import re
import sys
from collections import OrderedDict


def main():
    path, n = sys.argv[1], int(sys.argv[2])
    title = sys.argv[3] if len(sys.argv) > 3 else ""
    occ = int(sys.argv[4]) if len(sys.argv) > 4 else None  # start at the occ-th k_init_sample launch
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ki, mi, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    launches = [(r[ki], float(r[vi]), r[gi]) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    if occ is None:
        layer = launches[-n:]
    else:
        starts = [i for i, l in enumerate(launches) if l[0].startswith("k_init_sample")]
        layer = launches[starts[occ]:starts[occ] + n]
    agg = OrderedDict()
    for name, ns, grid in layer:
        short = re.sub(r"\(.*", "", name).strip()
        c = agg.setdefault(short, [0.0, 0])
        c[0] += ns / 1e3
        c[1] += 1
    total = sum(v[0] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised) -- "
          f"one layer = {n} launches")
    if title:
        print(f"# {title}")
    print("us\tlaunches\tshare\tkernel")
    for k, (us, c) in agg.items():
        print(f"{us:.1f}\t{c}\t{100 * us / total:.1f}%\t{k}")
    print(f"{total:.1f}\t{len(layer)}\t100%\ttotal")


if __name__ == "__main__":
    main()
