"""Summarise ncu reports into profiles/: key SOL metrics per kernel + per-launch DRAM traffic.

    python scripts/ncu_summary.py <report.ncu-rep> <out_prefix> [--traffic-json cfg budget]
"""
import csv, io, json, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, name in enumerate(hdr):
            if name in KEYS or name in ("Kernel Name", "ID"):
                d[name] = (r[i], units[i])
        res.append(d)
    return res


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    res = raw(rep)
    lines = []
    for d in res:
        lines.append("kernel: " + d.get("Kernel Name", ("?", ""))[0][:120])
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:90s} {d[k][0]} {d[k][1]}")
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if "--traffic-json" in sys.argv:
        i = sys.argv.index("--traffic-json")
        cfg, budget = sys.argv[i + 1], float(sys.argv[i + 2])
        d = res[0]
        def val(k):
            v, u = d[k]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        t = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        json.dump({"config": cfg, "budget": budget, "dram_bytes_per_launch": t,
                   "source": rep.split("/")[-1]}, open("profiles/attn_traffic.json", "w"), indent=1)


if __name__ == "__main__":
    main()
