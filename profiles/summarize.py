"""Summarise ncu captures (gpurun_out/*.ncu-rep) and launch lists into
profiles/ (tracked).  Usage:
  python profiles/summarize.py <tag> <report.ncu-rep>[:<sites>] ... [--launches <csv>]
<sites> = sites the captured launch processed (for bytes/site)."""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sector_hit_rate.pct", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                d[m] = r[hdr.index(m)] + (" " + units[hdr.index(m)] if units[hdr.index(m)] else "")
        res.append(d)
    return res


def to_bytes(s):
    v, u = s.split()[0], (s.split() + [""])[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return float(v.replace(",", "")) * scale


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        args = args[:i] + args[i + 2:]
    summary = {"tag": tag, "captures": []}
    md = [f"# ncu summary — {tag}", ""]
    for a in args:
        rep, _, sites = a.partition(":")
        for k in raw(rep):
            rb, wb = to_bytes(k["dram__bytes_read.sum"]), to_bytes(k["dram__bytes_write.sum"])
            entry = dict(report=rep.split("/")[-1], **k)
            if sites:
                entry["sites"] = int(sites)
                entry["dram_bytes_per_site"] = (rb + wb) / int(sites)
            summary["captures"].append(entry)
            md.append(f"## {entry['report']}: `{k['kernel'][:110]}`")
            for m in METRICS:
                if m in k:
                    md.append(f"- {m}: {k[m]}")
            if sites:
                md.append(f"- DRAM bytes per site (read+write): {entry['dram_bytes_per_site']:.1f} (algorithmic 376)")
            md.append("")
    if launches:
        lines = open(launches).read().splitlines()
        start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
        rows = list(csv.reader(lines[start:]))
        hdr = rows[0]
        kn, val = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[1:]:
            name = r[kn].split("(")[0]
            agg.setdefault(name, []).append(float(r[val].replace(",", "")))
        tot = sum(sum(v) for v in agg.values())
        md.append("## launch list (ncu gpu__time_duration, cold-cache, serialised)")
        md.append("| kernel | launches | total us | share |")
        md.append("|---|---|---|---|")
        for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{name[:80]}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
        summary["launch_shares"] = {n: sum(v) / tot for n, v in agg.items()}
    with open(f"profiles/{tag}.md", "w") as f:
        f.write("\n".join(md) + "\n")
    with open(f"profiles/{tag}.json", "w") as f:
        json.dump(summary, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
