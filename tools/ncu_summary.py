"""Summarise ncu outputs from gpurun_out/ into profiles/ (text, committed).
    python tools/ncu_summary.py <tag> <launches.csv> [<report.ncu-rep> ...]"""
import csv, collections, os, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "smsp__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    with open(out + "_launches.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "grid", "block", "duration_ns"])
        for d in data:
            w.writerow([d["ID"], d["Kernel Name"].split("(")[0][:80], d["Grid Size"], d["Block Size"],
                        d["Metric Value"]])
    agg = collections.OrderedDict()
    tot = 0.0
    for d in data:
        k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("dl::<unnamed>::", "")[:60]
        t = float(d["Metric Value"]) / 1e3
        agg.setdefault(k, [0, 0.0])
        agg[k][0] += 1
        agg[k][1] += t
        tot += t
    lines = [f"launches: {len(data)}, total {tot:.1f} us (ncu: serialized, cold caches -> compare shares)",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    return "\n".join(lines)


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        return f"(no data in {path})"
    hdr, units = rows[0], rows[1]
    out = [f"### {os.path.basename(path)}"]
    for d in rows[2:]:
        name = d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"* `{name[:90]}`")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  * {k} = {d[i]} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    tag = sys.argv[1]
    out = os.path.join("profiles", tag)
    text = [f"# ncu summary {tag}", "", launches(sys.argv[2], out), ""]
    for rep in sys.argv[3:]:
        text.append(report(rep))
        text.append("")
    with open(out + "_ncu.md", "w") as f:
        f.write("\n".join(text))
    print(out + "_ncu.md")
