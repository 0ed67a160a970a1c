"""Summarise ncu output into profiles/: per-kernel share of a launch list
(gpu__time_duration.sum, cold-cache serialised) and the key metrics of a
--set full capture.  Usage: ncu_summary.py launches.csv [prof.ncu-rep]"""
import collections, csv, io, subprocess, sys


def launches(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("unnamed>::", "")
        if "k_conv_tc" in r["Kernel Name"]:
            name = r["Kernel Name"].split("(")[0].replace("void unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r["Metric Value"]) / 1e3  # ns -> us
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {len(rows)}, summed device time {tot:.1f} us", "",
           "| kernel | launches | us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {w: hdr.index(w) for w in WANT if w in hdr}
    kn = hdr.index("Kernel Name")
    out = ["| kernel | " + " | ".join(f"{w} [{units[i]}]" for w, i in idx.items()) + " |",
           "|---" * (len(idx) + 1) + "|"]
    for r in rows[2:]:
        out.append(f"| `{r[kn].split('(')[0].replace('void unnamed>::', '')}` | " +
                   " | ".join(r[i] for i in idx.values()) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print("## Launch list (ncu gpu__time_duration.sum, --clock-control none)\n")
    print(launches(sys.argv[1]))
    if len(sys.argv) > 2:
        print("\n## Full capture (ncu --set full)\n")
        print(full(sys.argv[2]))
