"""profiles/traffic.json from an ncu_traffic.sh capture: the mean DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per launch of the tensor-core
conv kernel of the FP32 tier, keyed by the bench's kernel-family names
(fprop and dgrad launch the same k_conv_tc instantiations, so both families
get the mean over all of them).  Usage: traffic_json.py traffic.csv split"""
import collections, csv, io, json, sys

path, split = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "3xf16"
h16 = {"3xf16": "2", "3xbf16": "1", "3xtf32": None}[split]
rows = list(csv.DictReader(io.StringIO("".join(l for l in open(path) if l.startswith('"')))))
per = collections.defaultdict(dict)
for r in rows:
    per[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot, n = 0.0, 0
for (i, name), m in per.items():
    if "k_conv_tc" not in name:
        continue
    tmpl = name.split("k_conv_tc<")[1].split(">")[0].replace(" ", "").split(",")
    if (h16 and (len(tmpl) < 5 or tmpl[4] != h16)) or (not h16 and len(tmpl) > 4 and tmpl[4] != "0"):
        continue
    tot += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    n += 1
mean = tot / max(n, 1)
note = (f"mean dram__bytes_read.sum + dram__bytes_write.sum over the {n} k_conv_tc launches of "
        f"the {split} tier (fprop and dgrad share the kernel) in a 12-candidate single-stream "
        "bench under ncu (scripts/ncu_traffic.sh, profiles/r02_profile.md); below the algorithmic "
        "bytes of a layer (a 128@16x16 N=128 layer reads 16.8 MB of activations and writes "
        "16.8 MB): the previous layer's output is served from L2")
out = {f"conv_dgrad_tc_{split}_fisher": {"dram_bytes_per_launch": int(mean), "note": note},
       f"conv_fprop_tc_{split}": {"dram_bytes_per_launch": int(mean),
                                  "note": f"see conv_dgrad_tc_{split}_fisher (same kernel)"}}
json.dump(out, sys.stdout, indent=2)
print()
