"""Top stalled CUDA source lines of an ncu report (SourceCounters section,
--print-source cuda,sass) within a line range: python stall_lines.py rep lo hi"""
import csv, subprocess, sys
rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[2]
cols = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
def iv(x):
    try:
        return int(x)
    except ValueError:
        return 0
agg = []
for r in rows[3:]:
    if r and r[0] == "File Path":
        break
    if len(r) > 5 and r[0]:
        agg.append((int(r[0]), iv(r[4]), {h[6:]: iv(r[j]) for j, h in cols if iv(r[j])}, r[1].strip()[:80], iv(r[7])))
tot = sum(a[1] for a in agg)
sel = [a for a in agg if lo <= a[0] <= hi]
print("total samples", tot, "in range", sum(a[1] for a in sel))
st = {}
for a in sel:
    for k, v in a[2].items():
        st[k] = st.get(k, 0) + v
print(sorted(st.items(), key=lambda x: -x[1])[:10])
for a in sorted(sel, key=lambda a: -a[1])[:25]:
    print(a[0], a[1], a[4], sorted(a[2].items(), key=lambda x: -x[1])[:3], a[3])
