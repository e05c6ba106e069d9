"""Top source lines by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
start = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[start]
si = hdr.index("Warp Stall Sampling (All Samples)")
ni = hdr.index("Warp Stall Sampling (Not-issued Samples)")
data, tot = [], 0
for r in rows[start + 1:]:
    if r and r[0] and r[0] != "Line No" and len(r) > si and r[si] not in ("-", ""):
        try:
            s = int(r[si])
        except ValueError:
            continue
        tot += s
        data.append((s, int(r[ni]), r[0], r[1].strip()[:100]))
data.sort(reverse=True)
print("total samples", tot)
for s, ni_, l, src in data[:n]:
    print(f"{s:7d} {100*s/tot:5.1f}% (stall {ni_:6d}) L{l}: {src}")
