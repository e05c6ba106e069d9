"""Top SASS instructions by warp-stall samples from an .ncu-rep (run here, no GPU)."""
import csv, io, subprocess, sys
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)"); src = h.index("Source"); ex = h.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in body)
print(f"total samples {tot}, instructions {len(body)}")
for idx, r in sorted(enumerate(body), key=lambda x: -int(x[1][si] or 0))[:top]:
    print(f"{idx:5d} {int(r[si] or 0):6d} {100*int(r[si] or 0)/tot:5.1f}%  ex={r[ex]:>8s}  {r[src].strip()[:90]}")
