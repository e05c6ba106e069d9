"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections, csv, sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def table(path: str, header: str = "") -> str:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg, tot = collections.OrderedDict(), 0.0
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        k = r[ki].split("(")[0][:64]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    out = [header, "#       ms  share launches  kernel"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{t:10.3f} {100 * t / tot:5.1f}% {c:7d}  {k}")
    out.append(f"{tot:10.3f} total ms, {sum(c for c, _ in agg.values())} launches")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print(table(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""), end="")
