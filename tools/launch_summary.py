"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections
import csv
import sys


def summarise(path, top=30):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'us/launch':>10s} {'share':>6s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k:48s} {c:8d} {t:12.1f} {t / c:10.2f} {100 * t / tot:5.1f}%")
    out.append(f"{'TOTAL':48s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
