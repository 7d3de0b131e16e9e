"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys


def summary(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':28s} {'launches':>8s} {'total_us':>12s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:28s} {v[0]:8d} {v[1]:12.1f} {v[1] / tot:6.3f}")
    out.append(f"{'TOTAL':28s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
