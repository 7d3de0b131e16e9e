"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys


def hot(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[si]) if r[si].isdigit() else 0, k, r) for k, r in enumerate(rows[2:])]
    tot = sum(d[0] for d in data) or 1
    stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
    res = []
    for s, k, r in sorted(data, key=lambda x: -x[0])[:top]:
        why = sorted(((int(r[hdr.index(c)]) if r[hdr.index(c)].isdigit() else 0, c) for c in stall_cols),
                     reverse=True)[:2]
        res.append(f"{s / tot:6.1%} #{k:5d} {r[1].strip()[:60]:60s} {why}")
    return "\n".join(res)


if __name__ == "__main__":
    print(hot(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25))
