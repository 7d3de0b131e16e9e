"""DRAM traffic of the captured Schur launches vs their algorithmic bytes.

    python tools/ncu_traffic.py <report.ncu-rep> <schurlog.txt> <skip> [out.json]

The report comes from `ncu --set full -k regex:schur_oz -s <skip> -c N <cmd>` and the log from
the same command run with H2L_SCHURLOG=1 (one line per Schur launch, in launch order, with the
launch's algorithmic bytes: targets read + written once, X and Bg read once).  Launch
`skip + q` of the log is capture q of the report."""
import csv
import json
import re
import subprocess
import sys


def main():
    rep, log, skip = sys.argv[1], sys.argv[2], int(sys.argv[3])
    out = sys.argv[4] if len(sys.argv) > 4 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]

    def col(r, k):
        i = hdr.index(k)
        v, u = float(r[i].replace(",", "")), units[i]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "us": 1e-6,
                    "s": 1.0, "ns": 1e-9}.get(u, 1.0)

    lines = [ln for ln in open(log) if ln.startswith("schurlog")]
    caps = []
    for q, r in enumerate(rows[2:]):
        m = re.search(r"tiles=(\d+) shifts=(\d+) ms=([\d.]+) tflops=([\d.]+) alg_bytes=(\d+)",
                      lines[skip + q])
        rd, wr = col(r, "dram__bytes_read.sum"), col(r, "dram__bytes_write.sum")
        caps.append({"launch": skip + q, "tiles": int(m.group(1)), "shifts": int(m.group(2)),
                     "plain_run_ms": float(m.group(3)), "plain_run_tflops_fp64_equivalent": float(m.group(4)),
                     "algorithmic_bytes": float(m.group(5)), "dram_bytes_read": rd, "dram_bytes_write": wr,
                     "dram_over_algorithmic": (rd + wr) / float(m.group(5)),
                     "ncu_duration_ms": 1e3 * col(r, "gpu__time_duration.sum"),
                     "tensor_pipe_active_pct": col(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                     "l2_throughput_pct": col(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                     "dram_throughput_pct": col(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")})
    n = max(1, len(caps))
    res = {"kernel": "schur_oz_kernel", "captures": caps,
           "dram_bytes_per_launch_mean": sum(c["dram_bytes_read"] + c["dram_bytes_write"] for c in caps) / n,
           "algorithmic_bytes_per_launch_mean": sum(c["algorithmic_bytes"] for c in caps) / n}
    text = json.dumps(res, indent=1)
    print(text)
    if out:
        open(out, "w").write(text)


if __name__ == "__main__":
    main()
