#!/usr/bin/env python
"""Summarise an .ncu-rep (raw page) into one line per launch: duration,
DRAM bytes, throughput %, tensor/FMA pipe activity, occupancy, stalls."""
import csv, subprocess, sys

METRICS = [
    ("gpu__time_duration.sum", "us", 1e-3),  # base unit ns -> us
    ("dram__bytes_read.sum", "rd_MB", 1e-6),
    ("dram__bytes_write.sum", "wr_MB", 1e-6),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%", 1),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("lts__t_bytes.sum", "L2_MB", 1e-6),
]

def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    idx = {m: h.index(m) for m, _, _ in METRICS if m in h}
    kn = h.index("Kernel Name")
    units = rows[1]
    for r in rows[2:]:
        name = r[kn].split("(")[0][-40:]
        cells = []
        for m, lab, sc in METRICS:
            if m not in idx:
                continue
            v = r[idx[m]].replace(",", "")
            u = units[idx[m]]
            try:
                x = float(v)
                # normalise to base units before scaling
                mult = {"ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "nsecond": 1, "usecond": 1e3,
                        "msecond": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                        "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
                x = x * mult * sc
                cells.append(f"{lab}={x:.4g}")
            except ValueError:
                cells.append(f"{lab}={v}")
        print(f"{name:40s} " + " ".join(cells))

if __name__ == "__main__":
    main(sys.argv[1])
