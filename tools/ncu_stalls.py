#!/usr/bin/env python
"""Per-kernel top stall reasons, IPC, instruction count and smem bank
conflicts from an .ncu-rep (raw page)."""
import csv
import subprocess
import sys


def main(path, top=7):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    pre = "smsp__pcsamp_warps_issue_stalled_"
    for r in rows[2:]:
        d = dict(zip(h, r))
        st = []
        for k, v in d.items():
            if k.startswith(pre) and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k[len(pre):]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print(d["Kernel Name"][:40], [(k, int(v)) for v, k in st[:top]])
        print("   ipc", d.get("sm__inst_executed.avg.per_cycle_active"), "inst",
              d.get("smsp__inst_executed.sum"), "smem conflicts ld/st",
              d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
              d.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum"), "occ%",
              d.get("sm__warps_active.avg.pct_of_peak_sustained_active"))


if __name__ == "__main__":
    main(sys.argv[1])
