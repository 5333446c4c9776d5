"""Summarise an ncu --set full report (one entry per profiled kernel) into
the JSON kept under profiles/: time, DRAM/L2 traffic, issue and pipe
activity, registers, launch shape and stall reasons per issued instruction.

    python tools/ncu_extract.py report.ncu-rep > profiles/ncu_....json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct", "sm__inst_issued.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALL = "smsp__average_warps_issue_stalled_"
SUFFIX = "_per_issue_active.ratio"


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[head.index("Kernel Name")]
        ent = {"kernel": name[:110]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                ent[k] = f"{r[i]} {units[i]}".strip()
        st = {}
        for i, k in enumerate(head):
            if k.startswith(STALL) and k.endswith(SUFFIX):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.01:
                    st[k[len(STALL):-len(SUFFIX)]] = round(v, 3)
        ent["stalls_per_issue"] = st
        key = name.split("(")[0].replace("void ", "")
        res[key] = ent
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
