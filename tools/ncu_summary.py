"""Summarise an ncu report: key throughput metrics, stall reasons, instruction mix."""
import csv
import re
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return res


KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_eligible.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(rep):
    for d in raw(rep):
        print("kernel:", d.get("Kernel Name", ("?",))[0][:100])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k][1]:>10s} {d[k][0]}")
        st = []
        for k, (v, u) in d.items():
            m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio", k)
            if m:
                try:
                    st.append((float(v), m.group(1)))
                except ValueError:
                    pass
        print("  stalls (cycles per issued instruction):", ", ".join(f"{n}={v:.2f}" for v, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
