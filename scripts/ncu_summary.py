"""Summarise an ncu --set full report (one kernel) into the metrics DESIGN.md cites.

    python scripts/ncu_summary.py gpurun_out/k2_c4_v3.ncu-rep > profiles/r01/k2_c4_v3_ncu.txt
"""
import csv
import io
import subprocess
import sys

WANT = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("---")
        for i, h in enumerate(hdr):
            if h in WANT or (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
                v = r[i]
                if h.startswith("smsp__pcsamp") and v in ("0", ""):
                    continue
                print(f"{h:75s} {v} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
