"""Summarise an ncu report (raw page) per kernel: duration, DRAM bytes,
pipe utilisation, L1/smem wavefronts, bank conflicts, warp-stall mix.
usage: python profiles/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_thru%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe%"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "gld_wavefronts"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_st.sum", "gst_wavefronts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_thru%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_thru%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_thru%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("launch__registers_per_thread", "regs"),
]
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "mio_throttle", "lg_throttle", "math_pipe_throttle",
          "wait", "not_selected", "selected", "dispatch_stall", "no_instruction", "branch_resolving"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0]
        parts = []
        for k, short in KEYS:
            if k in col:
                parts.append(f"{short}={r[col[k]]}{units[col[k]] if units[col[k]] not in ('', '%') else ''}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in col:
                st.append(f"{s}={float(r[col[k]]):.2f}")
        print(name)
        print("   " + "  ".join(parts))
        print("   stalls/issue: " + " ".join(st))


if __name__ == "__main__":
    main(sys.argv[1])
