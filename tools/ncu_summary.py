"""Summarise an ncu report (development tool): key throughput / stall metrics
per kernel launch, each value with its ncu unit (ncu scales byte counts to
byte / Kbyte / Mbyte per metric).   python tools/ncu_summary.py report.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = (r'^(gpu__time_duration.sum|dram__bytes_read.sum|dram__bytes_write.sum|'
        r'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum|'
        r'smsp__inst_executed.sum|launch__registers_per_thread|launch__grid_size|'
        r'sm__warps_active.avg.pct_of_peak_sustained_active|smsp__issue_active.avg.pct_of_peak_sustained_active|'
        r'dram__throughput.avg.pct_of_peak_sustained_elapsed|l1tex__throughput.avg.pct_of_peak_sustained_active|'
        r'lts__t_sectors_srcunit_tex_op_write.sum|lts__t_sectors_srcunit_tex_op_read.sum|'
        r'smsp__pcsamp_warps_issue_stalled_(long_scoreboard|wait|short_scoreboard|selected|not_selected|'
        r'math_pipe_throttle|branch_resolving|mio_throttle|lg_throttle|drain|barrier|no_instruction))$')


def main():
    rep = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else "."
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    idx = [i for i, k in enumerate(h) if re.search(KEYS, k)]
    for r in rows[2:]:
        if not re.search(pat, r[ki]):
            continue
        print(r[ki][:70])
        for i in idx:
            print("    %-62s %s %s" % (h[i], r[i], units[i]))


if __name__ == "__main__":
    main()
