"""Print the headline metrics of every kernel in an .ncu-rep (raw page)."""
import csv
import re
import subprocess
import sys

KEYS = [r"^gpu__time_duration.sum$", r"^dram__bytes_read.sum$", r"^dram__bytes_write.sum$",
        r"^lts__t_sector_hit_rate.pct$", r"^l1tex__t_sector_hit_rate.pct$",
        r"^l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed$",
        r"^lts__throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed$",
        r"^sm__warps_active.avg.pct_of_peak_sustained_active$",
        r"^smsp__issue_active.avg.pct_of_peak_sustained_active$",
        r"^launch__registers_per_thread$", r"^launch__grid_size$",
        r"^l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum$",
        r"^lts__t_sectors.sum$",
        r"^smsp__average_warp_latency_issue_stalled_(long_scoreboard|lg_throttle|barrier|membar|short_scoreboard|wait|mio_throttle|math_pipe_throttle|no_instruction|drain)(_per_warp_active)?.*ratio$",
        ]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d.get("Kernel Name", "?")[:80])
    for k in hdr:
        if any(re.search(p, k) for p in KEYS):
            print(f"   {k:75s} {d[k]:>16s} {units[hdr.index(k)]}")
