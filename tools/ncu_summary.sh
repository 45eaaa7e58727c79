#!/bin/bash
# Summarise one ncu --set full report: key throughput/occupancy metrics, DRAM bytes, top source lines.
rep=$1
ncu -i "$rep" --page details --csv 2>/dev/null | awk -F'","' '{print $(NF-3)" | "$(NF-2)" | "$(NF-1)" | "$NF}' | \
  grep -E "Duration|Elapsed Cycles|SM Frequency|Compute \(SM\) Throughput|Memory Throughput|DRAM Throughput|Executed Ipc Active|Issue Slots Busy|No Eligible|Active Warps Per Scheduler|Warp Cycles Per Issued|L2 Hit Rate|Registers Per Thread|Dynamic Shared Memory Per Block|Theoretical Occupancy|Achieved Occupancy|Block Limit" | sed 's/"$//'
echo "--- dram bytes (read + write) and FP64 pipe"
ncu -i "$rep" --page raw --csv 2>/dev/null | python3 -c '
import csv, sys
rows = list(csv.reader(sys.stdin))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active", "sm__inst_executed_pipe_fp64",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak", "gpu__time_duration.sum")
sub = ("pipe_tensor_cycles_active", "subpipe_dmma", "lts__t_sectors.sum", "lts__throughput")
for v in vals:
    for i, h in enumerate(hdr):
        if any(h.startswith(w) for w in want) or any(w in h for w in sub):
            print(h, units[i], v[i])
'
echo "--- top source lines (warp stall samples)"
ncu -i "$rep" --page source --csv --print-source=cuda,sass > /tmp/_src.csv 2>/dev/null
python3 "$(dirname "$0")/ncu_lines.py" /tmp/_src.csv 20
