"""Key metrics from an ncu report (raw page) -> stdout / JSON."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_barrier",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append({k: (d.get(k), units[hdr.index(k)] if k in hdr else None) for k in KEYS + ["Kernel Name"]})
    return res


if __name__ == "__main__":
    for d in load(sys.argv[1]):
        print(d["Kernel Name"][0][:90])
        for k in KEYS:
            print(f"  {k:60s} {d[k][0]} {d[k][1] or ''}")
