"""Summarise one kernel of an ncu --set full report (raw page) into the profiles/ format."""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def summarise(rep, kernel_regex=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for v in data:
        d = {"Kernel Name": v[hdr.index("Kernel Name")]}
        if kernel_regex and kernel_regex not in d["Kernel Name"]:
            continue
        for n in WANT:
            if n in hdr:
                i = hdr.index(n)
                d[n] = (v[i] + " " + units[i]).strip()
        for n in hdr:
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                val = float(v[hdr.index(n)].replace(",", "") or 0)
                if val >= 0.05:
                    d["stall_" + n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(val, 3)
        res.append(d)
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None), indent=1))
