"""Key metrics of an `ncu --set full` report as JSON: python tools/ncu_summary.py rep.ncu-rep [kernel-regex]"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "smsp__average_warp_latency_per_inst_issued.ratio",
        "sm__cycles_elapsed.avg.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[head.index("Kernel Name")]
        if pat and not pat.search(name):
            continue
        m = {"kernel": name[:120]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                m[k] = f"{vals[i]} {units[i]}".strip()
        try:
            rd = float(vals[head.index("dram__bytes_read.sum")])
            wr = float(vals[head.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            m["dram_bytes_per_launch"] = rd * scale[units[head.index("dram__bytes_read.sum")]] + \
                wr * scale[units[head.index("dram__bytes_write.sum")]]
        except (ValueError, KeyError):
            pass
        out.append(m)
    print(json.dumps(out if len(out) != 1 else out[0], indent=1))


if __name__ == "__main__":
    main()
