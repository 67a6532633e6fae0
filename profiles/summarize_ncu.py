"""Summarise an `ncu --set full` report into the committed evidence files:
<name>_details.csv (the details page) and <name>_metrics.json (duration,
DRAM bytes, pipe utilisation, occupancy, top stall reasons).

    python profiles/summarize_ncu.py gpurun_out/x.ncu-rep profiles/r01/x [launch index]

The launch index selects one kernel of a multi-kernel report (default 0).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
]


def main(rep, out, idx=0):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(out + "_details.csv", "w").write(det)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2 + idx]
    m = {"kernel": v[h.index("Kernel Name")]}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            m[k] = [v[i], u[i]]
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    m["top_stalls_per_issue"] = [[n, round(x, 2)] for x, n in sorted(st, reverse=True)[:6]]
    json.dump(m, open(out + "_metrics.json", "w"), indent=1)
    print(json.dumps(m))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
