"""Key numbers of an ncu --set full report: duration, DMMA pipe, DRAM bytes
and throughput, issue activity, occupancy, top warp stalls.
usage: ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))


def main():
    d = raw(sys.argv[1])
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size"]
    for k in keys:
        if k in d:
            print(f"{k}: {d[k][:110]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and v.replace(".", "", 1).isdigit()}
    tot = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
    print("top stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()
