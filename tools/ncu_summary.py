"""Key metrics from an ncu --set full report (raw page)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
STALLS = "smsp__average_warps_issue_stalled_"


def main(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        print("==", d.get("Kernel Name", "?")[:60])
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]} {units[hdr.index(k)]}")
        st = sorted(((float(d[k]), k) for k in hdr if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio")
                     and d[k] not in ("", "n/a")), reverse=True)
        print("  stalls per issue:", ", ".join(f"{k[len(STALLS):-len('_per_issue_active.ratio')]}={v:.2f}" for v, k in st[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
