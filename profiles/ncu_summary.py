"""Print the headline metrics of an ncu report (run here, no GPU needed):
    python profiles/ncu_summary.py gpurun_out/div.ncu-rep"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__inst_executed.sum", "lts__t_bytes.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for row in r[2:]:
        print("kernel:", row[h.index("Kernel Name")][:90])
        for w in WANT:
            if w in h:
                i = h.index(w)
                print(f"  {w:62s} {row[i]:>16s} {units[i]}")
        stalls = [(float(row[i]), h[i]) for i in range(len(h))
                  if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not
                  h[i].endswith("not_issued") and row[i].replace('.', '', 1).isdigit()]
        for v, n in sorted(stalls, reverse=True)[:8]:
            print(f"  {n:62s} {v:16.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
