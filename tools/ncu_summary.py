"""Summarise an ncu --set full report (.ncu-rep) per kernel launch: duration,
DRAM traffic, DMMA / FP64 pipe activity, occupancy, top warp stalls."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_pipe_pct_active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct_active"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[col["Kernel Name"]][:90]
        print(f"== {name}")
        for k, label in KEYS:
            if k in col:
                print(f"   {label:24s} {r[col[k]]:>14s} {units[col[k]]}")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i].replace(',', '')), h))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            print("   top stalls (cycles per issued instruction): " +
                  ", ".join(f"{h.split('stalled_')[1].replace('_per_issue_active.ratio', '')} {v:.2f}" for v, h in stalls[:5]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
