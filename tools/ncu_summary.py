"""Summarise an .ncu-rep (one block per profiled kernel) from the raw page:
duration, issue/pipe utilisation, DRAM traffic, occupancy, top stall reasons."""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "XU (SFU) pipe %"),
    ("sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__pipe_fp64_cycles_active.sum.pct_of_peak_sustained_active", "FP64 cycles active %"),
    ("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", "ALU pipe %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader([l for l in raw if l.startswith('"')]))
    head, units, data = rows[0], rows[1], rows[2:]
    for row in data:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        print(f"## {d.get('Kernel Name', '?')[:110]}")
        for k, label in KEYS:
            if k in d:
                print(f"  {label:24s} {d[k]} {u.get(k, '')}")
        stalls = [(k.split("smsp__pcsamp_warps_issue_stalled_")[1], float(d[k] or 0)) for k in d
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1
        top = sorted(stalls, key=lambda x: -x[1])[:6]
        print("  stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
