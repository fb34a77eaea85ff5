"""Key metrics of every launch in an .ncu-rep (details page), one block per
launch.  python tools/ncu_details.py REP [metric-substring ...]"""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Achieved Occupancy", "Registers Per Thread", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Issue Slots Busy", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Memory Throughput", "Mem Busy", "Max Bandwidth"]


def main():
    rep = sys.argv[1]
    extra = sys.argv[2:]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    cur = None
    for r in rows[1:]:
        name = r[ix["Metric Name"]]
        if name in WANT or any(e in name for e in extra):
            key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0])
            if key != cur:
                print(f"== launch {key[0]} {key[1]}")
                cur = key
            print(f"   {name:40s} {r[ix['Metric Value']]:>14s} {r[ix['Metric Unit']]}")


if __name__ == "__main__":
    main()
