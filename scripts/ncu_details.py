"""Print the key `ncu --set full` metrics of every kernel in a report (ncu -i ... --page details --csv).

python scripts/ncu_details.py <report.ncu-rep> [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Eligible Warps Per Scheduler", "Issued Warp Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Waves Per SM", "Block Limit Registers", "Block Limit Shared Mem")


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if not rows:
            continue
        h = rows[0]
        print(f"## {rep}")
        last = None
        for r in rows[1:]:
            d = dict(zip(h, r))
            kid = (d.get("ID"), d.get("Kernel Name", "")[:60])
            if kid != last:
                print(f"\n### launch {kid[0]}: {kid[1]}  grid {d.get('Grid Size', '')}")
                last = kid
            if d.get("Metric Name") in KEYS:
                print(f"  {d['Metric Name']}: {d['Metric Value']} {d.get('Metric Unit', '')}")


if __name__ == "__main__":
    main()
