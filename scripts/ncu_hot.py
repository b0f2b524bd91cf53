"""Hottest SASS lines (warp-stall samples) of each kernel in an ncu report, with the
CUDA source line they map to (compile with -lineinfo).

python scripts/ncu_hot.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')
    for b in blocks[1:]:
        rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
        name = rows[0][1][:90]
        h = rows[1]
        data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
        key = "Warp Stall Sampling (All Samples)"
        tot = sum(float(d.get(key, 0) or 0) for d in data)
        print(f"## {name}  (samples {tot:.0f})")
        for d in sorted(data, key=lambda d: -float(d.get(key, 0) or 0))[:top]:
            print(f"  {float(d[key]) / max(tot, 1) * 100:5.1f}%  {d.get('Source', '')[:70]:70s} {d.get('Address', '')[-6:]}")


if __name__ == "__main__":
    main()
