"""Summarise an ncu per-kernel launch list (gpu__time_duration, dram bytes) of
scripts/prof_kernels.py L 1 precond into the DRAM traffic of ONE preconditioner
apply (the launches after the dense coarse inverse; prof_kernels runs the apply
twice, warm-up + 1 timed).  Writes profiles/round1_apply_traffic.json used by
bench.py's roofline "traffic" field.

python scripts/apply_traffic.py gpurun_out/traffic50.csv:50:1 gpurun_out/traffic150.csv:150:4
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", ""))
    items = list(d.items())
    gj = [i for i, (k, _) in enumerate(items) if "k_gj" in k[1]]
    ap = items[gj[-1] + 1:]
    ap = ap[: len(ap) // 2]  # the first (warm-up) apply
    t = sum(v["gpu__time_duration.sum"] for _, v in ap) * 1e-9
    b = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for _, v in ap)
    return dict(launches=len(ap), dram_bytes=b, serialised_s=t)


def main():
    out = {}
    for arg in sys.argv[1:]:
        path, L, seed = arg.split(":")
        r = one(path)
        r.update(L=int(L), seed=int(seed), W=16.5)
        out[L] = r
        print(L, r)
    out["how"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "--clock-control none -k regex:'k_apply|k_dense_mv|k_gj' python scripts/prof_kernels.py L 1 "
                  "precond seed; launches of one apply (cold-cache, serialised)")
    with open(os.path.join(ROOT, "profiles", "round1_apply_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
