"""Per-level time / DRAM bytes of the LAST preconditioner apply in an ncu launch list
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv).

python scripts/apply_levels.py <launches.csv>
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    k = {}
    for r in rows[hdr + 1:]:
        d = k.setdefault(int(r[0]), {"name": r[4].split("(")[0].replace("void ", "").replace("aj::", ""),
                                     "grid": r[8]})
        d[r[12]] = float(r[14].replace(",", ""))
    ks = [k[i] for i in sorted(k)]
    apps, cur, prev = [], [], None
    for x in ks:
        isap = x["name"].startswith("k_apply") or x["name"].startswith("k_dense_mv")
        if not isap:
            prev = None
            continue
        if x["name"].startswith("k_apply_fwd") and (prev is None or not prev.startswith("k_apply_fwd")) and cur:
            apps.append(cur)
            cur = []
        cur.append(x)
        prev = x["name"]
    apps.append(cur)
    a = apps[-1]
    T = lambda x: x.get("gpu__time_duration.sum", 0.0)  # noqa: E731
    B = lambda x: x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)  # noqa: E731
    tot, byt = sum(map(T, a)), sum(map(B, a))
    print(f"{len(apps)} applies; last: {len(a)} launches, {tot / 1e3:.1f} us (serialised, cold), "
          f"{byt / 1e9:.3f} GB DRAM, {byt / tot:.0f} GB/s")
    fw = [x for x in a if "fwd" in x["name"]]
    bw = list(reversed([x for x in a if "bwd" in x["name"]]))
    for label, lst in (("forward", fw), ("backward", bw)):
        print(f"{label}: {len(lst)} levels, {sum(map(T, lst)) / 1e3:.1f} us")
        for lo, hi in ((0, 1), (1, 5), (5, 15), (15, 30), (30, 60), (60, 100), (100, 200), (200, 400)):
            seg = lst[lo:hi]
            if not seg:
                continue
            t, b = sum(map(T, seg)), sum(map(B, seg))
            print(f"  levels {lo:3d}-{min(hi, len(lst)) - 1:3d}: {t / 1e3:8.1f} us ({t / tot * 100:4.1f} %) "
                  f"{b / 1e6:9.1f} MB {b / max(t, 1):7.0f} GB/s  kernels {sorted(set(x['name'] for x in seg))}")


if __name__ == "__main__":
    main()
