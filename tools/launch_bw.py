"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) per kernel and grid: launches, time, share, DRAM GB/s."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, gi, mi, idi = (h.index(c) for c in ("Kernel Name", "Metric Value", "Grid Size", "Metric Name", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        per[r[idi]]["name"] = r[ki].split("(")[0].split("<")[0].replace("void ", "") + " g=" + \
            r[gi].replace(", 1, 1)", ")")
        per[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for d in per.values():
        t = d.get("gpu__time_duration.sum", 0.0)
        b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a = agg[d["name"]]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{n[:40]:40s} {c:4d} {t / 1e6:8.2f} ms {t / c / 1e3:8.1f} us/l {t / tot * 100:5.1f}%  {b / max(t, 1):7.0f} GB/s")
    print(f"total {tot / 1e6:.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
