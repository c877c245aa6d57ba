"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram/lts bytes]).

    python tools/launch_table.py launches.csv [--skip N]
Prints per-kernel launch count, total/avg device time, share of the total,
and (when captured) DRAM bytes and L2 bytes per launch.
"""
import collections
import csv
import sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "s": 1e6, "second": 1e6}
BYTES = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9,
         "GB": 1e9, "Tbyte": 1e12, "TB": 1e12}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                 "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        per[r[ii]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
        names[r[ii]] = r[ki]
    agg = collections.OrderedDict()
    total = 0.0
    for i, m in per.items():
        t, u = m["gpu__time_duration.sum"]
        t *= TIME[u]
        a = agg.setdefault(names[i][:80], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += t
        for key, slot in (("dram__bytes_read.sum", 2), ("dram__bytes_write.sum", 2),
                          ("lts__t_bytes.sum", 3)):
            if key in m:
                a[slot] += m[key][0] * BYTES[m[key][1]]
        total += t
    print(f"{'launches':>8} {'total_ms':>10} {'avg_ms':>9} {'share':>6} {'dram_GB/l':>10} "
          f"{'l2_GB/l':>9}  kernel")
    for k, (c, t, d, l) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t / 1e3:10.3f} {t / c / 1e3:9.3f} {100 * t / total:5.1f}% "
              f"{d / c / 1e9:10.4f} {l / c / 1e9:9.3f}  {k}")
    print(f"total device time {total / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
