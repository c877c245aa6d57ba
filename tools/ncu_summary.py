"""Summarise one kernel of an ncu report for profiles/: the details page
(section / metric / unit / value) plus selected raw counters.

    python tools/ncu_summary.py report.ncu-rep "title line" "command line" > out.txt
"""
import csv
import io
import subprocess
import sys

RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
       "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
       "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")


def ncu(path, page):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path, title, cmd):
    print(f"# {title}")
    print(f"# command: {cmd}")
    rows = ncu(path, "details")
    h = rows[0]
    si, mi, ui, vi = (h.index(x) for x in ("Section Name", "Metric Name", "Metric Unit",
                                             "Metric Value"))
    for r in rows[1:]:
        print(f"{r[si][:34]:34s} {r[mi][:52]:52s} {r[ui]:16s} {r[vi]}")
    raw = ncu(path, "raw")
    h, u, v = raw[0], raw[1], raw[2]
    print("# selected raw counters")
    for name in RAW:
        if name in h:
            i = h.index(name)
            print(name, u[i], v[i])
    st = [(h[i], v[i]) for i in range(len(h))
          if h[i].startswith("smsp__average_warps_issue_stalled")
          and h[i].endswith("per_issue_active.ratio")]
    st.sort(key=lambda x: -float(x[1].replace(",", "") or 0))
    print("# top stall reasons (warps per issue)")
    for a, b in st[:6]:
        print(a, b)


if __name__ == "__main__":
    main(*sys.argv[1:4])
