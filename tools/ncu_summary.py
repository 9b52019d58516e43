"""Summarise an ncu --set full report: key metrics and the top stall sites.

    python tools/ncu_summary.py report.ncu-rep "title" > profiles/xxx.txt
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__cluster_dim_x",
        "launch__block_size", "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active"]


def main():
    rep, title = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    print(f"# {title}")
    print(f"# kernel: {v[h.index('Kernel Name')]}")
    print("## key metrics")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"{k:80s} {v[i]} {u[i]}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) > 2 and "Warp Stall Sampling (All Samples)" in rows[1]:
        hh = rows[1]
        si = hh.index("Warp Stall Sampling (All Samples)")
        ok = [x for x in rows[2:] if len(x) > si and x[si].isdigit()]
        sc = [i for i, x in enumerate(hh) if x.startswith("stall_") and "Not Issued" not in x]
        print("## top stall sites (SASS, samples)")
        for x in sorted(ok, key=lambda x: -int(x[si]))[:10]:
            st = sorted([(int(x[i]), hh[i]) for i in sc if x[i].isdigit() and int(x[i]) > 0], reverse=True)[:1]
            print(f"{int(x[si]):5d}  {x[1].strip()[:70]:72s} {st[0][1] if st else ''}")


if __name__ == "__main__":
    main()
