"""Summarise an ncu report: key raw metrics + top stall instructions (source page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
        "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed"]
for row in r[2:3]:
    for i, x in enumerate(r[0]):
        if any(x == w for w in want):
            print(f"{x:60s} {r[1][i]:>10s} {row[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
i_s = h.index("Warp Stall Sampling (All Samples)")
data = [(int(x[i_s]) if x[i_s].isdigit() else 0, x[0], x[1].strip()) for x in rows[2:] if len(x) > i_s]
tot = sum(d[0] for d in data) or 1
print("total stall samples", tot)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
addr = [d[1] for d in data]
for d in sorted(data, reverse=True)[:top]:
    k = addr.index(d[1])
    prev = data[k - 1][2][:50] if k else ""
    print(f"{d[0]:7d} {100*d[0]/tot:5.1f}%  {d[1][-5:]}  {d[2][:70]:70s} | prev: {prev}")
