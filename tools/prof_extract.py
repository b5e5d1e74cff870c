"""Summarise a round's ncu captures (tools/prof_round2.sh) into profiles/:
raw + details CSVs of each full capture, the launch lists, a key-metric table
(printed, markdown) and profiles/ncu_traffic.json (dram bytes per launch, read
by bench.py for roofline.traffic).

usage: python tools/prof_extract.py TAG [config_id]"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

TAG = sys.argv[1]
CFG = int(sys.argv[2]) if len(sys.argv) > 2 else 1
OUT, PROF = "gpurun_out", "profiles"
# algorithmic bytes per launch, config 1 (256^3): K2 reads 12 forward-pack arrays
# + phi and writes R = 14 touches per cell; K3 reads 3 backward-pack arrays + R
# + phi and writes phi = 6 touches
CELLS = {1: 256 ** 3}[CFG]
ALG = {"fwd": 14, "bwd": 6}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
            "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(u, 1.0)


traffic = {}
try:
    traffic = json.load(open(os.path.join(PROF, "ncu_traffic.json")))
except Exception:
    pass
rows_md = []
for prec in ("f64", "f32"):
    es = 8 if prec == "f64" else 4
    tr = {}
    for kind in ("fwd", "bwd"):
        rep = os.path.join(OUT, f"prof_{kind}_{TAG}_{prec}.ncu-rep")
        if not os.path.exists(rep):
            print("missing", rep)
            continue
        raw = ncu(rep, "raw")
        det = ncu(rep, "details")
        open(os.path.join(PROF, f"{TAG}_ncu_{kind}_{prec}_raw.csv"), "w").write(raw)
        open(os.path.join(PROF, f"{TAG}_ncu_{kind}_{prec}_details.csv"), "w").write(det)
        rr = list(csv.reader(io.StringIO(raw)))
        h, units, vals = rr[0], rr[1], rr[2]
        m = {}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                try:
                    m[k] = float(vals[i].replace(",", "")) * unit_scale(units[i])
                except ValueError:
                    m[k] = vals[i]
        dur = m.get("gpu__time_duration.sum", float("nan"))
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        alg = ALG[kind] * CELLS * es
        name = "k_forward" if kind == "fwd" else "k_backward"
        tr[f"{name}_bytes_per_launch"] = int(rd + wr)
        tr[f"{name}_alg_bytes_per_launch"] = alg
        tr[f"{name}_ncu_ms"] = dur * 1e3
        rows_md.append(f"| {name} {prec} | {dur * 1e3:.3f} ms | {rd / 1e9:.3f} / {wr / 1e9:.3f} GB | "
                       f"{alg / 1e9:.3f} GB | {(rd + wr) / alg:.2f} | {alg / dur / 1e9:.0f} GB/s | "
                       f"{m.get('launch__grid_size', '?'):.0f} x {m.get('launch__block_size', '?'):.0f}, "
                       f"{m.get('launch__registers_per_thread', '?'):.0f} regs | "
                       f"{m.get('lts__t_sector_hit_rate.pct', float('nan')):.0f} % |")
    if tr:
        traffic[f"config{CFG}_{prec}"] = tr
    ll = os.path.join(OUT, f"launches_{TAG}_{prec}.csv")
    if os.path.exists(ll):
        shutil.copy(ll, os.path.join(PROF, f"{TAG}_launches_config{CFG}_{prec}.csv"))
        print(f"launch list {prec}:")
        print(subprocess.run([sys.executable, "tools/launch_summary.py", ll], capture_output=True,
                             text=True).stdout)
traffic["note"] = (f"dram__bytes_read.sum + dram__bytes_write.sum of one K2 (k_forward) / K3 (k_backward) "
                   f"launch from the ncu --set full captures TAG {TAG} (profiles/{TAG}_ncu_*_raw.csv), "
                   f"config {CFG}; alg = 14 (K2) / 6 (K3) element touches per cell")
json.dump(traffic, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
print("| kernel | ncu duration | dram read / write | algorithmic | traffic/alg | alg. bytes / duration | grid x block, regs | L2 hit |")
print("|---|---|---|---|---|---|---|---|")
print("\n".join(rows_md))
b = os.path.join(OUT, f"bench_{TAG}.json")
if os.path.exists(b):
    shutil.copy(b, os.path.join(PROF, f"{TAG}_bench.json"))
