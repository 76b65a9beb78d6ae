"""Turn a tools/profile.sh run (gpurun_out/TAG/) into committed summaries under profiles/ (runs here,
no GPU): the launch list with each kernel's share of the C3 step, per case and kernel the key
`--set full` metrics (time, FMA-pipe and issue utilisation, executed FP32 instruction counts,
local-memory traffic, DRAM / L2 bytes, registers, occupancy, the warp-stall breakdown), and the FP32
peak microbenchmark output with the SM clocks sampled while it ran.

usage: python tools/summarize_ncu.py TAG"""
import collections
import csv
import gzip
import io
import json
import os
import shutil
import statistics
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(root, "gpurun_out", tag)
dst = os.path.join(root, "profiles")
os.makedirs(dst, exist_ok=True)

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.sum", "smsp__inst_executed.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "us": 1e3, "ms": 1e6,
         "nsecond": 1, "usecond": 1e3, "msecond": 1e6}  # times in ns, bytes in bytes


def read_csv(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        txt = f.read()
    i = txt.find('"ID"')
    return list(csv.reader(io.StringIO(txt[i:]))) if i >= 0 else []


def num(v, unit):
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1)


out = {"tag": tag, "cases": {}}
# 1) launch list of the bench: share of each kernel in the last step
lp = os.path.join(src, "launches.csv")
if os.path.exists(lp):
    rows = []
    with open(lp) as f:
        txt = f.read()
    txt = txt[txt.index('"ID"'):]
    for r in csv.DictReader(io.StringIO(txt)):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((int(r["ID"]), r["Kernel Name"].split("(")[0], float(r["Metric Value"].replace(",", ""))))
    with open(os.path.join(dst, f"{tag}_launches.csv"), "w") as f:
        f.write("id,kernel,gpu__time_duration_ns\n")
        for i, k, v in rows:
            f.write(f"{i},{k},{v:.0f}\n")
    tot = collections.Counter()
    for _, k, v in rows[-6:]:  # one full step: 3 precompute + forward + backward + stage 2
        tot[k] += v
    T = sum(tot.values())
    out["c3_step_share_from_launch_list"] = {k: {"ns": v, "share": round(v / T, 4)} for k, v in tot.items()}

# 2) per case, per kernel launch: key metrics and stalls from the raw page
for fn in sorted(os.listdir(src)) if os.path.isdir(src) else []:
    if not (fn.endswith(".raw.csv.gz") or fn.endswith(".raw.csv")):
        continue
    case = fn.split(".")[0]
    rr = read_csv(os.path.join(src, fn))
    if len(rr) < 3:
        continue
    hdr, units = rr[0], rr[1]
    kerns = []
    for r in rr[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                d[k] = num(r[hdr.index(k)], units[hdr.index(k)])
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                v = num(r[i], "")
                if isinstance(v, float) and v > 0.02:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        kerns.append(d)
    out["cases"][case] = kerns

json.dump(out, open(os.path.join(dst, f"{tag}_ncu_summary.json"), "w"), indent=1)

# 3) the C3 backward ring kernel's DRAM traffic per launch (bench.py roofline.traffic)
for d in out["cases"].get("c3", []):
    if "k_ring" in d["kernel"] and ", 3>" in d["kernel"]:
        json.dump({"kernel": d["kernel"], "dram_bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                   "lts_bytes_per_launch": d.get("lts__t_bytes.sum"), "source": f"profiles/{tag}_ncu_summary.json"},
                  open(os.path.join(dst, "bwd_traffic.json"), "w"), indent=1)

# 4) microbenchmarks + clocks
mb = os.path.join(src, "microbench.txt")
if os.path.exists(mb):
    shutil.copy(mb, os.path.join(dst, f"{tag}_fp32_microbench.txt"))
    clk = os.path.join(src, "clocks_microbench.csv")
    if os.path.exists(clk):
        sm = []
        for line in open(clk).read().splitlines()[1:]:
            p = [x.strip() for x in line.split(",")]
            try:
                sm.append(float(p[1].split()[0]))
            except (IndexError, ValueError):
                pass
        busy = [v for v in sm if v > 1000] or sm
        with open(os.path.join(dst, f"{tag}_fp32_microbench.txt"), "a") as f:
            f.write(f"\n# nvidia-smi SM clock while the microbenchmarks ran: {len(sm)} samples, median under load "
                    f"{statistics.median(busy) if busy else 'n/a'} MHz, min {min(busy) if busy else 'n/a'}, "
                    f"max {max(busy) if busy else 'n/a'}\n")
        shutil.copy(clk, os.path.join(dst, f"{tag}_fp32_microbench_clocks.csv"))
for fn in os.listdir(src) if os.path.isdir(src) else []:
    if fn.endswith(".source.csv.gz"):
        shutil.copy(os.path.join(src, fn), os.path.join(dst, f"{tag}_{fn}"))
print(json.dumps({c: [(k["kernel"][:40], k.get("gpu__time_duration.sum")) for k in v] for c, v in out["cases"].items()},
                 indent=1)[:4000])
