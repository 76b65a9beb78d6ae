"""Turn gpurun_out/ ncu artefacts into committed summaries under profiles/ (run here, no GPU)."""
import csv, io, json, os, subprocess, sys, collections

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go, pr = os.path.join(root, "gpurun_out"), os.path.join(root, "profiles")
os.makedirs(pr, exist_ok=True)

# 1) launch list -> per-kernel share of the step
rows = []
txt = open(os.path.join(go, f"launches_{tag}.csv")).read()
txt = txt[txt.index('"ID"'):]
for r in csv.DictReader(io.StringIO(txt)):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((int(r["ID"]), r["Kernel Name"].split("(")[0], float(r["Metric Value"])))
with open(os.path.join(pr, f"{tag}_launches.csv"), "w") as f:
    f.write("id,kernel,gpu__time_duration_ns\n")
    for i, k, v in rows:
        f.write(f"{i},{k},{v:.0f}\n")
# last full step (launches after warm-up): 8 launches per step (k_layout, k_flip, k_sigma_seg, k_sigma_fill, k_coef, fwd, bwd, reduce)
tot = collections.Counter()
for i, k, v in rows[-8:]:
    tot[k] += v
T = sum(tot.values())
share = {k: {"ns": v, "share": v / T} for k, v in tot.items()}

# 2) --set full capture -> key metrics per ring kernel
keys = ["gpu__time_duration.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__warps_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "launch__grid_size", "launch__block_size"]
raw = subprocess.run(["ncu", "-i", os.path.join(go, f"ring_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units = rr[0], rr[1]
kern = {}
for r in rr[2:]:
    name = r[hdr.index("Kernel Name")]
    d = {}
    for k in keys:
        if k in hdr:
            d[k] = {"value": r[hdr.index(k)], "unit": units[hdr.index(k)]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.02:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
    d["stalls_per_issue"] = stalls
    kern[name] = d
out = {"tag": tag, "step_share_from_launch_list": share, "ring_kernels_set_full": kern}
json.dump(out, open(os.path.join(pr, f"{tag}_ncu_summary.json"), "w"), indent=1)
# traffic of the backward ring kernel per launch (bench.py roofline.traffic)
for name, d in kern.items():
    if "3>" in name or ", 3>" in name:
        def gb(k):
            v = float(d[k]["value"]); u = d[k]["unit"]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        json.dump({"kernel": name, "dram_bytes_per_launch": gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum"),
                   "source": f"profiles/{tag}_ncu_summary.json"}, open(os.path.join(pr, "bwd_traffic.json"), "w"), indent=1)
print(json.dumps(share, indent=1))
