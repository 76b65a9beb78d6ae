#!/usr/bin/env python
"""Benchmark of the data-parallel hot path of arXiv 2106.00003 on B200.

One step = the whole hot path on one batch: coefficient precompute (schedule + cos/sin
table), forward Y = U(theta) X (all n-1 blocks), replay backward (dX, dtheta with the
two-stage reduction) and, for N > 1, the NCCL all_reduce of dtheta. Workload (BASELINE.json
configs[2], "C3"): n = 1024, m = 65536 columns, fp32, synthetic seeded inputs; m is sharded
over the N ranks (strong scaling: the total m is fixed).

metric = Givens rotations/s fwd+bwd: units = N_angles * m (one 2x2 rotation applied to one
column, forward and backward); value = units / (max-over-ranks device time
per step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches its own N ranks
(one process per GPU, torch.distributed.run's environment, 127.0.0.1) and exits with their status; under a launcher it checks that
WORLD_SIZE == --gpus.

--impl reference times the fp64 CPU oracle (the only reference this paper has: it released no
code) on the host cores, on a bounded column sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Givens rotations/s fwd+bwd at n=1024 (1/2/4/8 B200); U-build ms vs n"
UNIT = "rotations/s"
N_DIM = 1024
M_TOTAL = 65536
SEED = 0
FP32_LANES_PER_SM = 128           # B200 SM: 4 SMSP x 32 FP32 lanes (B200_PROFILING.md / guide)
FLOPS_FWD, FLOPS_BWD = 6, 16      # algorithmic flops per rotation-column
FP32_MICROBENCH_TFLOPS = 71.7     # FFMA loop, 148 SMs at 1965 MHz (profiles/r2b_fp32_microbench.txt)
SPIN_CYCLES = 4_000_000            # ~2 ms GPU spin ahead of short timed sequences (host enqueue hidden)


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DIM)
    ap.add_argument("--m", type=int, default=M_TOTAL)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-cols-per-step", type=int, default=0,
                    help="reference arm columns per step (default 64 per oracle thread, so every core works)")
    ap.add_argument("--no-ubuild", action="store_true", help="skip the U-build ms vs n table")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return None
        mx = max(r[1] for r in rows)
        load = [r[0] for r in rows if r[0] > 0.5 * mx] or [r[0] for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ reference arm (CPU oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    import oracle
    import synth
    n, m = args.n, args.m
    N = n * (n - 1) // 2
    cores = oracle.num_threads()
    # the oracle splits columns into 64-column blocks over its OpenMP threads: 64 per thread keeps
    # every host core busy
    cols = args.ref_cols_per_step or 64 * cores
    th = synth.theta(N, seed=SEED)
    times = []
    for s in range(args.warmup + args.steps):
        c0 = (s * cols) % m
        X = synth.normal_matrix(n, m, SEED, synth.TID_X, c0, c0 + cols).astype(np.float64)
        dY = synth.normal_matrix(n, m, SEED, synth.TID_DY, c0, c0 + cols).astype(np.float64)
        t0 = time.perf_counter()
        oracle.apply(n, th, X)
        oracle.backward(n, th, X, dY)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = N * cols / t
    sample = f"{cols} of {m} columns per step (n={n}), fp64 oracle: Alg. 1 forward + taped reverse-mode backward"
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C3: n={n}, m={m} fwd+bwd (column sample per step)", "n": n, "m": m,
                   "sample_cols_per_step": cols},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(out), flush=True)


def cpu_baseline(args, target_s: float = 12.0):
    """The fp64 oracle, as it stands, on the host cores, on a bounded column sample of the same
    workload: a 128-column probe sizes the sample to ~target_s seconds of CPU work."""
    import numpy as np

    import oracle
    import synth
    n = args.n
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=SEED)

    def run(cols):
        X = synth.normal_matrix(n, args.m, SEED, synth.TID_X, 0, cols).astype(np.float64)
        dY = synth.normal_matrix(n, args.m, SEED, synth.TID_DY, 0, cols).astype(np.float64)
        t0 = time.perf_counter()
        oracle.apply(n, th, X)
        oracle.backward(n, th, X, dY)
        return time.perf_counter() - t0

    cols, t = 128, run(128)
    while t < 0.5 * target_s and cols < args.m:  # grow the sample until it is ~target_s of CPU work
        cols = int(min(args.m, max(2 * cols, cols * target_s / max(t, 1e-3)))) // 64 * 64
        t = run(cols)
    return {"value": N * cols / t, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"first {cols} of {args.m} columns (n={n}): fp64 Alg. 1 forward + taped backward, "
                      f"{t:.1f} s wall",
            "single_core": single_core_rate(n, args.m)}


def single_core_rate(n, m, cols=64):
    """The same oracle on ONE host thread (OMP_NUM_THREADS=1, a fresh process), on `cols` columns."""
    code = ("import time,sys,numpy as np; sys.path.insert(0, %r); import oracle, synth\n"
            "n,m,c=%d,%d,%d; th=synth.theta(n*(n-1)//2, seed=%d)\n"
            "X=synth.normal_matrix(n,m,%d,synth.TID_X,0,c).astype(np.float64)\n"
            "dY=synth.normal_matrix(n,m,%d,synth.TID_DY,0,c).astype(np.float64)\n"
            "t0=time.perf_counter(); oracle.apply(n,th,X); oracle.backward(n,th,X,dY)\n"
            "print(oracle.num_threads(), time.perf_counter()-t0)" % (ROOT, n, m, cols, SEED, SEED, SEED))
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, OMP_NUM_THREADS="1"))
        thr, t = r.stdout.split()[-2:]
        N = n * (n - 1) // 2
        return {"value": N * cols / float(t), "unit": UNIT, "cores": int(thr),
                "sample": f"first {cols} columns (n={n}), {float(t):.2f} s"}
    except Exception as e:  # the single-core figure is context only
        return {"error": repr(e)[:200]}


def ubuild_table(g, torch, synth, dev, ns=(256, 512, 1024, 1120, 2000, 2048, 4096)):
    """Device ms of build_U (forward from U <- I, Alg. 2) and of its gradient (Alg. 3 via the replay
    backward with Gamma = dL/dU) per n; mean of 10 back-to-back calls after a warm-up call (the
    paper averaged 50 runs).
    n = 1120 and 2000 are the paper's CPU and GPU maxima."""
    table = {}
    for n in ns:
        N = n * (n - 1) // 2
        th = torch.from_numpy(synth.theta(N, seed=SEED)).to(dev)
        G = torch.from_numpy(synth.normal_matrix(n, n, SEED, synth.TID_GAMMA)).to(dev)
        ws = g.workspace(g.OP_BACKWARD, n, n, dev)
        U = torch.empty(n, n, device=dev)
        dth = torch.empty(N, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        g.build_U(th, n, out=U, ws=ws)
        g.backward(th, U, G, ws=ws, recompute=False, dtheta=dth, want_dX=False)
        reps = 50
        # `reps` calls back to back behind a GPU-side spin: the host has enqueued them all before
        # the GPU reaches them, so the events bracket device time (sub-millisecond kernels would
        # otherwise include host enqueue gaps), and the once-per-sequence shared-memory carveout
        # switch after the spin is amortised over the calls
        torch.cuda._sleep(SPIN_CYCLES)
        ev[0].record()
        for _ in range(reps):
            g.build_U(th, n, out=U, ws=ws)
        ev[1].record()
        torch.cuda._sleep(SPIN_CYCLES)
        ev[2].record()
        for _ in range(reps):
            g.backward(th, U, G, ws=ws, recompute=False, dtheta=dth, want_dX=False)
        ev[3].record()
        torch.cuda.synchronize()
        tf, tb = ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])
        table[str(n)] = {"build_U_ms": round(tf / reps, 4), "grad_ms": round(tb / reps, 4)}
    return table


# flops per complex rotation-column of the unitary kernels: two real three-shear rotations
# (2 x 6) + the phase multiply (6); backward: Z and D replay (2 x 18) + dtheta (8) + dphi (20)
UFLOPS_FWD, UFLOPS_BWD = 18, 64


def small_config_line(g, torch, synth, dev, n=256, m=4096, reps=50):
    """BASELINE config C2 (n=256, m=4096, 1 GPU): device ms of apply + backward (dX, dtheta), mean of
    `reps` after warm-up, L2 flushed before each; latency-bound (28 columns per SM)."""
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=SEED)).to(dev)
    X = torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_X)).to(dev)
    dY = torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_DY)).to(dev)
    ws = g.workspace(g.OP_BACKWARD, n, m, dev)
    Y, dX, dth = torch.empty_like(X), torch.empty_like(X), torch.empty(N, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(3):
        g.apply(th, X, out=Y, ws=ws)
        g.backward(th, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        ev[0].record()
        g.apply(th, X, out=Y, ws=ws)
        ev[1].record()
        g.backward(th, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    tf, tb = tf / reps, tb / reps
    return {"workload": f"C2 n={n}, m={m}: apply + backward (dX, dtheta)", "fwd_ms": round(tf, 4),
            "bwd_ms": round(tb, 4), "rotations_per_s": N * m / ((tf + tb) * 1e-3)}


def c5_shard_line(g, torch, synth, dev, n=2047, m=32768, m_keep=1024, reps=5):
    """BASELINE config C5 as one rank of its 8-GPU run: n = 2047 (odd: the bye vertex), the rank's
    m = 262144 / 8 = 32768 columns, the SURVEY §5 restriction mask m_keep = 1024 (pinned angles are
    identity rotations, dtheta = 0). Device ms of apply + backward (dX, dtheta), mean of `reps`
    after warm-up, L2 flushed before each. Rates count active (unpinned) angles."""
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=SEED)).to(dev)
    mask = torch.from_numpy(g.mask_from_keep(n, m_keep)).to(dev)
    X = torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_X)).to(dev)
    dY = torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_DY)).to(dev)
    ws = g.workspace(g.OP_BACKWARD, n, m, dev)
    Y, dX, dth = torch.empty_like(X), torch.empty_like(X), torch.empty(N, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(2):
        g.apply(th, X, mask=mask, out=Y, ws=ws)
        g.backward(th, Y, dY, mask=mask, ws=ws, recompute=False, dtheta=dth, dX=dX)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        ev[0].record()
        g.apply(th, X, mask=mask, out=Y, ws=ws)
        ev[1].record()
        g.backward(th, Y, dY, mask=mask, ws=ws, recompute=False, dtheta=dth, dX=dX)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    tf, tb = tf / reps, tb / reps
    active = int(mask.sum().item())  # 1 = free angle (include/givens.h)
    ne = n + (n & 1)
    executed = (ne - 1) * (ne // 2)  # every slot of every block runs, pinned and bye ones as identities
    return {"workload": f"C5 one rank of 8: n={n} (odd), m={m} of 262144 columns, mask m_keep={m_keep}: "
                        "apply + backward (dX, dtheta)",
            "fwd_ms": round(tf, 4), "bwd_ms": round(tb, 4), "active_angles": active, "executed_slots": executed,
            "active_rotations_per_s": active * m / ((tf + tb) * 1e-3),
            "executed_rotations_per_s": executed * m / ((tf + tb) * 1e-3)}


def unitary_line(g, torch, synth, dev, peak_tflops, n=1024, m=32768, reps=5):
    """the unitary U(n) path (Appendix A) at n = 1024 on m complex columns (the same
    2m = 65536 real columns as C3): device ms of u_apply and u_backward, mean of `reps` after
    warm-up, L2 flushed before each."""
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=SEED)).to(dev)
    ph = torch.from_numpy(synth.theta(N, seed=SEED + 1)).to(dev)
    X = torch.complex(torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_X)),
                      torch.from_numpy(synth.normal_matrix(n, m, SEED + 1, synth.TID_X))).to(dev)
    G = torch.complex(torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_DY)),
                      torch.from_numpy(synth.normal_matrix(n, m, SEED + 1, synth.TID_DY))).to(dev)
    wsb = g.workspace(g.OP_U_BACKWARD, n, m, dev)
    wsf = g.workspace(g.OP_U_APPLY, n, m, dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    Y = g.u_apply(th, ph, X, ws=wsf)
    g.u_backward(th, ph, Y, G, ws=wsb)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tf = tb = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        ev[0].record()
        g.u_apply(th, ph, X, out=Y, ws=wsf)
        ev[1].record()
        flush.fill_(2.0)
        ev[2].record()
        g.u_backward(th, ph, Y, G, ws=wsb)
        ev[3].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[2].elapsed_time(ev[3])
    tf, tb = tf / reps, tb / reps
    return {"workload": f"unitary n={n}, m={m} complex columns (fp32 re/im), u_apply + u_backward (dtheta, dphi, dX)",
            "fwd_ms": round(tf, 4), "bwd_ms": round(tb, 4),
            "complex_rotations_per_s": N * m / ((tf + tb) * 1e-3),
            "fwd_frac": UFLOPS_FWD * N * m / (tf * 1e-3) / 1e12 / peak_tflops,
            "bwd_frac": UFLOPS_BWD * N * m / (tb * 1e-3) / 1e12 / peak_tflops,
            "flops_per_complex_rotation_column": {"fwd": UFLOPS_FWD, "bwd": UFLOPS_BWD}}


def step_reps(g, torch, theta, X, dY, n, reps=50, m_cols=None):
    """The paper's protocol ("averaged over 50 runs"): `reps` timed steps (precompute +
    forward + backward), each after an L2 flush, CUDA events on the stream; mean / std / min ms.
    m_cols < m times the step on the first m_cols columns (one rank's shard of a G-GPU run)."""
    dev = X.device
    if m_cols is not None:
        X, dY = X[:, :m_cols].contiguous(), dY[:, :m_cols].contiguous()
    m = X.shape[1]
    ws = g.workspace(g.OP_BACKWARD, n, m, dev)
    Y, dX, dth = torch.empty_like(X), torch.empty_like(X), torch.empty_like(theta)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def step():
        g.apply(theta, X, out=Y, ws=ws)
        g.backward(theta, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
    for _ in range(3):
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for k in range(reps):
        flush.fill_(float(k))
        ev[k][0].record()
        step()
        ev[k][1].record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ev]
    return {"reps": reps, "m": m, "mean_ms": statistics.mean(t), "std_ms": statistics.stdev(t), "min_ms": min(t),
            "max_ms": max(t)}


def fast_givens_line(g, torch, synth, dev, peak_tflops, n=64, m=1 << 20, reps=20):
    """SURVEY §8(f4) measured beside the default: Y = U X at n = 64 (one-lane columns, where the
    factoring choice of fast Givens is warp-uniform) by the three-shear ring (3 FFMA per
    rotation-column) and by fast Givens (2 FFMA + the scaled store); device ms per call, mean of
    `reps` back to back after warm-up, and each against the FP32 FLOP roofline (6 flops per
    rotation-column)."""
    N = n * (n - 1) // 2
    th = torch.from_numpy(synth.theta(N, seed=SEED)).to(dev)
    X = torch.from_numpy(synth.normal_matrix(n, m, SEED, synth.TID_X)).to(dev)
    Y = torch.empty_like(X)
    ws = g.workspace(g.OP_APPLY, n, m, dev)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    ts = timed(lambda: g.apply(th, X, out=Y, ws=ws))
    tf = timed(lambda: g.fast_apply(th, X, out=Y, ws=ws))
    fl = FLOPS_FWD * N * m
    return {"workload": f"n={n}, m={m}: Y = U X (one-lane columns)", "three_shear_ms": round(ts, 4),
            "fast_givens_ms": round(tf, 4), "three_shear_frac": fl / (ts * 1e-3) / 1e12 / peak_tflops,
            "fast_givens_frac": fl / (tf * 1e-3) / 1e12 / peak_tflops, "speedup_fast_vs_three_shear": round(ts / tf, 3)}


def _measured_peak(key, default):
    """A number from the driver-written MEASURED_PEAKS.json, else the stated fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))[key])
    except Exception:
        return default


def gemm_path_line(g, torch, theta, X, dY, n, m, ring_ms, tf32_peak, reps=10):
    """SURVEY §8(f2) measured beside the ring: the same C3 fwd+bwd outputs (Y, dX, dtheta) from
    U-build (ring) + 3xTF32 tensor-core GEMMs + Alg. 3 on Gamma (givens_gemm_apply/backward).
    Device ms per step (mean of `reps` after warm-up, L2 flushed before each)."""
    dev = X.device
    ws = g.gemm_workspace(n, m, dev)
    Y = torch.empty_like(X)
    dX = torch.empty_like(X)
    dth = torch.empty_like(theta)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(3):
        g.gemm_apply(theta, X, out=Y, ws=ws)
        g.gemm_backward(theta, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tf = tb = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        ev[0].record()
        g.gemm_apply(theta, X, out=Y, ws=ws)
        ev[1].record()
        g.gemm_backward(theta, Y, dY, ws=ws, recompute=False, dtheta=dth, dX=dX)
        ev[2].record()
        torch.cuda.synchronize()
        tf += ev[0].elapsed_time(ev[1])
        tb += ev[1].elapsed_time(ev[2])
    tf, tb = tf / reps, tb / reps
    N = n * (n - 1) // 2
    gemm_flops = 3 * (3 * 2.0 * n * n * m)  # Y = U X, dX = U^T dY, M = dY Y^T; three TF32 products each
    return {"workload": f"C3 n={n}, m={m}: same outputs as the headline step (Y, dX, dtheta)",
            "path": "build_U (ring) + 3xTF32 GEMMs (own tcgen05 kernel: TMA, in-kernel hi/lo split, TMEM; K-chunked) + Alg. 3 on Gamma (ring replay, X = I)",
            "fwd_ms": round(tf, 4), "bwd_ms": round(tb, 4), "ms_per_step": round(tf + tb, 4),
            "equivalent_rotations_per_s": N * m / ((tf + tb) * 1e-3),
            "speedup_vs_ring": round(ring_ms / (tf + tb), 3),
            "tf32_gemm_flops_per_step": gemm_flops,
            "tf32_peak_tflops": tf32_peak,
            # the whole step's TF32 tensor-core work over the whole step's time (U-build and Alg. 3 included)
            "tf32_achieved_tflops_step": gemm_flops / ((tf + tb) * 1e-3) / 1e12,
            "tf32_frac_step": gemm_flops / ((tf + tb) * 1e-3) / 1e12 / tf32_peak,
            "note": "not the headline: the headline is the SURVEY 8(a) ring path; this is the 8(f2) row"}


# ------------------------------------------------------------------ our arm
def self_launch(args):
    """--gpus N > 1 without a launcher: start N ranks of this script on one node, as
    torch.distributed.run would (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR=127.0.0.1 / a free
    MASTER_PORT in each rank's environment), and return the worst exit status."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), GROUP_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2106_00003_b200 as g
    from paper_2106_00003_b200.dist import allreduce_dtheta, shard_columns

    # GIVENS_BENCH_SHARE_GPU=1 maps every rank to cuda:0 and uses gloo: a functional test of the
    # multi-rank flow on a 1-GPU box (never a scaling number)
    share = os.environ.get("GIVENS_BENCH_SHARE_GPU") == "1"
    dev = torch.device("cuda", 0 if share else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    n, m_total = args.n, args.m
    N = n * (n - 1) // 2
    c0, c1 = shard_columns(m_total, rank, world)
    m = c1 - c0

    # seeded synthetic inputs, generated for this rank's column shard only
    th_h = synth.theta(N, seed=SEED)
    X_h = synth.normal_matrix(n, m_total, SEED, synth.TID_X, c0, c1)
    dY_h = synth.normal_matrix(n, m_total, SEED, synth.TID_DY, c0, c1)
    theta = torch.from_numpy(th_h).to(dev)
    X = torch.from_numpy(X_h).to(dev)
    dY = torch.from_numpy(dY_h).to(dev)
    Y = torch.empty_like(X)
    dX = torch.empty_like(X)
    dtheta = torch.empty(N, dtype=torch.float32, device=dev)
    ws = g.workspace(g.OP_BACKWARD, n, m, dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step():
        g.apply(theta, X, out=Y, ws=ws)                                  # precompute + forward
        e_b0.record(stream)
        g.backward(theta, Y, dY, ws=ws, recompute=False, dtheta=dtheta, dX=dX)  # replay bwd + stage 2
        e_b1.record(stream)
        if world > 1:
            allreduce_dtheta(dtheta)

    e_b0 = torch.cuda.Event(enable_timing=True)
    e_b1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    bwd_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(float(k))          # L2 flush between timed steps (outside the step events)
        starts[k].record(stream)
        step()
        ends[k].record(stream)
        e_b1.synchronize()
        bwd_ms.append(e_b0.elapsed_time(e_b1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    step_stats = {"mean_ms": statistics.mean(step_ms), "min_ms": min(step_ms), "max_ms": max(step_ms),
                  "std_ms": statistics.stdev(step_ms) if len(step_ms) > 1 else 0.0}
    t_rank = torch.tensor([sum(step_ms) / len(step_ms), sum(bwd_ms) / len(bwd_ms)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_rank, op=dist.ReduceOp.MAX)
    ms_step, ms_bwd = float(t_rank[0]), float(t_rank[1])
    units = N * m_total
    value = units / (ms_step * 1e-3)

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # the step's inputs live in pinned host memory; HostPipeline overlaps the H2D copy of
        # batch k+1 with the compute of batch k and returns dtheta to the host every step
        Xp = torch.from_numpy(X_h).pin_memory()
        dYp = torch.from_numpy(dY_h).pin_memory()
        pipe = g.HostPipeline(theta, n, m, want_dX=True, device=dev,
                              allreduce=allreduce_dtheta if world > 1 else None)
        ks = max(3, args.steps // 2)
        total = 2 + ks
        pipe.submit(Xp, dYp)
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for k in range(total):
            if k == 2:
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                es.record(stream)
            if k + 1 < total:
                pipe.submit(Xp, dYp)
            pipe.step()
        ee.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([es.elapsed_time(ee) / ks], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": units / (float(te[0]) * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 2 * 4 * n * m,
               "d2h_bytes_per_step": 4 * N, "ms_per_step": float(te[0]),
               "api": "paper_2106_00003_b200.HostPipeline (H2D of batch k+1 overlapped with batch k)"}

    # ---------------- U-build ms vs n (the metric's second half; the paper's Fig. 2 axes)
    ubuild = None
    if rank == 0 and world == 1 and not args.no_ubuild:
        ubuild = ubuild_table(g, torch, synth, dev)

    if rank == 0:
        sm_mhz = (clk or {}).get("sm_mhz")
        peak_clock = 1965.0
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = n_sm * FP32_LANES_PER_SM * 2 * peak_clock * 1e6 / 1e12   # TFLOP/s at max boost clock
        achieved = FLOPS_BWD * N * m / (ms_bwd * 1e-3) / 1e12
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "bwd_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"C3: n={n}, m={m_total} fwd+bwd (precompute + forward + replay backward"
                                   f"{' + NCCL all_reduce(dtheta)' if world > 1 else ''}), m sharded over ranks",
                       "n": n, "m": m_total, "m_per_rank": m, "angles": N,
                       "l2": "flushed between steps (256 MiB write outside the step events); X is 256 MiB at N=1",
                       "seed": SEED, "parallelism": f"dp{world}"},
            "roofline": {"bound": "alu", "kernel": "givens_backward (k_ring<16,BWD> + k_dtheta_reduce)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "peak_basis": f"{n_sm} SM x {FP32_LANES_PER_SM} FP32 lanes x 2 flop x {peak_clock:.0f} MHz "
                                       "(max boost; DESIGN.md §5)",
                         "flops_per_rotation_column": FLOPS_BWD, "ms_per_launch": ms_bwd,
                         # the FFMA-loop microbenchmark's rate on this pool's B200s (tools/microbench.cu,
                         # profiles/r2b_fp32_microbench.txt, 1965 MHz): the frac against it, for context
                         "peak_measured_microbench": FP32_MICROBENCH_TFLOPS,
                         "frac_vs_microbench": achieved / FP32_MICROBENCH_TFLOPS,
                         # the whole step (precompute + forward + backward) against the same peak, at
                         # 6 + 16 algorithmic flops per rotation-column
                         "step_achieved": (FLOPS_FWD + FLOPS_BWD) * N * m / (ms_step * 1e-3) / 1e12,
                         "step_frac": (FLOPS_FWD + FLOPS_BWD) * N * m / (ms_step * 1e-3) / 1e12 / peak},
            "bwd_ms": ms_bwd, "fwd_ms": ms_step - ms_bwd, "step_ms_stats_rank0": step_stats,
            # forward-only (precompute + forward) and backward-only (replay + stage 2) rates
            "fwd_rotations_per_s": units / ((ms_step - ms_bwd) * 1e-3), "bwd_rotations_per_s": units / (ms_bwd * 1e-3),
            # our kernels per step: k_sigma_bits, k_coef (precompute), forward, backward, stage-2 reduce
            "gpu_launches": 5 * args.steps,
            "clocks": clk,
        }
        if e2e:
            out["e2e"] = e2e
        if ubuild:
            out["ubuild_ms_vs_n"] = ubuild
        if world == 1 and not args.no_ubuild:
            out["paper_protocol_50"] = step_reps(g, torch, theta, X, dY, n)
            # one rank's share of a G-GPU run of the same C3 step, timed here: the per-rank device
            # time at G GPUs is this plus the dtheta all_reduce
            scan = {}
            for G in (2, 4, 8):
                r = step_reps(g, torch, theta, X, dY, n, reps=20, m_cols=m // G)
                scan[str(G)] = {"m_per_rank": m // G, "mean_ms": r["mean_ms"], "min_ms": r["min_ms"],
                                "speedup_no_comm": out["paper_protocol_50"]["mean_ms"] / r["mean_ms"]}
            out["shard_scan"] = scan
            out["c2"] = small_config_line(g, torch, synth, dev)
            out["c5_shard"] = c5_shard_line(g, torch, synth, dev)
            out["unitary"] = unitary_line(g, torch, synth, dev, peak)
            out["f4_fast_givens"] = fast_givens_line(g, torch, synth, dev, peak)
            bf16 = _measured_peak("bf16_tflops", 2250.0)
            out["f2_gemm_path"] = gemm_path_line(g, torch, theta, X, dY, n, m, ms_step, bf16 / 2)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
