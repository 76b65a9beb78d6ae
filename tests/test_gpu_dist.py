"""The multi-GPU product path executed on one GPU: two ranks (gloo; both
mapped to cuda:0, as bench.py's GIVENS_BENCH_SHARE_GPU mode) each run the CUDA apply + backward
on their contiguous column shard and all-reduce dtheta (sum and deterministic modes). dtheta is a
sum over columns ("d <- A 1"), so the sharded result must equal the oracle's
full-batch dtheta; Y and dX are per-column (each column's arithmetic does not depend on the rank
or slab that computes it), so they must equal the 1-rank run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from _parity import rel
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2106_00003_b200 as g
    from paper_2106_00003_b200.dist import allreduce_dtheta, shard_columns
    N = n * (n - 1) // 2
    c0, c1 = shard_columns(m, rank, world)
    th = torch.from_numpy(synth.theta(N, seed=5)).cuda()
    X = torch.from_numpy(synth.normal_matrix(n, m, 5, synth.TID_X, c0, c1)).cuda()
    dY = torch.from_numpy(synth.normal_matrix(n, m, 5, synth.TID_DY, c0, c1)).cuda()
    Y = g.apply(th, X)
    dth, dX = g.backward(th, Y, dY)
    d_sum = allreduce_dtheta(dth.clone())
    d_det = allreduce_dtheta(dth.clone(), deterministic=True)
    d_det2 = allreduce_dtheta(dth.clone(), deterministic=True)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"Y{rank}.npy"), Y.cpu().numpy())
    np.save(os.path.join(out_dir, f"dX{rank}.npy"), dX.cpu().numpy())
    if rank == 0:
        np.save(os.path.join(out_dir, "sum.npy"), d_sum.cpu().numpy())
        np.save(os.path.join(out_dir, "det.npy"), d_det.cpu().numpy())
        np.save(os.path.join(out_dir, "det2.npy"), d_det2.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,m", [(256, 4096), (1024, 2048), (2047, 301)])
def test_two_rank_shard_allreduce(tmp_path, n, m):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_00003_b200 as g
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), n, m, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=5)
    X = synth.normal_matrix(n, m, 5, synth.TID_X)
    dY = synth.normal_matrix(n, m, 5, synth.TID_DY)
    # the 1-rank run on the same device
    tt = torch.from_numpy(th).cuda()
    Y1 = g.apply(tt, torch.from_numpy(X).cuda())
    d1, dX1 = g.backward(tt, Y1, torch.from_numpy(dY).cuda())
    Y2 = np.concatenate([np.load(tmp_path / f"Y{r}.npy") for r in range(world)], axis=1)
    dX2 = np.concatenate([np.load(tmp_path / f"dX{r}.npy") for r in range(world)], axis=1)
    assert np.array_equal(Y2, Y1.cpu().numpy())
    assert np.array_equal(dX2, dX1.cpu().numpy())
    d_sum, d_det, d_det2 = (np.load(tmp_path / f) for f in ("sum.npy", "det.npy", "det2.npy"))
    assert np.array_equal(d_det, d_det2)  # deterministic mode: bitwise reproducible
    dto, _ = oracle.backward(n, th, X.astype(np.float64), dY.astype(np.float64), want_dX=False)
    assert rel(d_sum, dto) <= 1e-4
    assert rel(d_det, dto) <= 1e-4
    assert rel(d_det, d1.cpu().numpy()) <= 1e-5  # 2 shards vs 1: only the summation order differs


def test_bench_two_rank_share_gpu():
    """bench.py --gpus 2 launches its own two ranks (torch.distributed.run) when WORLD_SIZE is
    unset; with GIVENS_BENCH_SHARE_GPU=1 both map to cuda:0 (a functional run of the multi-rank
    flow, never a scaling number): one JSON line with n_gpus = 2."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GIVENS_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--n", "256", "--m", "4096", "--no-cpu-baseline", "--no-ubuild"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["config"]["parallelism"] == "dp2" and out["value"] > 0
