"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel plumbing: the m columns
are sharded over ranks, each rank computes its shard's dtheta, and one all_reduce(SUM) gives the
full-batch dtheta (dtheta is a sum over columns). The per-shard dtheta here
comes from the fp64 oracle (CPU), so the test exercises the sharding and the collective, not
the kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_00003_b200.dist import allreduce_dtheta, shard_columns


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, m, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    N = n * (n - 1) // 2
    c0, c1 = shard_columns(m, rank, world)
    th = synth.theta(N, seed=3)
    X = synth.normal_matrix(n, m, 3, synth.TID_X, c0, c1).astype(np.float64)
    dY = synth.normal_matrix(n, m, 3, synth.TID_DY, c0, c1).astype(np.float64)
    d, _ = oracle.backward(n, th, X, dY, want_dX=False)
    t1 = torch.from_numpy(d.copy())
    t2 = torch.from_numpy(d.copy())
    allreduce_dtheta(t1)
    allreduce_dtheta(t2, deterministic=True)
    if rank == 0:
        np.save(os.path.join(out_dir, "sum.npy"), t1.numpy())
        np.save(os.path.join(out_dir, "det.npy"), t2.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [40, 41])
def test_sharded_dtheta_allreduce_gloo(tmp_path, m):
    import oracle
    import synth
    n, world = 9, 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n, m, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    N = n * (n - 1) // 2
    th = synth.theta(N, seed=3)
    X = synth.normal_matrix(n, m, 3, synth.TID_X).astype(np.float64)
    dY = synth.normal_matrix(n, m, 3, synth.TID_DY).astype(np.float64)
    full, _ = oracle.backward(n, th, X, dY, want_dX=False)
    np.testing.assert_allclose(np.load(tmp_path / "sum.npy"), full, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.load(tmp_path / "det.npy"), full, rtol=1e-12, atol=1e-12)


def test_shard_columns_cover():
    for m in [1, 7, 64, 65536, 65537]:
        for w in [1, 2, 3, 4, 8]:
            spans = [shard_columns(m, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
