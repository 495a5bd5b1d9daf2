"""Product-level data parallelism with world_size 2 (SPEC S:336
"path m depends only on (seed, m), so any partitioning yields identical
results", "shard gradients are summed before adam_step").

Two processes, each with its own libbsde context on cuda:0 owning the global
paths [rB/2, (r+1)B/2) (rank/world given, no NCCL communicator: the
collective-free shard mode), sum their gradients and Σ R² through a
torch.distributed `gloo` allreduce, and must reproduce the single context over
all B paths.  The two ranks' kernels never wait on each other (the exchange is
on the host), so sharing one GPU is safe.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {"tc": ("allen_cahn", 100, 110, 4, 0.3, 1000, "bf16", "tc"),
         "simt": ("hjb", 100, 110, 3, 1.0, 600, "fp32", "simt")}


def _worker(rank, world, port, case, params, q):
    import torch
    import torch.distributed as dist
    from paper_1910_11623_b200 import BSDE
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank,
                            world_size=world)
    prob, d, w, N, T, B, prec, kern = CASES[case]
    s = BSDE(prob, d, N, T, w, B, precision=prec, kernel=kern, rank=rank, world=world)
    s.set_params(params)
    loss = s.compute_grad()
    g = torch.from_numpy(s.get_grads().astype(np.float64))
    L = torch.tensor([loss], dtype=torch.float64)
    dist.all_reduce(g)
    dist.all_reduce(L)
    q.put((rank, L.item(), g.numpy()))
    s.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_world2_gloo_shards_equal_single_context(case):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_1910_11623_b200 import BSDE
    prob, d, w, N, T, B, prec, kern = CASES[case]
    full = BSDE(prob, d, N, T, w, B, precision=prec, kernel=kern)
    p = full.get_params()
    p[1:] += (0.003 * np.random.default_rng(11).standard_normal(p.size - 1)).astype(np.float32)
    full.set_params(p)
    lf = full.compute_grad()
    gf = full.get_grads().astype(np.float64)
    full.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict((r, (l, g)) for r, l, g in (q.get(timeout=300) for _ in procs))
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    (l0, g0), (l1, g1) = out[0], out[1]
    assert l0 == l1 and np.array_equal(g0, g1)          # both ranks hold the same sum
    assert abs(l0 - lf) <= 1e-5 * lf, (l0, lf)
    assert np.linalg.norm(g0 - gf) <= 1e-5 * np.linalg.norm(gf)
    assert np.max(np.abs(g0 - gf)) <= 1e-4 * np.max(np.abs(gf))
