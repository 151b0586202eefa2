"""Multi-process (gloo, world_size 2, CPU) checks of the batch-sharding path.

Each rank computes its shard's interval-bound gradients with the CPU oracle
(the per-shard compute stands in for the GPU kernels, which need a device) and
the ranks all-reduce them with ``allreduce_interval_grads`` — the one
collective of the multi-GPU path.  The result must equal the
full-batch d(a, b, c), and the sharding must cover every row exactly once.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_04194_b200.distributed import allreduce_interval_grads, shard_rows


def test_shard_rows_partition():
    for B in (1, 2, 7, 1024, 4097):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                sl = shard_rows(B, r, world)
                seen.extend(range(sl.start, sl.stop))
            assert seen == list(range(B))
            sizes = [shard_rows(B, r, world).stop - shard_rows(B, r, world).start for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, L, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "..", "oracle"))
    import stl_oracle
    import paper_2501_04194_b200 as P
    rng = np.random.default_rng(5)
    x = np.asarray(rng.normal(0.3, 1, (B, L)), dtype=np.float32).astype(np.float64)
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f = P.Always(P.Pred("x", ">", 0.0), si)
    cfg = P.SemanticsConfig(mode=P.LogSumExp(5.0))
    sl = shard_rows(B, rank, world)
    _, _, dabc = stl_oracle.trace_and_grad(f, {"x": x[sl]}, cfg, smooth_binding=(si.a, si.b, si.c))
    params = [torch.tensor(v, dtype=torch.float64, requires_grad=True) for v in (si.a, si.b, si.c)]
    for p_, g in zip(params, dabc):
        p_.grad = torch.tensor(g, dtype=torch.float64)
    allreduce_interval_grads(params)
    out_q.put((rank, [float(p_.grad) for p_ in params]))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_of_interval_grads_equals_full_batch():
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "..", "oracle"))
    import stl_oracle
    import paper_2501_04194_b200 as P
    B, L, world = 6, 80, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, L, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    rng = np.random.default_rng(5)
    x = np.asarray(rng.normal(0.3, 1, (B, L)), dtype=np.float32).astype(np.float64)
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f = P.Always(P.Pred("x", ">", 0.0), si)
    cfg = P.SemanticsConfig(mode=P.LogSumExp(5.0))
    _, _, full = stl_oracle.trace_and_grad(f, {"x": x}, cfg, smooth_binding=(si.a, si.b, si.c))
    for r in range(world):
        np.testing.assert_allclose(res[r], full, rtol=1e-12, atol=1e-12)


def _none_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = [torch.tensor(v, dtype=torch.float64, requires_grad=True) for v in (0.3, 0.65, 9.0)]
    if rank == 0:  # rank 1 has no interval gradient at all (e.g. its rows skipped the binding)
        for p_, g in zip(params, (1.0, 2.0, 3.0)):
            p_.grad = torch.tensor(g, dtype=torch.float64)
        allreduce_interval_grads(params)
    else:
        allreduce_interval_grads([None, params[1], None])
    out_q.put((rank, [None if p_.grad is None else float(p_.grad) for p_ in params]))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_joins_ranks_without_grads():
    """a rank without gradients must still join the collective (zeros)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_none_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert res[0] == [1.0, 2.0, 3.0]
    assert res[1] == [None, 2.0, None]


def test_sharded_trace_argument_checks():
    import paper_2501_04194_b200 as P
    from paper_2501_04194_b200.distributed import sharded_trace
    f = P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 3))
    with pytest.raises(ValueError, match="cannot be sharded"):
        sharded_trace(f, {"x": torch.zeros(16)}, P.SemanticsConfig(), rank=0, world=2)
    with pytest.raises(ValueError, match="batch size"):
        sharded_trace(f, {"x": torch.zeros(4, 16), "y": torch.zeros(3, 16)}, P.SemanticsConfig(),
                      rank=0, world=2)
