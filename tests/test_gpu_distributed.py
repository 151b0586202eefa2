"""The multi-GPU path with the product kernels: two ranks, each running
``sharded_trace`` (libstlg.so) on its row block, then ``allreduce_interval_grads``.

Only one GPU is available, so both ranks run on cuda:0 over the gloo backend (CUDA
tensors); the ranks' kernels never wait on each other — the only interaction is the
host-side all-reduce — so this exercises the same code the NCCL path runs.  The
gathered traces / signal gradients must equal the single-process full batch row for
row (bitwise: rows are independent), and d(a, b, c) must equal the full-batch value.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

B, T = 96, 600


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    import paper_2501_04194_b200 as P
    x = np.asarray(P.synth_step_dataset(3, B, T), dtype=np.float32)
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f = P.Always(P.Pred("x", ">", 0.0), si)
    return P, x, si, f, P.SemanticsConfig(mode=P.LogSumExp(5.0))


def _step(P, xt, si, f, cfg, **kw):
    import torch
    from paper_2501_04194_b200.distributed import allreduce_interval_grads, sharded_trace
    abc = [torch.tensor(v, dtype=torch.float64, device=xt.device, requires_grad=True)
           for v in (si.a, si.b, si.c)]
    xt = xt.clone().requires_grad_(True)
    out, sl = sharded_trace(f, {"x": xt}, cfg, smooth_binding=tuple(abc), **kw)
    out.backward(torch.ones_like(out))
    allreduce_interval_grads(abc)
    return out.detach().cpu().numpy(), xt.grad, sl, [float(a.grad) for a in abc]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, x, si, f, cfg = _problem()
    xt = torch.tensor(x, device="cuda")
    out, gx, sl, dabc = _step(P, xt, si, f, cfg)
    gx = gx[sl].cpu().numpy()
    q.put((rank, sl.start, sl.stop, out, gx, dabc))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_step_matches_single_process(cuda):
    import torch
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p_ in procs:
        p_.join(timeout=120)
        assert p_.exitcode == 0
    P, x, si, f, cfg = _problem()
    out, gx, _, dabc = _step(P, torch.tensor(x, device="cuda"), si, f, cfg, rank=0, world=1)
    gx = gx.cpu().numpy()
    for rank, lo, hi, o, g, d in res:
        assert np.array_equal(o, out[lo:hi])
        assert np.array_equal(g, gx[lo:hi])
        np.testing.assert_allclose(d, dabc, rtol=1e-9, atol=0)
    assert res[0][2] == res[1][1] and res[0][1] == 0 and res[1][2] == B
