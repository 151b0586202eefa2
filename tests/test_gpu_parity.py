"""Device path (libstlg.so via the public API) against the reference and the oracle.

Tolerances (BASELINE.json north star):
  * hard mode: trace bit-exact against float32(reference), including signed
    zeros; gradients exact for the ones cotangent (they are small integers),
    1e-6 relative otherwise (fp32 sums of fp32 cotangents);
  * smooth modes (LSE / softmax): |gpu - ref| / max(1, |ref|) <= 1e-5 for the
    trace and every gradient (the reference's own FD convention,
    autodiff.py:126).
"""

import numpy as np
import pytest

import golden_io
import stl_oracle
from devhelp import assert_hard_equal, device_supports, rel_err, run_device

import paper_2501_04194_b200 as P

pytestmark = pytest.mark.gpu

SMOOTH_TOL = 1e-5
CASES = [c for c in golden_io.load_all()]


def _check(case_mode, tr, g, ref_tr, ref_g, cot, dabc=None, ref_dabc=None, exact=True):
    """exact=False: hard mode over a NormPred (fp32 sqrt) is compared under the smooth tolerance."""
    if case_mode == "Hard" and exact:
        assert_hard_equal(tr, np.asarray(ref_tr).astype(np.float32))
        ones = np.all(np.asarray(cot) == 1.0)
        for k in ref_g:
            if ones:
                np.testing.assert_array_equal(g[k], ref_g[k])
            else:
                assert rel_err(g[k], ref_g[k]) <= 1e-6, k
    else:
        assert rel_err(tr, ref_tr) <= SMOOTH_TOL
        for k in ref_g:
            assert rel_err(g[k], ref_g[k]) <= SMOOTH_TOL, (k, rel_err(g[k], ref_g[k]))
    if ref_dabc is not None:
        assert rel_err(dabc, ref_dabc) <= SMOOTH_TOL, (dabc, ref_dabc)


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_golden_reference_vectors(cuda, case):
    if not device_supports(case.formula, case.cfg):
        pytest.skip("operator not on the device path in this build")
    binding = (case.si.a, case.si.b, case.si.c) if case.dabc is not None else None
    tr, g, dabc = run_device(case.formula, case.arrays, case.cfg, case.cot, binding)
    from devhelp import has_op
    _check(case.mode, tr, g, case.trace, case.grads, case.cot, dabc, case.dabc,
           exact=not has_op(case.formula, ("NormPred",)))


# --- random corpus at moderate sizes against the oracle --------------------------

def _rand_formula(rng, depth, chans=("x", "y"), until_ok=True, max_a=40, max_w=120):
    ops = ["pred", "not", "and", "or", "F", "G"] + (["U"] if until_ok else [])
    w = np.array([0.3, 0.08, 0.12, 0.12, 0.14, 0.14] + ([0.1] if until_ok else []))
    op = "pred" if depth == 0 else rng.choice(ops, p=w / w.sum())

    def iv():
        if rng.random() < 0.3:
            return None
        a = int(rng.integers(0, max_a))
        return P.StepInterval(a, a + int(rng.integers(0, max_w)))
    if op == "pred":
        if rng.random() < 0.05:
            return P.TRUE
        return P.Pred(str(rng.choice(chans)), str(rng.choice([">", "<"])),
                      float(np.float32(rng.normal(0, 1))))
    if op == "not":
        return P.Not(_rand_formula(rng, depth - 1, chans, until_ok, max_a, max_w))
    if op in ("and", "or"):
        cls = P.And if op == "and" else P.Or
        return cls(_rand_formula(rng, depth - 1, chans, until_ok, max_a, max_w),
                   _rand_formula(rng, depth - 1, chans, until_ok, max_a, max_w))
    if op in ("F", "G"):
        cls = P.Eventually if op == "F" else P.Always
        return cls(_rand_formula(rng, depth - 1, chans, until_ok, max_a, max_w), iv())
    return P.Until(_rand_formula(rng, depth - 1, chans, until_ok, max_a, max_w),
                   _rand_formula(rng, depth - 1, chans, until_ok, max_a, max_w), iv())


MODES = [P.Hard(), P.LogSumExp(1.0), P.LogSumExp(10.0), P.SoftMax(3.0)]


@pytest.mark.parametrize("seed", range(24))
def test_random_formulas_vs_oracle(cuda, seed):
    rng = np.random.default_rng(1000 + seed)
    mode = MODES[seed % len(MODES)]
    pad = P.PaddingPolicy.last_value() if seed % 3 else P.PaddingPolicy.constant(-0.75)
    cfg = P.SemanticsConfig(mode=mode, padding=pad, top_value=100.0)
    f = _rand_formula(rng, int(rng.integers(1, 4)))
    if not device_supports(f, cfg):
        pytest.skip("operator not on the device path in this build")
    B, L = 3, int(rng.integers(20, 400))
    arrays = {c: np.asarray(rng.normal(0, 1.5, (B, L)), dtype=np.float32).astype(np.float64)
              for c in ("x", "y")}
    cot = np.ones((B, L)) if seed % 2 == 0 else \
        np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, arrays, cfg, cot)
    tr, g, _ = run_device(f, arrays, cfg, cot)
    _check(type(mode).__name__, tr, {k: g[k] for k in ref_g}, ref_tr, ref_g, cot)


@pytest.mark.parametrize("seed", range(16))
def test_independent_operands_vs_oracle(cuda, seed):
    """Root And / Or over operands on disjoint channels: the executor deals them to two
    streams with per-lane scratch (exec.cu assign_lanes); same results as the oracle."""
    rng = np.random.default_rng(7000 + seed)
    mode = MODES[seed % len(MODES)]
    cfg = P.SemanticsConfig(mode=mode, top_value=100.0)
    ops = [P.Eventually(_rand_formula(rng, 1, chans=("x",)), P.StepInterval(int(rng.integers(0, 5)), int(rng.integers(6, 60)))),
           _rand_formula(rng, 2, chans=("y", "z")),
           P.Always(_rand_formula(rng, 1, chans=("w",)))]
    f = P.And(ops[0], ops[1]) if seed % 2 else P.Or(ops[0], ops[1])
    if seed % 3 == 0:
        f = P.And(f, ops[2]) if seed % 2 else P.Or(ops[2], f)
    if not device_supports(f, cfg):
        pytest.skip("operator not on the device path in this build")
    B, L = 3, int(rng.integers(60, 400))
    arrays = {c: np.asarray(rng.normal(0, 1.5, (B, L)), dtype=np.float32).astype(np.float64)
              for c in ("x", "y", "z", "w")}
    arrays = {c: arrays[c] for c in sorted(P.variables(f))}
    cot = np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
    ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, arrays, cfg, cot)
    tr, g, _ = run_device(f, arrays, cfg, cot)
    _check(type(mode).__name__, tr, {k: g[k] for k in ref_g}, ref_tr, ref_g, cot)


# --- headline shapes: full size on device, rows sampled for the oracle ----------------

def _walk(B, T, seed):
    rng = np.random.default_rng(seed)
    p0 = rng.uniform(-1, 1, (B, 1, 2))
    p = p0 + np.cumsum(0.05 * rng.normal(0, 1, (B, T, 2)), axis=1)
    return np.asarray(p, dtype=np.float32)


@pytest.mark.parametrize("mode", [P.LogSumExp(10.0), P.Hard(), P.SoftMax(10.0)])
def test_c2_full_size_rows_vs_oracle(cuda, mode):
    import torch
    B, T = 1024, 10_000
    p = _walk(B, T, 1)
    f = P.Eventually(P.NormPred(("px", "py"), "<", 0.5), P.StepInterval(10, 100))
    cfg = P.SemanticsConfig(mode=mode)
    dev = torch.device("cuda", 0)
    pt = torch.tensor(p, device=dev)
    px = pt[..., 0].clone().requires_grad_(True)
    py = pt[..., 1].clone().requires_grad_(True)
    out = P.trace(f, {"px": px, "py": py}, cfg)
    out.backward(torch.ones_like(out))
    tol = SMOOTH_TOL  # softmax included: its window kernels run in fp64 (csrc/fg_soft64.cu)
    rows = [0, 517, 1023]
    for r in rows:
        arrays = {"px": p[r:r + 1, :, 0].astype(np.float64), "py": p[r:r + 1, :, 1].astype(np.float64)}
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, arrays, cfg)
        tr = out[r:r + 1].detach().double().cpu().numpy()
        assert rel_err(tr, ref_tr) <= SMOOTH_TOL
        assert rel_err(px.grad[r:r + 1].double().cpu().numpy(), ref_g["px"]) <= tol
        assert rel_err(py.grad[r:r + 1].double().cpu().numpy(), ref_g["py"]) <= tol


def test_hard_window_full_size_bit_exact(cuda):
    import torch
    B, T = 1024, 10_000
    rng = np.random.default_rng(5)
    x = np.asarray(rng.normal(0, 1, (B, T)), dtype=np.float32)
    f = P.Eventually(P.Pred("x", ">", 0.5), P.StepInterval(10, 100))
    xt = torch.tensor(x, device="cuda").requires_grad_(True)
    out = P.trace(f, {"x": xt}, P.SemanticsConfig())
    out.backward(torch.ones_like(out))
    for r in (0, 333, 1023):
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": x[r:r + 1].astype(np.float64)},
                                                     P.SemanticsConfig())
        assert_hard_equal(out[r:r + 1].detach().cpu().numpy(), ref_tr.astype(np.float32))
        np.testing.assert_array_equal(xt.grad[r:r + 1].cpu().numpy(), ref_g["x"])
    # size-independent property: the ones-cotangent gradient of a hard window
    # sums to the number of outputs per row (each output routes one unit)
    assert torch.all(xt.grad.sum(dim=1) == T)


def test_duality_exact_on_device(cuda):
    """G(phi) == -F(~phi) bit for bit (test_masking.py:255-268), full-size batch."""
    import torch
    rng = np.random.default_rng(7)
    x = torch.tensor(np.asarray(rng.normal(0, 1, (256, 4000)), dtype=np.float32), device="cuda")
    for mode in (P.Hard(), P.LogSumExp(4.0)):
        cfg = P.SemanticsConfig(mode=mode)
        for iv in (P.StepInterval(3, 40), None):
            a = P.trace(P.Always(P.Pred("x", ">", 0.2), iv), {"x": x}, cfg)
            b = P.trace(P.Eventually(P.Not(P.Pred("x", ">", 0.2)), iv), {"x": x}, cfg)
            assert torch.equal(a, -b)


# --- smooth intervals -----------------------------------------

def _step_dataset(seed, n, length, truth=(0.23, 0.59), noise=0.05):
    """Noisy step signals as apps.synth_step_dataset (apps.py:252-269)."""
    import math
    rng = np.random.default_rng(seed)
    lo, hi = int(math.ceil(truth[0] * length)), int(math.floor(truth[1] * length))
    data = np.zeros((n, length))
    for r in range(n):
        jlo = lo + int(rng.integers(-1, 2))
        jhi = hi + int(rng.integers(-1, 2))
        data[r, max(jlo, 0):min(jhi, length - 1) + 1] = 1.0
    data += rng.normal(0.0, noise, (n, length))
    return np.asarray(data, dtype=np.float32)


@pytest.mark.parametrize("mode", [P.Hard(), P.LogSumExp(5.0), P.SoftMax(2.0)])
@pytest.mark.parametrize("pad", [P.PaddingPolicy.last_value(), P.PaddingPolicy.constant(-0.25)])
def test_smooth_interval_vs_oracle(cuda, mode, pad):
    rng = np.random.default_rng(77)
    B, L = 5, 300
    x = np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
    y = np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f = P.And(P.Always(P.Pred("x", ">", 0.0), si), P.Eventually(P.Pred("y", ">", -0.5), si))
    cfg = P.SemanticsConfig(mode=mode, padding=pad)
    binding = (si.a, si.b, si.c)
    ref_tr, ref_g, ref_abc = stl_oracle.trace_and_grad(f, {"x": x, "y": y}, cfg,
                                                       smooth_binding=binding)
    tr, g, dabc = run_device(f, {"x": x, "y": y}, cfg, None, binding)
    _check(type(mode).__name__, tr, g, ref_tr, ref_g, np.ones_like(tr), dabc,
           None if type(mode).__name__ == "Hard" else np.array(ref_abc))
    if type(mode).__name__ == "Hard":
        assert np.all(dabc == 0.0)


def test_c4_full_size(cuda):
    """C4: G_smooth(0.3, 0.65, c=9)(x > 0), LSE(5), B=4096, T=2000; rows vs oracle and
    d(a,b,c) additivity over batch shards (the quantity the multi-GPU path all-reduces)."""
    import torch
    B, T = 4096, 2000
    data = _step_dataset(3, B, T)
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f = P.Always(P.Pred("x", ">", 0.0), si)
    cfg = P.SemanticsConfig(mode=P.LogSumExp(5.0))
    dev = torch.device("cuda", 0)

    def run(rows):
        xt = torch.tensor(data[rows], device=dev).requires_grad_(True)
        abc = tuple(torch.tensor(v, dtype=torch.float64, device=dev, requires_grad=True)
                    for v in (si.a, si.b, si.c))
        out = P.trace(f, {"x": xt}, cfg, smooth_binding=abc)
        gs = torch.autograd.grad(out, [xt, *abc], torch.ones_like(out))
        return out.detach(), gs[0], np.array([float(v) for v in gs[1:]])

    out, gx, dabc = run(slice(0, B))
    for r in (0, 2047, 4095):
        ref_tr, ref_g, _ = stl_oracle.trace_and_grad(f, {"x": data[r:r + 1].astype(np.float64)}, cfg,
                                                     smooth_binding=(si.a, si.b, si.c))
        assert rel_err(out[r:r + 1].double().cpu().numpy(), ref_tr) <= SMOOTH_TOL
        assert rel_err(gx[r:r + 1].double().cpu().numpy(), ref_g["x"]) <= SMOOTH_TOL
    _, _, d1 = run(slice(0, B // 2))
    _, _, d2 = run(slice(B // 2, B))
    assert rel_err(d1 + d2, dabc) <= 1e-6
    # small-batch d(a,b,c) against the oracle
    ref_tr, ref_g, ref_abc = stl_oracle.trace_and_grad(f, {"x": data[:4].astype(np.float64)}, cfg,
                                                       smooth_binding=(si.a, si.b, si.c))
    _, _, d4 = run(slice(0, 4))
    assert rel_err(d4, np.array(ref_abc)) <= SMOOTH_TOL


def test_batch_beyond_one_launch_grid(cuda):
    """B > 65535 rows (the kernels' grid.y limit): the API splits the batch into row
    chunks; every row must equal the same row computed in a small batch."""
    import torch
    import paper_2501_04194_b200 as P
    B, T = 65535 + 7, 64
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(B, T, device="cuda", generator=g)
    f = P.Eventually(P.Pred("x", ">", 0.5), P.StepInterval(2, 9))
    cfg = P.SemanticsConfig(mode=P.LogSumExp(3.0))
    xt = x.clone().requires_grad_(True)
    out = P.trace(f, {"x": xt}, cfg)
    (gx,) = torch.autograd.grad(out, [xt], torch.ones_like(out))
    rows = [0, 65534, 65535, B - 1]
    xs = x[rows].clone().requires_grad_(True)
    out_s = P.trace(f, {"x": xs}, cfg)
    (gs,) = torch.autograd.grad(out_s, [xs], torch.ones_like(out_s))
    assert torch.equal(out[rows], out_s)
    assert torch.equal(gx[rows], gs)


@pytest.mark.parametrize("pad", [P.PaddingPolicy.last_value(), P.PaddingPolicy.constant(0.75)],
                         ids=["last", "const"])
@pytest.mark.parametrize("zero_frac", [0.0, 0.5, 0.995])
@pytest.mark.parametrize("mode", [P.LogSumExp(5.0), P.SoftMax(2.0)])
def test_smooth_interval_cotangent_density(cuda, mode, zero_frac, pad):
    """Smooth-interval VJP with dense, half-sparse and nearly one-hot cotangents: the
    backward kernels switch per staged tile between a branch-free dense loop and the
    zero-skipping loop (csrc/smooth.cu); both must match the oracle (masking.py:207-215).
    'last' padding exercises the closed-form pad tail (k_smooth_bwd_pad), constant
    padding the dropped virtual pad positions (masking.py:94-148)."""
    rng = np.random.default_rng(1234)
    B, L = 4, 1500
    if type(mode).__name__ == "LogSumExp":  # random walks, |x| up to ~10
        x = np.cumsum(np.asarray(rng.normal(0, 0.3, (B, L)), dtype=np.float32), axis=1).astype(np.float64)
    else:  # softmax: iid N(0,1)
        x = np.asarray(rng.normal(0, 1, (B, L)), dtype=np.float32).astype(np.float64)
    si = P.SmoothInterval(0.2, 0.6, 9.0)
    f = P.Always(P.Pred("x", ">", 0.0), si)
    cfg = P.SemanticsConfig(mode=mode, padding=pad)
    # positive weights: the child gradient is then a sum of same-sign terms, so the
    # elementwise tolerance measures the kernel, not fp32 cancellation over ~600 terms
    cot = rng.uniform(0.25, 1.75, (B, L))
    cot[rng.random((B, L)) < zero_frac] = 0.0
    cot = np.asarray(cot, dtype=np.float32).astype(np.float64)
    binding = (si.a, si.b, si.c)
    ref_tr, ref_g, ref_abc = stl_oracle.trace_and_grad(f, {"x": x}, cfg, cotangent=cot,
                                                       smooth_binding=binding)
    tr, g, dabc = run_device(f, {"x": x}, cfg, cot, binding)
    # softmax d_b is ~1e2 out of summands up to ~3e4 (dw/db peaks at c L / 4 = 3375): its
    # d/dw terms run in fp64 against the forward's double-float M and L (csrc/smooth.cu)
    _check(type(mode).__name__, tr, g, ref_tr, ref_g, cot, dabc, np.array(ref_abc))


def test_smooth_interval_graph_capture(cuda):
    """smooth-interval forward + backward (weight table built on the device, no
    host copies) capture into one CUDA graph and replay to the eager results."""
    import ctypes
    import torch
    from paper_2501_04194_b200.engine import compile_formula
    B, T = 64, 700
    x = torch.tensor(np.asarray(P.synth_step_dataset(3, B, T), dtype=np.float32), device="cuda")
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    comp = compile_formula(P.Always(P.Pred("x", ">", 0.0), si), ["x"], P.SemanticsConfig(mode=P.LogSumExp(5.0)))
    params = comp.smooth_params()
    fb, bb = comp.workspace_bytes(B, T)
    fws = torch.empty(fb, dtype=torch.uint8, device="cuda")
    bws = torch.empty(bb, dtype=torch.uint8, device="cuda")
    ones = torch.ones(B, T, device="cuda")

    def run(out, dx, dabc):
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        comp.forward([x], params, out, fws, st)
        dabc.zero_()
        comp.backward([x], params, out, ones, [dx], dabc, fws, bws, st)

    eager = [torch.empty(B, T, device="cuda"), torch.empty(B, T, device="cuda"),
             torch.zeros(3, dtype=torch.float64, device="cuda")]
    run(*eager)
    torch.cuda.synchronize()
    cap = [torch.empty(B, T, device="cuda"), torch.empty(B, T, device="cuda"),
           torch.zeros(3, dtype=torch.float64, device="cuda")]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run(*cap)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    for t in cap:
        t.zero_()
    with torch.cuda.graph(g):
        run(*cap)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, cap):
        assert torch.equal(a, b)


@pytest.mark.parametrize("mode", [P.Hard(), P.LogSumExp(5.0)], ids=["hard", "lse5"])
def test_two_lane_plan_graph_capture(cuda, mode):
    """Independent operands run on a library side stream forked from / joined into the
    caller's stream (exec.cu): inside a CUDA graph they become parallel branches.  Eager and
    captured forward + backward (random cotangent) give the same bits, and the captured
    graph replays correctly after the inputs change."""
    import ctypes
    import torch
    from paper_2501_04194_b200.engine import compile_formula
    B, T = 48, 3000
    f = P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 60))),
              P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0), P.StepInterval(0, 90)))
    comp = compile_formula(f, ["x", "y", "z"], P.SemanticsConfig(mode=mode))
    gen = torch.Generator(device="cuda").manual_seed(21)
    ch = [torch.round(torch.randn(B, T, device="cuda", generator=gen) * 2) for _ in range(3)]
    cot = torch.randn(B, T, device="cuda", generator=gen)
    fb, bb = comp.workspace_bytes(B, T)
    fws = torch.empty(fb, dtype=torch.uint8, device="cuda")
    bws = torch.empty(bb, dtype=torch.uint8, device="cuda")

    def run(out, d):
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        comp.forward(ch, [], out, fws, st)
        comp.backward(ch, [], out, cot, d, None, fws, bws, st)

    def fresh():
        return torch.empty(B, T, device="cuda"), [torch.empty(B, T, device="cuda") for _ in range(3)]

    eager = fresh()
    run(*eager)
    torch.cuda.synchronize()
    cap = fresh()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run(*cap)  # warm-up on the capture stream (creates the side stream outside capture)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    cap[0].zero_()
    for t in cap[1]:
        t.zero_()
    with torch.cuda.graph(g):
        run(*cap)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(eager[0], cap[0])
    for a, b in zip(eager[1], cap[1]):
        assert torch.equal(a, b)
    # new inputs in place: the replay follows them, as a fresh eager run does
    for c in ch:
        c.copy_(torch.round(torch.randn(B, T, device="cuda", generator=gen) * 2))
    g.replay()
    ref = fresh()
    run(*ref)
    torch.cuda.synchronize()
    assert torch.equal(ref[0], cap[0])
    for a, b in zip(ref[1], cap[1]):
        assert torch.equal(a, b)
