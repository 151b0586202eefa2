"""Benchmark: signal-timesteps/s, forward + backward (robustness trace + gradients).

Headline workload (BASELINE.json configs[1]): Eventually[10,100](||p - g|| < 0.5),
LogSumExp(temp=10), p = fp32 2-D random walks, B = 1024 signals x T = 10,000 samples
per GPU.  One step = the full robustness trace [B, T] (masking.trace_var semantics)
plus the VJP of that trace with the ones cotangent (tape.backward default) into
d p (both channels).  `value` = B*T*N / step time with inputs resident in HBM;
`e2e` = the same through the public API with pinned-host inputs copied in and the
trace + gradients copied out every step.

Side legs in the same JSON line: `hard_c1` (C1's formula at C2 scale, HBM-bound),
`c3` (BASELINE configs[2] at B=256, T=4000, Hard and LSE(10)), `c4` (configs[3]: the
smooth-interval Always with gradients to x and (a, b, c), B=4096, T=2000, batch-sharded
over the N ranks with the NCCL fp64 all-reduce of d(a,b,c) inside every timed step,
weak and strong scaling), and the paper's 90k-interval sweep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU: one process per GPU.  Under torchrun the rank comes from the environment;
`--gpus N` (N > 1) without a torchrun environment re-launches itself under
`torch.distributed.run` on 127.0.0.1.  C2 is weak scaling (B rows per GPU, no
data-path collective); time = max over ranks.
`--impl reference` times the reference's own CPU implementation (`stlmask` from
baseline/_ref: masking.trace_var + tape.backward) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "signal-timesteps/sec fwd+bwd (robustness+grads) at T=10k; % HBM/SFU roofline"
UNIT = "signal-timesteps/s"
B_PER_GPU, T_LEN = 1024, 10_000
WINDOW = (10, 100)
TEMP = 10.0
RADIUS = 0.5
C4_B, C4_T = 4096, 2000
NOMINAL_CLK_MHZ = 1965.0
SMS = 148


def _config(n):
    return {"workload": "C2: F[10,100](||p-g||<0.5) LSE(temp=10), 2-D random walks",
            "global_batch": B_PER_GPU * n, "seq_len": T_LEN, "channels": 2,
            "parallelism": f"batch-shard dp{n}" if n > 1 else "single",
            "cotangent": "ones (full-trace VJP)",
            "l2": "rotating 3 input/output sets (3 x 205 MB > 126 MB L2)",
            "timing": "CUDA events around K replays of one CUDA graph per step (fwd + bwd launches); the fwd / bwd split from per-phase graph replays"}


def _walk(B, T, seed):
    import numpy as np
    rng = np.random.default_rng(seed)
    p0 = rng.uniform(-1, 1, (B, 1, 2))
    return np.asarray(p0 + np.cumsum(0.05 * rng.normal(0, 1, (B, T, 2)), axis=1), dtype=np.float32)


def _formula(P):
    return P.Eventually(P.NormPred(("px", "py"), "<", RADIUS, (0.0, 0.0)),
                        P.StepInterval(*WINDOW))


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # the first sample lands before the timed region ends
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs: the reference itself (stlmask from baseline/_ref) and the oracle port
# ---------------------------------------------------------------------------
def _import_reference():
    """The unmodified reference package (pip-installed into baseline/_ref), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(path, "stlmask")) and path not in sys.path:
        sys.path.append(path)
    try:
        import stlmask  # noqa: F401
        from stlmask import masking, tape  # noqa: F401
        return sys.modules["stlmask"]
    except Exception:
        return None


def _ref_rows(args):
    """C2 on `rows` signals through the reference's public path: trace_var over the
    channels with the distance built on the reference tape as sqrt(dx^2 + dy^2) (the
    reference has no norm predicate; apps.py:150-151 builds it the same way, without
    its +1e-12), then tape.backward with the ones seed (tape.py:114-134)."""
    rows, seed, chunk = args
    import numpy as np
    from stlmask import masking, tape
    from stlmask.core import LogSumExp, SemanticsConfig, StepInterval
    from stlmask.formula import Eventually, Pred
    p = _walk(rows, T_LEN, seed).astype(np.float64)
    f = Eventually(Pred("d", "<", RADIUS), StepInterval(*WINDOW))
    cfg = SemanticsConfig(mode=LogSumExp(TEMP))
    t0 = time.perf_counter()
    for r in range(0, rows, chunk):
        px, py = tape.Var(p[r:r + chunk, :, 0]), tape.Var(p[r:r + chunk, :, 1])
        d = tape.sqrt(tape.square(px) + tape.square(py))
        out = masking.trace_var(f, {"px": px, "py": py, "d": d}, T_LEN, cfg)
        tape.backward(out)
    return time.perf_counter() - t0


def _port_rows(args):
    """The same step through the oracle port (oracle/stl_oracle.py; numpy f64)."""
    rows, seed, chunk = args
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import stl_oracle
    import paper_2501_04194_b200.core as C
    import paper_2501_04194_b200.formula as F
    p = _walk(rows, T_LEN, seed).astype(np.float64)
    f = F.Eventually(F.NormPred(("px", "py"), "<", RADIUS, (0.0, 0.0)), C.StepInterval(*WINDOW))
    cfg = C.SemanticsConfig(mode=C.LogSumExp(TEMP))
    t0 = time.perf_counter()
    for r in range(0, rows, chunk):
        q = p[r:r + chunk]
        stl_oracle.trace_and_grad(f, {"px": q[..., 0], "py": q[..., 1]}, cfg)
    return time.perf_counter() - t0


def cpu_rate(kind, rows_per_proc, procs, chunk=4):
    """signal-timesteps/s of `kind` ('reference' | 'port') over procs x rows_per_proc rows
    (row-parallel processes, chunked so each process holds (chunk, T, K) windows)."""
    fn = _ref_rows if kind == "reference" else _port_rows
    if procs <= 1:
        fn((1, 99, chunk))  # warm-up (imports, allocator)
        t0 = time.perf_counter()
        fn((rows_per_proc, 1, chunk))
        dt = time.perf_counter() - t0
        return rows_per_proc * T_LEN / dt, dt
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(fn, [(1, 99, chunk)] * procs)
        t0 = time.perf_counter()
        pool.map(fn, [(rows_per_proc, i, chunk) for i in range(procs)])
        dt = time.perf_counter() - t0
    return rows_per_proc * procs * T_LEN / dt, dt


def _host_info():
    info = {"cores": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                info["cpu"] = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return info


def run_reference(args, rank, world):
    if rank != 0:
        return
    host = _host_info()
    cores = host["cores"]
    kind = "reference" if _import_reference() is not None else "port"
    rows_per_proc = 4
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.warmup):
        cpu_rate(kind, 1, cores)
    for _ in range(args.steps):
        v, _ = cpu_rate(kind, rows_per_proc, cores)
        vals.append(v)
    value = statistics.median(vals)
    sample = (f"{rows_per_proc * cores} rows x T={T_LEN} per step (of B={B_PER_GPU} per GPU), "
              f"row-parallel over {cores} processes, 4-row chunks; per-step time extrapolated "
              f"linearly to the full batch")
    src = ("stlmask 0.1.0 from baseline/_ref (masking.trace_var + tape.backward, unmodified)"
           if kind == "reference" else "oracle/stl_oracle.py port (baseline/_ref missing)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": B_PER_GPU * world * T_LEN / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample, "source": src, "host": host},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device legs
# ---------------------------------------------------------------------------
def _graph_timed(steps, warmup, sets, fwd, bwd, stream, flush=None):
    """CUDA graphs per (set, phase) and per (set, whole step), replayed round-robin; returns
    per-step (fwd_ms, bwd_ms) from the phase graphs and step_ms from the whole-step graphs."""
    import torch
    for i in range(max(warmup, 3)):
        fwd(i % len(sets))
        bwd(i % len(sets))
    torch.cuda.synchronize()
    graphs = []
    for s in range(len(sets)):
        gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf):
            fwd(s)
        with torch.cuda.graph(gb):
            bwd(s)
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            fwd(s)
            bwd(s)
        graphs.append((gf, gb, g1))
    for i in range(max(warmup, 3)):
        for g in graphs[i % len(sets)]:
            g.replay()
    torch.cuda.synchronize()
    es = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush()
        es[i][0].record(stream)
        graphs[i % len(sets)][2].replay()
        es[i][1].record(stream)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush()
        ev[i][0].record(stream)
        graphs[i % len(sets)][0].replay()
        ev[i][1].record(stream)
        graphs[i % len(sets)][1].replay()
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    return ([e[0].elapsed_time(e[1]) for e in ev], [e[1].elapsed_time(e[2]) for e in ev],
            [e[0].elapsed_time(e[1]) for e in es])


def _hard_c1(P, compile_formula, dev, B, T, args, cur_stream):
    """C1's formula Always[0,50](x > 0.5) (Hard, last pad) on a contiguous 1-D fp32
    N(0,1) signal at B x T: fwd + ones-cotangent bwd through CUDA graphs over 3
    rotating sets (3 x 123 MB > L2).  Algorithmic bytes 16 B / unit."""
    import torch
    f = P.Always(P.Pred("x", ">", 0.5), P.StepInterval(0, 50))
    comp = compile_formula(f, ["x"], P.SemanticsConfig(mode=P.Hard()))
    g = torch.Generator(device=dev).manual_seed(0)
    sets = [{"x": torch.randn(B, T, device=dev, generator=g), "out": torch.empty(B, T, device=dev),
             "dx": torch.empty(B, T, device=dev)} for _ in range(3)]
    fb, bb = comp.workspace_bytes(B, T)
    fws = torch.empty(max(fb, 1), dtype=torch.uint8, device=dev)
    bws = torch.empty(max(bb, 1), dtype=torch.uint8, device=dev)
    ones = torch.ones(B, T, device=dev)

    def fwd(s):
        comp.forward([sets[s]["x"]], [], sets[s]["out"], fws, cur_stream())

    def bwd(s):
        comp.backward([sets[s]["x"]], [], sets[s]["out"], ones, [sets[s]["dx"]], None, fws, bws, cur_stream())
    fw, bw, sw = _graph_timed(args.steps, args.warmup, sets, fwd, bwd, torch.cuda.current_stream())
    fwd_ms, bwd_ms, ms = statistics.mean(fw), statistics.mean(bw), statistics.mean(sw)
    return {"formula": "Always[0,50](x > 0.5), Hard, 1-D N(0,1)", "global_batch": B, "seq_len": T,
            "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "ms_per_step": ms, "value": B * T / (ms / 1e3), "unit": UNIT,
            "alg_bytes_per_unit": 16}


def _c3(P, compile_formula, dev, args, cur_stream, hbm):
    """BASELINE configs[2] / SURVEY §8(d) C3: G(F[0,200](x > 0)) & ((y < 1) U (z > 0)) with
    untimed G and U, x, y, z ~ N(0,1), B=256, T=4000; Hard and LSE(10)."""
    import torch
    B, T = 256, 4000
    f = P.And(P.Always(P.Eventually(P.Pred("x", ">", 0.0), P.StepInterval(0, 200))),
              P.Until(P.Pred("y", "<", 1.0), P.Pred("z", ">", 0.0)))
    g = torch.Generator(device=dev).manual_seed(2)
    res = {"formula": "G(F[0,200](x>0)) & ((y<1) U (z>0)), untimed G / U", "global_batch": B, "seq_len": T,
           "l2": "inputs 12 MB fit in L2 (reported as is; the LSE path is compute-bound)"}
    for name, mode in (("hard", P.Hard()), ("lse10", P.LogSumExp(10.0))):
        comp = compile_formula(f, ["x", "y", "z"], P.SemanticsConfig(mode=mode))
        sets = []
        for _ in range(2):
            sets.append({"ch": [torch.randn(B, T, device=dev, generator=g) for _ in range(3)],
                         "out": torch.empty(B, T, device=dev),
                         "d": [torch.empty(B, T, device=dev) for _ in range(3)]})
        fb, bb = comp.workspace_bytes(B, T)
        fws = torch.empty(max(fb, 1), dtype=torch.uint8, device=dev)
        bws = torch.empty(max(bb, 1), dtype=torch.uint8, device=dev)
        ones = torch.ones(B, T, device=dev)

        def fwd(s, comp=comp, sets=sets, fws=fws):
            comp.forward(sets[s]["ch"], [], sets[s]["out"], fws, cur_stream())

        def bwd(s, comp=comp, sets=sets, fws=fws, bws=bws, ones=ones):
            comp.backward(sets[s]["ch"], [], sets[s]["out"], ones, sets[s]["d"], None, fws, bws, cur_stream())
        steps = args.steps if name == "hard" else max(3, min(args.steps, 5))
        fw, bw, sw = _graph_timed(steps, min(args.warmup, 3), sets, fwd, bwd, torch.cuda.current_stream())
        ms = statistics.mean(sw)
        entry = {"fwd_ms": statistics.mean(fw), "bwd_ms": statistics.mean(bw), "ms_per_step": ms,
                 "value": B * T / (ms / 1e3), "unit": UNIT}
        if name == "hard":
            # 32 algorithmic bytes per unit (3 channels read, trace write,
            # cotangent read, 3 gradients written -> 4 * (3 + 1 + 1 + 3) = 32)
            entry["roofline"] = {"bound": "hbm", "achieved": 32.0 * B * T / (ms / 1e3) / 1e9, "peak": hbm,
                                 "unit": "GB/s", "frac": 32.0 * B * T / (ms / 1e3) / 1e9 / hbm}
        res[name] = entry
    return res


def _c4_bound(P, B, T, si, clk_mhz):
    """Re-derived C4 bound for the factorised smooth-interval kernels (csrc/smooth.cu): the
    forward, the child backward (real positions; the 'last'-padding tail is closed form) and
    the d/dw pass each do one FMA per kept (t, i) pair; the ex2s are one per staged element
    (O(T) per tile, not per pair).  Returns the bound in ms at clk_mhz."""
    import numpy as np
    from paper_2501_04194_b200.lower import smooth_weights_np
    w = smooth_weights_np(si.a, si.b, si.c, si.eps, T)
    kept = np.flatnonzero(w > 0)
    i_lo, i_hi = int(kept[0]), int(kept[-1])
    K = i_hi - i_lo + 1
    t = np.arange(T)
    real = np.clip(np.minimum(i_hi, T - 1 - t) - i_lo + 1, 0, None).sum()
    fma_pairs = 2.0 * B * T * K + 1.0 * B * real
    fma_peak = SMS * 128 * clk_mhz * 1e6
    return {"kept_offsets": K, "fma_pairs": fma_pairs, "mufu_pairs": 0.0,
            "fma_peak_per_s": fma_peak, "bound_ms": fma_pairs / fma_peak * 1e3}


def _c4(P, compile_formula, dev, args, cur_stream, dist, rank, world):
    """BASELINE configs[3] / SURVEY §8(d) C4: Always(x > 0, SmoothInterval(0.3, 0.65, 9)),
    LSE(5), x = synth_step_dataset(seed=3, n=4096, length=2000) (apps.py:252-269); one step
    = forward + backward (d x and d(a, b, c)) + the fp64 all-reduce of d(a, b, c) over the
    ranks, all inside the timed region.  weak: 4096 rows per GPU (rank r
    uses seed 3 + r); strong: 4096 rows in total, sharded by distributed.shard_rows."""
    import numpy as np
    import torch
    from paper_2501_04194_b200.distributed import shard_rows
    si = P.SmoothInterval(0.3, 0.65, 9.0)
    f = P.Always(P.Pred("x", ">", 0.0), si)
    comp = compile_formula(f, ["x"], P.SemanticsConfig(mode=P.LogSumExp(5.0)))
    params = comp.smooth_params()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"formula": "G_smooth(0.3,0.65,c=9)(x > 0), LSE(5)", "seq_len": C4_T,
           "data": "synth_step_dataset(seed=3 [+rank for weak], n=4096, length=2000) (apps.py:252-269)",
           "l2": "256 MB L2 flush between timed steps (outside the events)",
           "collective": "NCCL all_reduce(sum) of fp64 d(a,b,c) (24 B) per step" if world > 1 else "none (1 rank)"}
    for scaling in ("weak", "strong"):
        if scaling == "weak":
            x_host = P.synth_step_dataset(3 + rank, C4_B, C4_T)
            Bg = C4_B * world
        else:
            sl = shard_rows(C4_B, rank, world)
            x_host = P.synth_step_dataset(3, C4_B, C4_T)[sl]
            Bg = C4_B
        B = x_host.shape[0]
        x = torch.tensor(np.asarray(x_host, dtype=np.float32), device=dev)
        o = torch.empty(B, C4_T, device=dev)
        dx = torch.empty(B, C4_T, device=dev)
        d_abc = torch.zeros(3, dtype=torch.float64, device=dev)
        fb, bb = comp.workspace_bytes(B, C4_T)
        fws = torch.empty(max(fb, 1), dtype=torch.uint8, device=dev)
        bws = torch.empty(max(bb, 1), dtype=torch.uint8, device=dev)
        ones = torch.ones(B, C4_T, device=dev)
        stream = torch.cuda.current_stream()

        def step():
            comp.forward([x], params, o, fws, cur_stream())
            d_abc.zero_()
            comp.backward([x], params, o, ones, [dx], d_abc, fws, bws, cur_stream())
            if dist is not None:
                dist.all_reduce(d_abc, op=dist.ReduceOp.SUM)

        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        steps = max(3, min(args.steps, 10))
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        for i in range(steps):
            flush_buf.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
        if dist is not None:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        bound = _c4_bound(P, B, C4_T, si, NOMINAL_CLK_MHZ)
        out[scaling] = {"global_batch": Bg, "per_gpu_batch": B, "n_gpus": world, "ms_per_step": ms,
                        "value": Bg * C4_T / (ms / 1e3), "unit": UNIT,
                        "d_abc": [float(v) for v in d_abc.cpu()],
                        "roofline": {"bound": "fma (factorised smooth kernels: one FMA per kept pair)",
                                     "bound_ms": bound["bound_ms"], "frac": bound["bound_ms"] / ms,
                                     "kept_offsets": bound["kept_offsets"],
                                     "mufu_pairs": bound["mufu_pairs"], "fma_pairs": bound["fma_pairs"],
                                     "clock_mhz": NOMINAL_CLK_MHZ,
                                     "survey_brute_force_bound_ms": B * C4_T * 4001 / (SMS * 16 * NOMINAL_CLK_MHZ * 1e6) * 1e3}}
    return out


def _interval_sweep(dev, args):
    """The paper's interval sweep: the robustness-based mining
    objective of G_[aT, bT](s > 0) for 90,000 (a, b) pairs in one launch of
    stlg_mining_grid, over one signal of T = 20 and over a 64-row T = 200 dataset."""
    import ctypes
    import torch
    from paper_2501_04194_b200 import _lib
    lib = _lib.load()
    out = {"pairs": 90000, "formula": "G_[aT,bT](s > 0), smooth window c=9, LSE(5)",
           "paper": "1.87 ms for 90,000 pairs at T=20 (JAX+JIT, M2 MacBook Pro)"}
    g = torch.Generator(device=dev).manual_seed(3)
    a = torch.rand(90000, generator=g, device=dev, dtype=torch.float64) * 0.5
    b = a + 0.05 + torch.rand(90000, generator=g, device=dev, dtype=torch.float64) * 0.45
    loss = torch.empty(90000, dtype=torch.float64, device=dev)
    for name, (n, L) in (("T20_n1", (1, 20)), ("T200_n64", (64, 200))):
        x = torch.randn(n, L, generator=g, device=dev) + 0.5
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

        def run():
            _lib.check(lib.stlg_mining_grid(x.data_ptr(), n, L, x.stride(0), a.data_ptr(), b.data_ptr(),
                                            90000, 9.0, 0.0, 2, 5.0, 0.15, loss.data_ptr(), None, stream))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(args.steps, 5)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[name] = {"n": n, "T": L, "ms": ms, "ns_per_interval": ms * 1e6 / 90000}
    return out


def _pcie(dev, nbytes_in, nbytes_out):
    """Measured pinned-host copy bandwidths (the e2e leg's own roofline)."""
    import torch
    h_in = torch.empty(nbytes_in, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nbytes_in, dtype=torch.uint8, device=dev)
    d_out = torch.empty(nbytes_out, dtype=torch.uint8, device=dev)
    h_out = torch.empty(nbytes_out, dtype=torch.uint8).pin_memory()
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}
    for _ in range(2):
        d_in.copy_(h_in, non_blocking=True)
        h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    for name, fn in (("h2d_gbs", lambda: d_in.copy_(h_in, non_blocking=True)),
                     ("d2h_gbs", lambda: h_out.copy_(d_out, non_blocking=True))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        n = nbytes_in if name == "h2d_gbs" else nbytes_out
        res[name] = 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    res["duplex_ms_per_step"] = e0.elapsed_time(e1) / 5
    return res


def run_b200(args, rank, world):
    import ctypes
    import numpy as np
    import torch
    import paper_2501_04194_b200 as P
    from paper_2501_04194_b200 import _lib
    from paper_2501_04194_b200.engine import compile_formula

    local = int(os.environ.get("LOCAL_RANK", 0))
    # BENCH_ONE_DEVICE=1 + BENCH_DIST_BACKEND=gloo: a control-flow check of the N > 1 path on
    # a one-GPU box (all ranks on cuda:0, host-side collectives); its timings mean nothing
    one_dev = os.environ.get("BENCH_ONE_DEVICE") == "1"
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = 0 if one_dev else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    B, T = B_PER_GPU, T_LEN
    f = _formula(P)
    cfg = P.SemanticsConfig(mode=P.LogSumExp(TEMP))
    comp = compile_formula(f, ["px", "py"], cfg)
    lib = _lib.load()
    stream = torch.cuda.current_stream()

    def _cur_stream():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback"
    if dist is not None and backend != "nccl":
        hbm_src += f"; {backend} backend, ranks sharing cuda:{local}: control-flow check only"

    NSET = 3
    host = _walk(B, T, 1 + rank)
    sets = []
    for s in range(NSET):
        p = torch.tensor(np.roll(host, s * 17, axis=1), device=dev)  # [B, T, 2] interleaved
        sets.append({"px": p[..., 0], "py": p[..., 1], "p": p,
                     "out": torch.empty(B, T, device=dev),
                     "dp": torch.zeros(B, T, 2, device=dev)})
    fb, bb = comp.workspace_bytes(B, T)
    fws = torch.empty(fb, dtype=torch.uint8, device=dev)
    bws = torch.empty(bb, dtype=torch.uint8, device=dev)
    ones = torch.ones(B, T, device=dev)
    params = comp.smooth_params()

    def fwd(s):
        d = sets[s]
        comp.forward([d["px"], d["py"]], params, d["out"], fws, _cur_stream())

    def bwd(s):
        d = sets[s]
        comp.backward([d["px"], d["py"]], params, d["out"], ones,
                      [d["dp"][..., 0], d["dp"][..., 1]], None, fws, bws, _cur_stream())

    # stlg kernel launches of one fwd + bwd step (counted once, eagerly)
    lib.stlg_launch_count(1)
    fwd(0)
    bwd(0)
    torch.cuda.synchronize()
    launches_per_step = lib.stlg_launch_count(1)

    for i in range(max(args.warmup, 3)):
        fwd(i % NSET)
        bwd(i % NSET)
    torch.cuda.synchronize()
    # One CUDA graph per (set, phase): replaying them keeps Python / ctypes launch
    # overhead out of the device timeline (the kernels and their order are unchanged).
    graphs = []
    for s in range(NSET):
        gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf):
            fwd(s)
        with torch.cuda.graph(gb):
            bwd(s)
        graphs.append((gf, gb))
    # and one graph per set holding the whole step (fwd + bwd): the timed steps
    steps_g = []
    for s in range(NSET):
        g1 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g1):
            fwd(s)
            bwd(s)
        steps_g.append(g1)
    for i in range(max(args.warmup, 3)):
        graphs[i % NSET][0].replay()
        graphs[i % NSET][1].replay()
        steps_g[i % NSET].replay()
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for i in range(args.steps):
            steps_g[i % NSET].replay()
        stop.record(stream)
        # the fwd / bwd split (roofline of each kernel): the per-phase graphs, events between
        for i in range(args.steps):
            gf, gb = graphs[i % NSET]
            evs[i][0].record(stream)
            gf.replay()
            evs[i][1].record(stream)
            gb.replay()
            evs[i][2].record(stream)
        torch.cuda.synchronize()
        if clk.proc is not None and len(clk.lines) < 3:
            # the timed region is shorter than the sampling period: keep the GPU under the
            # same load (more replays, untimed) until the sampler has seen it
            t_end = time.time() + 0.5
            while time.time() < t_end:
                for s in range(NSET):
                    graphs[s][0].replay()
                    graphs[s][1].replay()
                torch.cuda.synchronize()
    # launches inside the timed region: the graphs replay the captured stlg launches
    launches = launches_per_step * args.steps
    ms = start.elapsed_time(stop)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    bwd_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    ms_step = ms / args.steps
    value = B * T * world / (ms_step / 1e3)

    # ---- side legs ----
    hard = _hard_c1(P, compile_formula, dev, B, T, args, _cur_stream)
    c3 = _c3(P, compile_formula, dev, args, _cur_stream, hbm)
    c4 = _c4(P, compile_formula, dev, args, _cur_stream, dist, rank, world)
    sweep = _interval_sweep(dev, args)

    # ---- e2e through the public API: pinned host -> device -> host ----------
    # Every step: H2D of the step's inputs from pinned memory, P.trace + autograd
    # (the public API), D2H of the trace and both gradients into pinned memory.
    # Standard copy/compute overlap: uploads on one stream, compute on another,
    # downloads on a third (PCIe is full duplex), two buffer slots ordered by events.
    e2e_steps = max(10, min(args.steps, 20))
    hp = [torch.tensor(np.roll(host, 31 * k, axis=1)).pin_memory() for k in range(2)]
    h_out = [{k: torch.empty(B, T).pin_memory() for k in ("tr", "dx", "dy")} for _ in range(2)]
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    d_in = [torch.empty(B, T, 2, device=dev) for _ in range(2)]
    in_free = [torch.cuda.Event() for _ in range(2)]    # compute finished reading slot
    in_ready = [torch.cuda.Event() for _ in range(2)]   # upload finished
    out_ready = [torch.cuda.Event() for _ in range(2)]  # compute finished writing results
    out_free = [torch.cuda.Event() for _ in range(2)]   # download finished (host slot reusable)
    keep = [None, None]

    def e2e_run(nsteps, t0=None, t1=None):
        for i in range(nsteps):
            k = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(in_free[k])
                if i == 0 and t0 is not None:
                    t0.record(s_h2d)
                d_in[k].copy_(hp[k], non_blocking=True)
                in_ready[k].record(s_h2d)
            with torch.cuda.stream(s_cmp):
                s_cmp.wait_event(in_ready[k])
                px = d_in[k][..., 0].detach().requires_grad_(True)
                py = d_in[k][..., 1].detach().requires_grad_(True)
                out = P.trace(f, {"px": px, "py": py}, cfg)
                out.backward(ones)
                in_free[k].record(s_cmp)
                if i >= 2:
                    s_cmp.wait_event(out_free[k])
                res = (out.detach(), px.grad, py.grad)
                out_ready[k].record(s_cmp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(out_ready[k])
                for name, tsr in zip(("tr", "dx", "dy"), res):
                    h_out[k][name].copy_(tsr, non_blocking=True)
                    tsr.record_stream(s_d2h)
                out_free[k].record(s_d2h)
            keep[k] = res
        if t1 is not None:
            t1.record(s_d2h)

    # warm-up: enough pipelined steps that the caching allocator holds every per-step
    # buffer (record_stream defers reuse), so no cudaMalloc lands in the timed region
    e2e_run(6)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_run(e2e_steps, e0, e1)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = B * T * world / (e2e_ms / 1e3)
    # the last step's results reached the host: spot-check them against the device
    assert torch.equal(h_out[(e2e_steps - 1) % 2]["tr"], keep[(e2e_steps - 1) % 2][0].cpu())
    h2d_b, d2h_b = B * T * 2 * 4, B * T * 4 + B * T * 2 * 4
    pcie = _pcie(dev, h2d_b, d2h_b)

    if rank == 0:
        # algorithmic bytes: fwd reads px, py (8 B) and writes the
        # trace (4 B); bwd reads the cotangent (4 B) and writes d px, d py (8 B)
        alg = {"fwd": 12.0 * B * T, "bwd": 12.0 * B * T}
        kern = {"fwd": fwd_ms, "bwd": bwd_ms}
        dom = max(kern, key=kern.get)
        achieved = alg[dom] / (kern[dom] / 1e3) / 1e9
        step_ach = (alg["fwd"] + alg["bwd"]) / ((fwd_ms + bwd_ms) / 1e3) / 1e9
        prof = {}
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        except Exception:
            pass
        traffic = prof.get(dom)
        cores = 1
        cpu_kind = "reference" if _import_reference() is not None else "port"
        cpu_v, cpu_dt = cpu_rate(cpu_kind, 48, cores)
        port_v, port_dt = cpu_rate("port", 48, cores) if cpu_kind == "reference" else (cpu_v, cpu_dt)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": _config(world),
                "roofline": {"bound": "hbm", "kernel": f"stlg {dom} (timed F/G LSE)",
                             "achieved": achieved, "peak": hbm, "unit": "GB/s",
                             "frac": achieved / hbm, "peak_source": hbm_src,
                             "traffic": traffic,
                             "alg_bytes_per_launch": alg[dom],
                             "step_achieved_gbs": step_ach, "step_frac": step_ach / hbm,
                             "fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                             "mufu_per_sample": prof.get("mufu_per_sample"),
                             "ncu_source": prof.get("source")},
                "cpu_baseline": {"value": cpu_v, "unit": UNIT, "cores": cores, "kind": cpu_kind,
                                 "sample": f"48 rows x T={T_LEN} fwd+bwd in 4-row chunks, single process, "
                                           f"{cpu_dt:.1f}s; "
                                           + ("stlmask from baseline/_ref (masking.trace_var + tape.backward)"
                                              if cpu_kind == "reference" else "oracle/stl_oracle.py port"),
                                 "port_value": port_v, "host": _host_info()},
                "e2e": {"value": e2e_val, "unit": UNIT,
                        "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
                        "ms_per_step": e2e_ms, "path": "paper_2501_04194_b200.trace + autograd",
                        "overlap": "H2D / compute / D2H on three streams, 2 buffer slots",
                        "pcie": pcie},
                "gpu_launches": int(launches),
                "hard_c1": dict(hard, roofline_frac=(16.0 * B * T / (hard["ms_per_step"] / 1e3)) / 1e9 / hbm),
                "c3": c3,
                "c4": c4,
                "interval_sweep": sweep,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _spawn(argv, n):
    """Re-launch this script under torch.distributed.run with n ranks on 127.0.0.1."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        sys.exit(_spawn(sys.argv[1:], args.gpus))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.impl == "reference" else 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world)


if __name__ == "__main__":
    main()
