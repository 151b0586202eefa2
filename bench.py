"""Benchmark: signal-timesteps/s, forward + backward (robustness trace + gradients).

Workload (BASELINE.json configs[1]): Eventually[10,100](||p - g|| < 0.5),
LogSumExp(temp=10), p = fp32 2-D random walks, B = 1024 signals x T = 10,000 samples
per GPU.  One step = the full robustness trace [B, T] (masking.trace_var semantics)
plus the VJP of that trace with the ones cotangent (tape.backward default) into
d p (both channels).  `value` = B*T*N / step time with inputs resident in HBM;
`e2e` = the same through the public API with pinned-host inputs copied in and the
trace + gradients copied out every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU (torchrun): every rank runs its own B rows (weak scaling); there is no
data-path collective for this workload; time = max over ranks.
`--impl reference` times the CPU reference path (the oracle port of the
reference algorithm, oracle/stl_oracle.py) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
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


def _config(n):
    return {"workload": "C2: F[10,100](||p-g||<0.5) LSE(temp=10), 2-D random walks",
            "global_batch": B_PER_GPU * n, "seq_len": T_LEN, "channels": 2,
            "parallelism": f"batch-shard dp{n}" if n > 1 else "single",
            "cotangent": "ones (full-trace VJP)",
            "l2": "rotating 3 input/output sets (3 x 205 MB > 126 MB L2)",
            "timing": "CUDA events around CUDA-graph replays of the fwd / bwd launches"}


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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
# CPU baseline (oracle port of the reference algorithm)
# ---------------------------------------------------------------------------
def _cpu_rows(args):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import stl_oracle
    import paper_2501_04194_b200.core as C
    import paper_2501_04194_b200.formula as F
    rows, seed = args
    p = _walk(rows, T_LEN, seed).astype(np.float64)
    f = F.Eventually(F.NormPred(("px", "py"), "<", RADIUS, (0.0, 0.0)), C.StepInterval(*WINDOW))
    cfg = C.SemanticsConfig(mode=C.LogSumExp(TEMP))
    t0 = time.perf_counter()
    for r in range(0, rows, 16):  # 16-row chunks bound the (rows, T, K) window arrays
        q = p[r:r + 16]
        stl_oracle.trace_and_grad(f, {"px": q[..., 0], "py": q[..., 1]}, cfg)
    return time.perf_counter() - t0


def cpu_baseline(rows=8, cores=1):
    """Time the oracle port on `rows` x T signals; returns signal-timesteps/s."""
    if cores <= 1:
        _cpu_rows((2, 99))  # warm-up (imports, allocator)
        t0 = time.perf_counter()
        _cpu_rows((rows, 1))
        dt = time.perf_counter() - t0
        return rows * T_LEN / dt, dt
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(_cpu_rows, [(1, 99)] * cores)
        t0 = time.perf_counter()
        pool.map(_cpu_rows, [(max(rows // cores, 1), i) for i in range(cores)])
        dt = time.perf_counter() - t0
    return max(rows // cores, 1) * cores * T_LEN / dt, dt


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    rows = 2 * cores
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.warmup):
        cpu_baseline(rows=cores, cores=cores)
    for _ in range(args.steps):
        v, _ = cpu_baseline(rows=rows, cores=cores)
        vals.append(v)
    value = statistics.median(vals)
    sample = f"{rows} rows x T={T_LEN} per step (of B={B_PER_GPU}), row-parallel over {cores} processes"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": B_PER_GPU * T_LEN / value * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": _config(world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


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
    graphs = []
    for d in sets:
        comp.forward([d["x"]], [], d["out"], fws, cur_stream())
        comp.backward([d["x"]], [], d["out"], ones, [d["dx"]], None, fws, bws, cur_stream())
    torch.cuda.synchronize()
    for d in sets:
        gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf):
            comp.forward([d["x"]], [], d["out"], fws, cur_stream())
        with torch.cuda.graph(gb):
            comp.backward([d["x"]], [], d["out"], ones, [d["dx"]], None, fws, bws, cur_stream())
        graphs.append((gf, gb))
    for i in range(3):
        graphs[i % 3][0].replay()
        graphs[i % 3][1].replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record(stream)
        graphs[i % 3][0].replay()
        ev[i][1].record(stream)
        graphs[i % 3][1].replay()
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    bwd_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    return {"formula": "Always[0,50](x > 0.5), Hard, 1-D N(0,1)", "global_batch": B, "seq_len": T,
            "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "value": B * T / ((fwd_ms + bwd_ms) / 1e3), "unit": UNIT,
            "alg_bytes_per_unit": 16}


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


def run_b200(args, rank, world):
    import numpy as np
    import torch
    import paper_2501_04194_b200 as P
    from paper_2501_04194_b200 import _lib
    from paper_2501_04194_b200.engine import compile_formula

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    B, T = B_PER_GPU, T_LEN
    f = _formula(P)
    cfg = P.SemanticsConfig(mode=P.LogSumExp(TEMP))
    comp = compile_formula(f, ["px", "py"], cfg)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sptr = __import__("ctypes").c_void_p(stream.cuda_stream)

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

    def _cur_stream():
        return __import__("ctypes").c_void_p(torch.cuda.current_stream().cuda_stream)

    # stlg kernel launches of one fwd + bwd step (counted once, eagerly)
    lib.stlg_launch_count(1)
    comp.forward([sets[0]["px"], sets[0]["py"]], params, sets[0]["out"], fws, _cur_stream())
    comp.backward([sets[0]["px"], sets[0]["py"]], params, sets[0]["out"], ones,
                  [sets[0]["dp"][..., 0], sets[0]["dp"][..., 1]], None, fws, bws, _cur_stream())
    torch.cuda.synchronize()
    launches_per_step = lib.stlg_launch_count(1)

    def fwd(s):
        d = sets[s]
        comp.forward([d["px"], d["py"]], params, d["out"], fws, _cur_stream())

    def bwd(s):
        d = sets[s]
        comp.backward([d["px"], d["py"]], params, d["out"], ones,
                      [d["dp"][..., 0], d["dp"][..., 1]], None, fws, bws, _cur_stream())

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
    for i in range(max(args.warmup, 3)):
        graphs[i % NSET][0].replay()
        graphs[i % NSET][1].replay()
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.stlg_launch_count(1)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record(stream)
        for i in range(args.steps):
            gf, gb = graphs[i % NSET]
            evs[i][0].record(stream)
            gf.replay()
            evs[i][1].record(stream)
            gb.replay()
            evs[i][2].record(stream)
        stop.record(stream)
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

    # ---- hard mode at the same scale (C1's formula, SURVEY §8(d) HBM row) ----
    hard = _hard_c1(P, compile_formula, dev, B, T, args, _cur_stream)
    # ---- interval sweep ----
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

    if rank == 0:
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"
        # algorithmic bytes: fwd reads px, py (8 B) and writes the
        # trace (4 B); bwd reads the cotangent (4 B) and writes d px, d py (8 B)
        alg = {"fwd": 12.0 * B * T, "bwd": 12.0 * B * T}
        kern = {"fwd": fwd_ms, "bwd": bwd_ms}
        dom = max(kern, key=kern.get)
        achieved = alg[dom] / (kern[dom] / 1e3) / 1e9
        step_ach = (alg["fwd"] + alg["bwd"]) / ((fwd_ms + bwd_ms) / 1e3) / 1e9
        traffic = None
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(dom)
        except Exception:
            pass
        cores = 1
        cpu_v, cpu_dt = cpu_baseline(rows=96, cores=cores)
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
                             "fwd_ms": fwd_ms, "bwd_ms": bwd_ms},
                "cpu_baseline": {"value": cpu_v, "unit": UNIT, "cores": cores, "kind": "port",
                                 "sample": f"96 rows x T={T_LEN} fwd+bwd, oracle/stl_oracle.py "
                                           f"(numpy f64, single process), {cpu_dt:.1f}s"},
                "e2e": {"value": e2e_val, "unit": UNIT,
                        "h2d_bytes_per_step": B * T * 2 * 4,
                        "d2h_bytes_per_step": B * T * 4 + B * T * 2 * 4,
                        "ms_per_step": e2e_ms, "path": "paper_2501_04194_b200.trace + autograd",
                        "overlap": "H2D / compute / D2H on three streams, 2 buffer slots"},
                "gpu_launches": int(launches),
                "hard_c1": dict(hard, roofline_frac=(16.0 * B * T / ((hard["fwd_ms"] + hard["bwd_ms"]) / 1e3))
                                / 1e9 / hbm),
                "interval_sweep": sweep,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world)


if __name__ == "__main__":
    main()
