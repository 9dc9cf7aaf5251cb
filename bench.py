"""Benchmark: ternary-linear decode tokens/s on BASELINE.json configs[4].

Headline workload (the largest configuration of BASELINE.json that fits one
B200): cfg4, the ~100B-parameter ternary projection stack -- 80 layers,
hidden 10240 (q/o 10240x10240, k/v 10240->1280, gate/up 10240->32768, down
32768->10240), I2_S, M=1 decode -- exactly the reference bench's token pass
(pkg/src/ternpack/bench.py:138-153): per layer, two freshly quantised
activation vectors (hidden for q/k/v/o/gate/up, intermediate for down) and 7
exact int32 GEMVs rescaled by w_scale * a_scale.  One step = one token
through all 80 layers (24.9 GB of packed weights, far above the 126 MB L2,
so every step streams from HBM with no flush needed).

  value     device-resident throughput: K token passes captured in one CUDA
            graph (one fused step launch per layer), inputs already in HBM.
  e2e       the same token passes through the public API with HOST buffers:
            tb.HostPipeline over the 80 layers -- per token, the 80 layers'
            float32 inputs copied in from pinned host memory and all 560
            float32 output vectors copied back, inside the timed region.
  roofline  the fused step kernel (one launch per layer): algorithmic bytes
            per launch / its mean launch duration over the
            timed region, against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the unmodified reference (baseline/_ref: ternpack's own
            token pass, numba) on one layer, timed on the host cores, x 80;
            the C port of its byte-table kernels (oracle/c) beside it.
  configs   every other BASELINE config (cfg0, cfg1, cfg2 I2_S / TL2, cfg3
            prefill, cfg4 M=8), each with its own value, roofline fraction,
            e2e and cpu_baseline.

``--gpus N`` (N > 1) runs tensor parallel, strong scaling: the same cfg4
stack sharded over N ranks (column-parallel q/k/v/gate/up, row-parallel
o/down), the row-parallel int32 partials summed by our NVLink peer-memory
kernel (``--collective peer``, default) or NCCL (``--collective nccl``).
Without torchrun in the environment, ``--gpus N`` launches the N ranks
itself.  ``--impl reference`` times the unmodified reference package
(baseline/_ref, ternpack's own token pass) on the host cores on the same
workload, the C port beside it.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ternary-linear tokens/s (M=1 decode)"
H1, I1 = 4096, 14336           # cfg1 / cfg2 / cfg3 shapes (Llama-3-8B)
CFG4 = {"hidden": 10240, "kv": 1280, "inter": 32768, "layers": 80}
STACK_SEED = 11


def headline_config(world: int) -> dict:
    """The workload dict of the headline line -- identical in both arms."""
    return {"workload": "cfg4: ~100B-shaped ternary projection stack, 80 layers, hidden 10240 "
                        "(q/o 10240x10240, k/v 10240->1280, gate/up 10240->32768, "
                        "down 32768->10240), I2_S, M=1 decode",
            "format": "I2_S", "layers": 80, "tokens_per_step": 1,
            "weights": "seeded N(0,0.02) latent -> absmean ternary (core.py:104-113)",
            "activations": "fresh N(0,1) per layer, per-token absmax int8 (bench.py:141-142)",
            "l2": "24.9 GB packed weights per step >> 126 MB L2 (no flush needed)",
            "parallelism": f"tp{world}"}


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------

def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_int8_frac(tops):
    """tops against twice the measured dense bf16 burst rate of
    MEASURED_PEAKS.json (int8 tensor-core rate = 2 x bf16), or None."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return round(tops / (2.0 * float(json.load(f)["bf16_tflops"])), 4)
    except Exception:
        return None


def measured_traffic(name):
    """dram bytes read + write per launch of the named kernel capture
    (profiles/r2_traffic.json, from an ncu --set full capture), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            d = json.load(f)[name]
        return int(d["dram_bytes_read"] + d["dram_bytes_write"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def graph_time(torch, fn, reps=1):
    """Capture fn() once into a CUDA graph, replay once untimed, then time
    ``reps`` replays with CUDA events on the capture stream (ms per replay)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, g


def roofline(bytes_per_launch, launch_us, kernel, traffic=None, source=""):
    peak, kind = measured_peak()
    ach = bytes_per_launch / (launch_us * 1e-6) / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
            "frac": round(ach / peak, 4), "frac_vs_nominal_8000": round(ach / 8000.0, 4),
            "traffic": traffic, "kernel": kernel, "bytes_per_launch": int(bytes_per_launch),
            "launch_us": round(launch_us, 3), "launch_us_source": source,
            "peak_kind": f"{kind} hbm_gbs (copy)"}


# ---------------------------------------------------------------------------
# CPU port of the reference (oracle/c): cpu_baseline and --impl reference
# ---------------------------------------------------------------------------

def _co():
    from oracle import c_oracle as CO
    return CO


def cpu_stack_layer(fmt, mats, h, i):
    """f(xh, xi, threads): one layer of the reference token pass on the CPU
    port (bench.py:138-153): 2 quantisations (+ TL2 LUTs), 7 byte-table GEMVs.
    ``mats``: [(reference planes tuple, input index)] in layer order."""
    CO = _co()
    pad = 4 if fmt == "i2s" else 3

    def run(xh, xi, threads):
        qh, _ = CO.quantize(xh, pad)
        qi, _ = CO.quantize(xi, pad)
        if fmt == "tl2":
            # weights.groups = padded_cols / 3, cols padded to 6 (packing.py:50-53)
            luts = [CO.lut_tl2(qh, -(-h // 6) * 2), CO.lut_tl2(qi, -(-i // 6) * 2)]
        for planes, src in mats:
            if fmt == "i2s":
                CO.gemv_i2s(planes[0], qh if src == 0 else qi, threads)
            else:
                CO.gemv_tl2(planes[0], planes[1], luts[src], threads)
    return run


def time_cpu(run, args_fn, budget_s, threads_list):
    """Best rate (calls/s) over the thread counts, each timed for ~budget/len."""
    best = None
    for t in threads_list:
        run(*args_fn(0), t)  # warm
        n, t0 = 0, time.perf_counter()
        while True:
            run(*args_fn(n), t)
            n += 1
            el = time.perf_counter() - t0
            if el >= budget_s / len(threads_list):
                break
        rate = n / el
        if best is None or rate > best[0]:
            best = (rate, t, n)
    return best


def cpu_threads():
    CO = _co()
    ncpu = os.cpu_count() or 1
    return sorted({1, CO.max_threads(), ncpu}), ncpu


def cpu_baseline_stack(fmt, mats, h, i, layers, budget_s):
    rng = np.random.default_rng(7)
    X = [(rng.standard_normal(h).astype(np.float32), rng.standard_normal(i).astype(np.float32))
         for _ in range(4)]
    run = cpu_stack_layer(fmt, mats, h, i)
    ths, ncpu = cpu_threads()
    rate, t, n = time_cpu(run, lambda k: X[k % 4], budget_s, ths)
    return {"value": round(rate / layers, 4), "unit": "tokens/s", "cores": t, "kind": "port",
            "sample": f"{n} layers (2 quantise + 7 {fmt.upper()} byte-table GEMVs, M=1) on {t} "
                      f"thread(s), rate / {layers} layers; best of threads in {ths}; host "
                      f"{ncpu} CPUs ({cpu_model()})"}


# ---------------------------------------------------------------------------
# the unmodified reference package (baseline/_ref, pip --target install of
# /root/reference/pkg): ternpack's own token pass on the host cores
# ---------------------------------------------------------------------------

def ref_ternpack():
    """Import ``ternpack`` from baseline/_ref, or None when it is absent."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isfile(os.path.join(path, "ternpack", "__init__.py")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    # numba's on-disk cache: keep it out of the repo copy
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tb_numba_cache")
    try:
        import ternpack
        import ternpack.bench  # noqa: F401
        return ternpack
    except Exception:
        return None


def ref_layer(tp, fmt, mats):
    """One layer of reference packed matrices from [(planes, scale, rows,
    cols)] -- the bytes our generator (or LayerStack) produced, wrapped in
    the reference's own PackedI2S / PackedTL2 (packing.py:77-197)."""
    out = []
    for planes, scale, rows, cols in mats:
        if fmt == "i2s":
            out.append(tp.PackedI2S(rows=rows, cols=cols, padded_cols=-(-cols // 4) * 4,
                                    data=planes[0], scale=float(scale)))
        else:
            out.append(tp.PackedTL2(rows=rows, cols=cols, padded_cols=-(-cols // 6) * 6,
                                    index_data=planes[0], sign_data=planes[1],
                                    scale=float(scale)))
    return out


def time_ref_layer(tp, fmt, layer, h, i, budget_s, min_steps=1, max_steps=None, threads=None):
    """ternpack.bench._token_pass_int (bench.py:138-153) over ONE layer: its
    own 2 quantisations (+ TL2 LUTs) and 7 gemv_parallel calls, activations
    from its own rng.  One warm call (numba JIT, validate()) untimed; then
    layers until the budget (at least ``min_steps``).  -> (s per layer, n, threads)."""
    kind = tp.KernelKind.I2_S if fmt == "i2s" else tp.KernelKind.TL2
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(1)
    tp.bench._token_pass_int(kind, [layer], h, i, rng, threads)
    n, t0 = 0, time.perf_counter()
    while True:
        tp.bench._token_pass_int(kind, [layer], h, i, rng, threads)
        n += 1
        el = time.perf_counter() - t0
        if n >= min_steps and (el >= budget_s or (max_steps and n >= max_steps)):
            break
    return el / n, n, threads


def ref_baseline_stack(fmt, mats, h, i, layers, budget_s):
    """cpu_baseline from the real reference (kind "reference"); None when
    baseline/_ref is not importable (the caller then uses the C port)."""
    tp = ref_ternpack()
    if tp is None:
        return None
    layer = ref_layer(tp, fmt, mats)
    dt, n, th = time_ref_layer(tp, fmt, layer, h, i, budget_s)
    return {"value": round(1.0 / (layers * dt), 5), "unit": "tokens/s", "cores": th,
            "kind": "reference",
            "sample": f"{n} layers of ternpack.bench._token_pass_int ({fmt.upper()}, M=1: 2 "
                      f"quantize_activations + 7 gemv_parallel, numba) on {th} threads, "
                      f"tokens/s = 1 / ({layers} x layer time); host {os.cpu_count()} CPUs "
                      f"({cpu_model()}); unmodified reference from baseline/_ref"}


def stack_cpu_baselines(fmt, st, h, i, layers, budget_s):
    """(cpu_baseline, port line): the reference itself when it is installed
    (the port timed beside it), else the C port alone."""
    p0 = [p.p for p in st.layers[0]]
    if fmt == "i2s":
        planes = [(p.data.cpu().numpy(),) for p in p0]
    else:
        planes = [(p.index_data.cpu().numpy(), p.sign_data.cpu().numpy()) for p in p0]
    port = cpu_baseline_stack(fmt, [(pl, sh[3]) for pl, sh in zip(planes, st.shapes)],
                              h, i, layers, budget_s / 2)
    ref = ref_baseline_stack(fmt, [(pl, p.scale, sh[1], sh[2])
                                   for pl, p, sh in zip(planes, p0, st.shapes)],
                             h, i, layers, budget_s / 2)
    if ref is None:
        return port, None
    return ref, port


# ---------------------------------------------------------------------------
# headline: cfg4 stack, M=1, tp = world
# ---------------------------------------------------------------------------

def make_collective(args, rank, world):
    import torch.distributed as dist

    from paper_2410_16144_b200 import tp as TP
    if world == 1:
        return None
    if args.collective == "peer" and dist.get_backend() == "nccl":
        return TP.PeerAllReduce(rank, world)
    return TP.TorchAllReduce()


def tp_layer0_matches(torch, st, XH, XI):
    """Layer 0 of a tensor-parallel stack (after a token pass) against the
    same layer built whole on this GPU: this rank's rows of the column-parallel
    projections and the full reduced rows of o/down, bit for bit."""
    from paper_2410_16144_b200.stack import LayerStack
    ref = LayerStack(CFG4, fmt="i2s", seed=STACK_SEED, tokens=1, layers=1)
    ref.token_pass([XH[0]], [XI[0]])
    torch.cuda.synchronize()
    want, got = ref.outputs(0), st.outputs(0)
    ok = True
    for name, rows, cols, src, kind, lo, hi in st.plan:
        w = want[name] if kind == "row" else want[name][lo:hi]
        ok = ok and bool(torch.equal(got[name], w))
    del ref
    torch.cuda.empty_cache()
    return ok


def run_headline(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2410_16144_b200 as tb
    from paper_2410_16144_b200.stack import LayerStack

    dev = torch.cuda.current_device()
    coll = make_collective(args, rank, world)
    t0 = time.perf_counter()
    st = LayerStack(CFG4, fmt="i2s", seed=STACK_SEED, tokens=1, tp_rank=rank, tp_world=world,
                    collective=coll)
    build_s = time.perf_counter() - t0
    L, h, i = CFG4["layers"], CFG4["hidden"], CFG4["inter"]
    g = torch.Generator(device="cuda").manual_seed(99)  # same inputs on every rank
    XH = torch.randn(L, h, generator=g, device="cuda")
    XI = torch.randn(L, i, generator=g, device="cuda")
    xh, xi = list(XH), list(XI)

    def run_steps(n):
        for _ in range(n):
            st.token_pass(xh, xi)

    run_steps(args.warmup)
    torch.cuda.synchronize()
    tp_check = None
    if world > 1:
        # on-hardware parity of the sharded pass: layer 0 of this rank's stack
        # against the same layer built unsharded (bit-identical);
        # a peer reduction that timed out or disagrees falls back to NCCL
        ok = tp_layer0_matches(torch, st, XH, XI) and not getattr(coll, "timed_out", lambda: 0)()
        t = torch.tensor([int(ok)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        tp_check = {"layer": 0, "bit_identical_to_tp1": bool(t.item()),
                    "collective": type(coll).__name__}
        if not t.item() and type(coll).__name__ == "PeerAllReduce":
            del st
            torch.cuda.empty_cache()
            from paper_2410_16144_b200 import tp as TP
            coll = TP.TorchAllReduce()
            st = LayerStack(CFG4, fmt="i2s", seed=STACK_SEED, tokens=1, tp_rank=rank,
                            tp_world=world, collective=coll)
            run_steps(args.warmup)
            torch.cuda.synchronize()
            t = torch.tensor([int(tp_layer0_matches(torch, st, XH, XI))], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            tp_check = {"layer": 0, "bit_identical_to_tp1": bool(t.item()),
                        "collective": "TorchAllReduce (fallback: the peer kernel failed "
                                      "the check)"}
    capturable = coll is None or coll.capturable
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = None
    if capturable:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                run_steps(args.steps)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            graph.replay()  # untimed (uploads the graph)
        torch.cuda.synchronize()

        def timed():
            graph.replay()
    else:
        def timed():
            run_steps(args.steps)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        with torch.cuda.stream(s):
            e0.record()
            timed()
            e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    # the timed region is the step-kernel chain (80 fused launches per token,
    # + at tp > 1 one peer reduction per layer): a launch's mean duration is
    # the region time / launches (conservative: the tail finalize is inside)
    launch_us = ms_step * 1e3 / L
    per_launch = st.algo_bytes / L
    res = {
        "metric": METRIC, "value": round(1000.0 / ms_step, 3), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "i8",
        "data": "synthetic (seeded N(0,0.02) latent weights -> absmean ternary I2_S; "
                "N(0,1) activations)",
        "config": headline_config(world),
        "roofline": roofline(per_launch, launch_us,
                             "tgemv_kernel<I2S,1,fused>: one layer = quantise x_h, x_i + "
                             "q/k/v/o/gate/up/down grouped GEMV + previous layer's finalize"
                             + (f" (this rank's tp{world} shards)" if world > 1 else ""),
                             measured_traffic("cfg4_layer_step") if world == 1 else None,
                             f"timed region / ({args.steps} steps x {L} layer launches)"),
        "gpu_launches": args.steps * (L + 1 + (L if world > 1 else 0)),
        "clocks": clk.summary(),
        "build_s": round(build_s, 1),
    }
    if world > 1:
        res["collective"] = type(coll).__name__
        res["tp_check"] = tp_check
        res["roofline"]["note"] = ("per-rank bytes of its shards; the launch time includes "
                                   "the row-parallel reduction")
    graph = None
    # ---- e2e: the public API from host memory (rank 0, tp1)
    if rank == 0 and world == 1 and not args.no_e2e:
        res["e2e"] = e2e_stack(torch, tb, st, args.steps)
    elif world > 1:
        res["e2e"] = None
        res["e2e_note"] = "tp > 1: host-buffer pass not measured (device-resident value only)"
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"], port = stack_cpu_baselines("i2s", st, h, i, L, args.cpu_budget)
        if port is not None:
            res["cpu_baseline_port"] = port
    del st
    torch.cuda.empty_cache()
    return res


def e2e_stack(torch, tb, st, steps):
    """One token pass through tb.HostPipeline per step: the layers' inputs
    from pinned host memory in, every projection's fp32 output out."""
    L, h, i = st.nlayers, st.ks[0], st.ks[1]
    pairs = [[(p, sh[3]) for p, sh in zip(plans, st.shapes)] for plans in st.layers]
    pipe = tb.HostPipeline(pairs, [h, i], steps=L)
    g = torch.Generator().manual_seed(5)
    pipe.inputs[0].copy_(torch.randn(L, h, generator=g))
    pipe.inputs[1].copy_(torch.randn(L, i, generator=g))
    for _ in range(2):
        pipe.run()
    n = max(5, min(steps, 50))
    t0 = time.perf_counter()
    for _ in range(n):
        pipe.run()
    dt = (time.perf_counter() - t0) / n
    rows = sum(sh[1] for sh in st.shapes)
    out = {"value": round(1.0 / dt, 3), "unit": "tokens/s",
           "h2d_bytes_per_step": L * (h + i) * 4, "d2h_bytes_per_step": L * rows * 4,
           "steps": n,
           "path": f"tb.HostPipeline.run() over the {L} layers: per token, the layers' f32 "
                   "inputs H2D from pinned host memory and all 7 f32 output vectors of every "
                   "layer D2H to pinned host memory, copies on two streams overlapping the "
                   "fused-step chain; wall clock incl. the per-token sync"}
    del pipe
    return out


# ---------------------------------------------------------------------------
# the other BASELINE configs (rank 0, one GPU)
# ---------------------------------------------------------------------------

def run_cfg0(torch, tb, args, copies=32, steps=200):
    """configs[0]: one I2_S GEMV, M=1, 4096 x 4096 -- one fused launch per
    token (quantise + GEMV + its own finalize), rotating over 32 weight
    copies (134 MB > L2) in a CUDA graph."""
    n = k = 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    plans, steps_obj = [], []
    for _ in range(copies):
        w = torch.randn(n, k, generator=g, device="cuda") * 0.02
        plan = tb.GemvPlan(tb.encode_i2s(tb.ternarize_weights(w, n, k)), out_dtype=torch.float32)
        plans.append(plan)
        # independent GEMVs: every launch finalises its own outputs and none
        # waits for its predecessor (TB_STEP_INDEPENDENT; a step is reused
        # after 31 other launches), so they overlap instead of completing in
        # launch order
        steps_obj.append(tb.GemvStep([(plan, 0)], [k], independent=True))
        del w
    X = torch.randn(16, k, generator=g, device="cuda")

    def run(cnt):
        for j in range(cnt):
            steps_obj[j % copies].run([X[j % 16]])

    run(copies)
    torch.cuda.synchronize()
    ms, _ = graph_time(torch, lambda: run(steps))
    us = ms * 1e3 / steps
    algo = n * k // 4 + k + 4 * n
    out = {"workload": "cfg0: I2_S GEMV M=1, 4096x4096, one fused launch per token "
                       "(32 rotating weight copies, 134 MB > L2)",
           "value": round(1e6 / us, 1), "unit": "tokens/s", "us_per_gemv": round(us, 3),
           "roofline": roofline(algo, us, "tgemv_kernel<I2S,1,fused>, self-finalising independent launches (one GEMV each)",
                                measured_traffic("cfg0_gemv"), "graph of 200 chained launches")}
    if not args.no_e2e:
        pipe = tb.HostPipeline([[(p, 0)] for p in plans[:8]], [k], steps=400)
        pipe.inputs[0].copy_(torch.randn(400, k))
        for _ in range(2):
            pipe.run()
        reps = []
        for _ in range(5):
            t0 = time.perf_counter()
            pipe.run()
            reps.append(time.perf_counter() - t0)
        e = sorted(reps)[2] / 400
        out["e2e"] = {"value": round(1 / e, 1), "unit": "tokens/s", "h2d_bytes_per_step": 4 * k,
                      "d2h_bytes_per_step": 4 * n, "steps": 400,
                      "path": "tb.HostPipeline: 400 independent GEMVs per run, pinned host f32 "
                              "inputs in / f32 outputs out, median of 5 runs"}
        del pipe
    if not args.no_cpu_baseline:
        CO = _co()
        packed = plans[0].p.data.cpu().numpy()
        xs = [np.random.default_rng(s).standard_normal(k).astype(np.float32) for s in range(4)]

        def one(x, t):
            q, _ = CO.quantize(x, 4)
            CO.gemv_i2s(packed, q, t)
        ths, ncpu = cpu_threads()
        rate, t, cnt = time_cpu(one, lambda j: (xs[j % 4],), args.cpu_budget / 4, ths)
        out["cpu_baseline"] = {"value": round(rate, 2), "unit": "tokens/s", "cores": t,
                               "kind": "port",
                               "sample": f"{cnt} GEMVs (quantise + I2_S byte-table gather) on {t} "
                                         f"thread(s); best of {ths}; {ncpu} CPUs ({cpu_model()})"}
    return out


def run_cfg1(torch, tb, args, ncopy=6, nx=64):
    """configs[1]: the TL1 FFN block at M=1 -- gate and up (4096 -> 14336) on
    one quantised vector, down (14336 -> 4096) on another, one fused launch
    per token, rotating over 6 weight copies (264 MB > L2)."""
    plans = []
    for c in range(ncopy):
        gen = torch.Generator(device="cuda").manual_seed(1000 + c)
        mats = {}
        for name, rows, cols in (("gate", I1, H1), ("up", I1, H1), ("down", H1, I1)):
            w = torch.randn(rows, cols, generator=gen, device="cuda", dtype=torch.float32) * 0.02
            mats[name] = tb.encode_tl1(tb.ternarize_weights(w, rows, cols))
            del w
        pl = {k: tb.GemvPlan(v, out_dtype=torch.float32) for k, v in mats.items()}
        pl["mats"] = mats
        pl["step"] = tb.GemvStep([(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)], [H1, I1])
        plans.append(pl)
    gen = torch.Generator(device="cuda").manual_seed(77)
    XH = torch.randn(nx, H1, generator=gen, device="cuda")
    XI = torch.randn(nx, I1, generator=gen, device="cuda")

    def run(n):
        prev = None
        for j in range(n):
            pl = plans[j % ncopy]
            pl["step"].run([XH[j % nx], XI[j % nx]], prev=prev["step"] if prev else None)
            prev = pl
        prev["step"].finalize()

    run(max(args.warmup, ncopy))
    torch.cuda.synchronize()
    K = 400
    ms, _ = graph_time(torch, lambda: run(K))
    us = ms * 1e3 / K
    tl1 = lambda r, c: r * (-(-(-(-c // 2) * 2 // 2) // 2))  # noqa: E731  packing.py:46-48
    algo = 2 * (tl1(I1, H1) + H1 + 4 * I1) + tl1(H1, I1) + I1 + 4 * H1
    out = {"workload": "cfg1: TL1 FFN block, gate/up 4096->14336 + down 14336->4096, M=1, one "
                       "fused launch per token (6 rotating weight copies, 264 MB > L2)",
           "value": round(1e6 / us, 1), "unit": "tokens/s", "us_per_step": round(us, 3),
           "roofline": roofline(algo, us, "tgemv_kernel<TL1,1,fused>: quantise x_h, x_i + "
                                "gate/up/down + previous finalize",
                                measured_traffic("cfg1_step"), f"graph of {K} chained launches")}
    if not args.no_e2e:
        pipe = tb.HostPipeline([[(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)]
                                for pl in plans], [H1, I1], steps=400)
        g = torch.Generator().manual_seed(6)
        pipe.inputs[0].copy_(torch.randn(400, H1, generator=g))
        pipe.inputs[1].copy_(torch.randn(400, I1, generator=g))
        for _ in range(3):
            pipe.run()
        reps = []
        for _ in range(5):
            t0 = time.perf_counter()
            pipe.run()
            reps.append(time.perf_counter() - t0)
        e = sorted(reps)[2] / 400
        out["e2e"] = {"value": round(1 / e, 1), "unit": "tokens/s",
                      "h2d_bytes_per_step": (H1 + I1) * 4, "d2h_bytes_per_step": (2 * I1 + H1) * 4,
                      "steps": 400, "path": "tb.HostPipeline: 400 independent FFN tokens per "
                                            "run, pinned host in/out, median of 5 runs"}
        del pipe
        # one token at a time, synchronous (decode latency)
        hosts = [tb.HostStep([(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)], [H1, I1])
                 for pl in plans]
        xh_h = torch.randn(nx, H1).pin_memory()
        xi_h = torch.randn(nx, I1).pin_memory()
        for j in range(5):
            hosts[j % ncopy]([xh_h[j % nx], xi_h[j % nx]])
        n = 50
        t0 = time.perf_counter()
        for j in range(n):
            hosts[j % ncopy]([xh_h[j % nx], xi_h[j % nx]])
        dt = (time.perf_counter() - t0) / n
        out["e2e_sync"] = {"value": round(1 / dt, 1), "unit": "tokens/s",
                           "us_per_token": round(dt * 1e6, 2), "steps": n,
                           "path": "tb.HostStep: one token per call (H2D, step, finalize into "
                                   "mapped pinned memory, sync)"}
        # the reference call pattern: quantize_activations + gemv_parallel x3
        KK = tb.KernelKind
        for _ in range(2):  # warm every copy's lazily built workspace and outputs
            for pl in plans:
                m = pl["mats"]
                qa = tb.quantize_activations(xh_h[0], pad_to=2)
                for nm in ("gate", "up"):
                    tb.gemv_parallel(KK.TL1, m[nm], qa)
                tb.gemv_parallel(KK.TL1, m["down"], tb.quantize_activations(xi_h[0], pad_to=2))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j in range(n):
            m = plans[j % ncopy]["mats"]
            qh = tb.quantize_activations(xh_h[j % nx], pad_to=2)
            rg = tb.gemv_parallel(KK.TL1, m["gate"], qh)
            ru = tb.gemv_parallel(KK.TL1, m["up"], qh)
            rd = tb.gemv_parallel(KK.TL1, m["down"], tb.quantize_activations(xi_h[j % nx],
                                                                              pad_to=2))
            rg.output.cpu(), ru.output.cpu(), rd.output.cpu()
        dt = (time.perf_counter() - t0) / n
        out["e2e_reference_api"] = {
            "value": round(1 / dt, 1), "unit": "tokens/s", "steps": n,
            "h2d_bytes_per_step": (H1 + I1) * 4, "d2h_bytes_per_step": (2 * I1 + H1) * 8,
            "path": "tb.quantize_activations + tb.gemv_parallel(TL1) x3 per token (the "
                    "reference call pattern, bench.py:138-153), float64 outputs to host"}
    if not args.no_cpu_baseline:
        CO = _co()
        host = {k: plans[0]["mats"][k].data.cpu().numpy() for k in ("gate", "up", "down")}
        rng = np.random.default_rng(7)
        xs = [(rng.standard_normal(H1).astype(np.float32),
               rng.standard_normal(I1).astype(np.float32)) for _ in range(4)]

        def one(xh, xi, t):
            qh, _ = CO.quantize(xh, 2)
            lh = CO.lut_tl1(qh, H1 // 2)
            CO.gemv_tl1(host["gate"], lh, t)
            CO.gemv_tl1(host["up"], lh, t)
            qi, _ = CO.quantize(xi, 2)
            CO.gemv_tl1(host["down"], CO.lut_tl1(qi, I1 // 2), t)
        ths, ncpu = cpu_threads()
        rate, t, cnt = time_cpu(one, lambda j: xs[j % 4], args.cpu_budget / 2, ths)
        out["cpu_baseline"] = {"value": round(rate, 2), "unit": "tokens/s", "cores": t,
                               "kind": "port",
                               "sample": f"{cnt} TL1 FFN tokens (quantise + LUT + byte-table "
                                         f"gathers) on {t} thread(s); best of {ths}; {ncpu} CPUs "
                                         f"({cpu_model()})"}
    del plans
    torch.cuda.empty_cache()
    return out


def run_stack_cfg(torch, tb, args, name, fmt, tokens, passes=10):
    """configs[2] (cfg2, I2_S / TL2) and configs[4] at M=8: M-token decode
    through the whole stack, one launch per layer (M=1) or glue + grouped
    GEMV per layer (M > 1)."""
    from paper_2410_16144_b200.stack import STACKS, LayerStack
    cfg = STACKS[name]
    t0 = time.perf_counter()
    st = LayerStack(cfg, fmt=fmt, seed=STACK_SEED, tokens=tokens)
    build_s = time.perf_counter() - t0
    g = torch.Generator(device="cuda").manual_seed(99)
    L, h, i = st.nlayers, cfg["hidden"], cfg["inter"]
    if tokens == 1:
        XH = torch.randn(L, h, generator=g, device="cuda")
        XI = torch.randn(L, i, generator=g, device="cuda")
        xh, xi, glues = list(XH), list(XI), None
    else:
        XH = torch.randn(L, tokens, h, generator=g, device="cuda")
        XI = torch.randn(L, tokens, i, generator=g, device="cuda")
        xh = xi = None
        glues = st.make_glues(XH, XI)
    st.token_pass(xh, xi, glues)
    torch.cuda.synchronize()
    ms, _ = graph_time(torch, lambda: [st.token_pass(xh, xi, glues) for _ in range(passes)])
    ms /= passes
    launches = L if tokens == 1 else 2 * L
    kern = (f"tgemv_kernel<{fmt.upper()},1,fused> per layer" if tokens == 1 else
            f"glue_kernel (quantise, previous finalize) + tgemv_kernel<{fmt.upper()},{tokens},records table> "
            "per layer, pipelined through per-layer counters")
    out = {"workload": f"{name}: {L} layers, hidden {h}, {fmt.upper()}, M={tokens}",
           "value": round(tokens * 1000.0 / ms, 2), "unit": "tokens/s",
           "ms_per_token_pass": round(ms, 4), "algo_bytes_per_pass": int(st.algo_bytes),
           "roofline": roofline(st.algo_bytes / L, ms * 1e3 / L, kern,
                                measured_traffic(f"{name}_{fmt}_m{tokens}"),
                                f"graph of {passes} token passes / {L} layers"),
           "launches_per_pass": launches + 1, "build_s": round(build_s, 1)}
    if tokens > 1:
        from paper_2410_16144_b200 import _lib as tb_lib
        out["pipelined_layers"] = bool(getattr(st, "piped", False))
        out["sync_timeouts"] = int(tb_lib.load().tb_sync_timeouts())  # bounded waits that expired: 0
    if tokens == 1 and not args.no_e2e:
        out["e2e"] = e2e_stack(torch, tb, st, 20)
    if not args.no_cpu_baseline:
        cb, port = stack_cpu_baselines(fmt, st, h, i, L, args.cpu_budget / 2)
        if tokens > 1:  # the reference has no multi-token path: M tokens = M passes
            cb["sample"] += f"; M={tokens} costs {tokens} such passes (rate is per token)"
        out["cpu_baseline"] = cb
        if port is not None:
            out["cpu_baseline_port"] = port
    del st
    torch.cuda.empty_cache()
    return out


def run_cfg3(torch, tb, args, copies=2, reps=10):
    """configs[3]: one Llama-3-8B-shaped layer at M=512 (I2_S): per-token
    quantisation of x_h [512, 4096] and x_i [512, 14336], their tensor-core
    tiling (tb_gemm_tile_act) and ONE grouped tcgen05 kind::i8 launch over
    q/k/v/o/gate/up/down -- all inside the timed region.
    int8 TOPS = 2 * M * sum(N * K) / time."""
    import ctypes as C

    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    M, KV = 512, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    XH = torch.randn(M, H1, generator=g, device="cuda")
    XI = torch.randn(M, I1, generator=g, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    sc = {k: torch.empty(M, dtype=torch.float64, device="cuda") for k in (H1, I1)}
    til = {k: torch.empty(lib.tb_gemm_act_bytes(M, k), dtype=torch.uint8, device="cuda")
           for k in (H1, I1)}
    shapes = [(H1, H1), (KV, H1), (KV, H1), (H1, H1), (I1, H1), (I1, H1), (H1, I1)]
    ops = 2 * M * sum(n * k for n, k in shapes)
    layers = []
    for _ in range(copies):
        descs = (L.GemmDesc * len(shapes))()
        keep = []
        for d, (n, k) in zip(descs, shapes):
            w = torch.randn(n, k, generator=g, device="cuda") * 0.02
            p = tb.encode_i2s(tb.ternarize_weights(w, n, k))
            del w
            main, _ = p.tiled()
            out = torch.empty((M, n), dtype=torch.float32, device="cuda")
            d.tiled, d.rows, d.cols, d.act_tiled = main.data_ptr(), n, k, til[k].data_ptr()
            d.a_scale, d.w_scale, d.out32 = sc[k].data_ptr(), float(p.scale), out.data_ptr()
            keep.append((p, main, out))
        layers.append((descs, keep))

    def gemm(j):
        L.check(lib.tb_gemm_batch(L.I2S, len(shapes), C.cast(layers[j % copies][0], C.c_void_p),
                                  M, L.stream_ptr()), "gemm_batch")

    def layer(j, xh=XH, xi=XI):
        # quantize_activations of both inputs straight into the GEMM operand
        # layout (tb_gemm_quantize_act_multi: one launch pair for both), then
        # the GEMM as its programmatic dependent
        qd = (L.QactDesc * 2)()
        for d, (x, k) in zip(qd, ((xh, H1), (xi, I1))):
            d.x, d.cols, d.ldx = x.data_ptr(), k, k
            d.scale, d.nonfinite_flag, d.act_tiled = (sc[k].data_ptr(), flag.data_ptr(),
                                                      til[k].data_ptr())
        L.check(lib.tb_gemm_quantize_act_multi(2, C.cast(qd, C.c_void_p), M, L.stream_ptr()),
                "gemm_quantize_act_multi")
        gemm(j)

    layer(0)
    torch.cuda.synchronize()
    ms, _ = graph_time(torch, lambda: [layer(j) for j in range(reps)])
    ms /= reps
    ms_gemm, _ = graph_time(torch, lambda: [gemm(j) for j in range(reps)])
    ms_gemm /= reps
    a = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
    bt = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
    torch._int_mm(a, bt)  # cuBLASLt init / workspace outside the capture
    torch.cuda.synchronize()
    pk_ms, _ = graph_time(torch, lambda: [torch._int_mm(a, bt) for _ in range(5)])
    peak = 2 * 8192 ** 3 / (pk_ms / 5 * 1e-3) / 1e12
    del a, bt
    tops = ops / (ms * 1e-3) / 1e12
    tops_g = ops / (ms_gemm * 1e-3) / 1e12
    out = {"workload": "cfg3: one Llama-3-8B-shaped layer (q,k,v,o,gate,up,down), M=512, I2_S: "
                       "one grouped quantise-to-operand launch pair + one grouped tcgen05 kind::i8 GEMM launch",
           "value": round(M * 1000.0 / ms, 1), "unit": "tokens/s (prefill, one layer)",
           "tops": round(tops, 1), "us_per_layer": round(ms * 1e3, 1),
           "gemm_only_tops": round(tops_g, 1), "gemm_only_us": round(ms_gemm * 1e3, 1),
           "gop": round(ops / 1e9, 1),
           "roofline": {"bound": "tensor", "achieved": round(tops_g, 1), "peak": round(peak, 1),
                        "unit": "TOPS", "frac": round(tops_g / peak, 4),
                        "frac_vs_nominal_4500": round(tops_g / 4500.0, 4),
                        "frac_vs_2x_measured_bf16": measured_int8_frac(tops_g),
                        "kernel": "tgemm_kernel (tcgen05.mma kind::i8, TMEM accumulators)",
                        "peak_kind": "cuBLASLt int8 (torch._int_mm 8192^3) measured in this run",
                        "traffic": None}}
    if not args.no_e2e:
        xh_h = torch.randn(M, H1).pin_memory()
        xi_h = torch.randn(M, I1).pin_memory()
        outs_h = [torch.empty((M, n), dtype=torch.float32).pin_memory() for n, _ in shapes]
        xh_d, xi_d = torch.empty_like(XH), torch.empty_like(XI)

        def e2e_layer():
            xh_d.copy_(xh_h, non_blocking=True)
            xi_d.copy_(xi_h, non_blocking=True)
            layer(0, xh_d, xi_d)
            for oh, (_, _, od) in zip(outs_h, layers[0][1]):
                oh.copy_(od, non_blocking=True)
        e2e_layer()
        torch.cuda.synchronize()
        n = 10
        t0 = time.perf_counter()
        for _ in range(n):
            e2e_layer()
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        rows = sum(nn for nn, _ in shapes)
        out["e2e"] = {"value": round(M / dt, 1), "unit": "tokens/s (prefill, one layer)",
                      "h2d_bytes_per_step": M * (H1 + I1) * 4, "d2h_bytes_per_step": M * rows * 4,
                      "steps": n, "path": "pinned host f32 x_h, x_i -> H2D -> quantise + tile + "
                                          "GEMM -> all 7 f32 [512, N] outputs D2H; wall clock"}
    if not args.no_cpu_baseline:
        CO = _co()
        packed = layers[0][1][0][0].data.cpu().numpy()  # q projection, 4096 x 4096
        xs = XH[:16].cpu().numpy()

        def one(x, t):
            qq, _ = CO.quantize(x, 4)
            CO.gemv_i2s(packed, qq, t)
        ths, ncpu = cpu_threads()
        rate, t, cnt = time_cpu(one, lambda j: (xs[j % 16],), args.cpu_budget / 4, ths)
        # q-projection GEMVs/s -> layer tokens/s by the MAC ratio
        frac_q = (H1 * H1) / sum(nn * kk for nn, kk in shapes)
        out["cpu_baseline"] = {"value": round(rate * frac_q, 3),
                               "unit": "tokens/s (prefill, one layer)",
                               "tops": round(rate * 2 * H1 * H1 / 1e12, 5), "cores": t,
                               "kind": "port",
                               "sample": f"{cnt} per-token q-projection GEMVs (4096x4096, quantise"
                                         f" + byte-table gather; the reference has no GEMM, "
                                         f"SPEC.md:346) on {t} thread(s), scaled to the "
                                         f"7-projection layer by MACs; best of {ths}; {ncpu} CPUs "
                                         f"({cpu_model()})"}
    del layers
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# --impl reference
# ---------------------------------------------------------------------------

def host_stack_layer(seed, cfg):
    """One cfg4 layer generated on the host: seeded N(0, 0.02) float32 latent
    matrices, absmean-ternarised (core.py:104-113 arithmetic, in row blocks)
    and packed to the reference I2_S bytes (packing.py:200-206).
    -> [((packed,), scale, rows, cols, input)]."""
    from oracle import ternpack_oracle as O
    from paper_2410_16144_b200.stack import stack_shapes
    mats = []
    for mi, (name, rows, cols, src) in enumerate(stack_shapes(cfg)):
        rng = np.random.default_rng(seed * 1_000_003 + mi)
        w = rng.standard_normal((rows, cols), dtype=np.float32)
        w *= np.float32(0.02)
        blk = max(1, (64 << 20) // (8 * cols))
        tot = 0.0
        for r0 in range(0, rows, blk):
            tot += float(np.abs(w[r0:r0 + blk].astype(np.float64)).sum())
        scale = tot / (rows * cols)
        packed = np.empty((rows, -(-cols // 4)), dtype=np.uint8)
        for r0 in range(0, rows, blk):
            v = np.clip(O.round_half_away(w[r0:r0 + blk].astype(np.float64) / scale), -1, 1)
            packed[r0:r0 + blk] = O.encode_i2s(v.astype(np.int8))
        del w
        mats.append(((packed,), scale, rows, cols, src))
    return mats


def run_reference(args, world):
    """The reference's CPU path on the headline workload, all host threads.
    Each timed step is one layer of the 80-layer token pass, run by the
    UNMODIFIED reference (baseline/_ref: ternpack.bench._token_pass_int --
    2 quantize_activations + 7 gemv_parallel, numba byte-table kernels);
    value = 1 / (80 x mean layer time).  The C port (oracle/c) is timed
    beside it on a short sample; it alone is used if baseline/_ref is absent."""
    t0 = time.perf_counter()
    mats = host_stack_layer(STACK_SEED, CFG4)
    gen_s = time.perf_counter() - t0
    h, i, L = CFG4["hidden"], CFG4["inter"], CFG4["layers"]
    threads = os.cpu_count() or 1
    # the C port, a short sample beside the reference
    run = cpu_stack_layer("i2s", [(pl, src) for pl, _, _, _, src in mats], h, i)
    rng = np.random.default_rng(7)
    X = [(rng.standard_normal(h).astype(np.float32), rng.standard_normal(i).astype(np.float32))
         for _ in range(4)]
    run(*X[0], threads)
    np_, t0 = 0, time.perf_counter()
    while np_ < 3 or time.perf_counter() - t0 < 3.0:
        run(*X[np_ % 4], threads)
        np_ += 1
    port_v = 1.0 / (L * (time.perf_counter() - t0) / np_)
    tp = ref_ternpack()
    if tp is not None:
        layer = ref_layer(tp, "i2s", [(pl, sc, r, c) for pl, sc, r, c, _ in mats])
        for _ in range(max(0, args.warmup - 1)):  # time_ref_layer makes one more warm call
            tp.bench._token_pass_int(tp.KernelKind.I2_S, [layer], h, i,
                                     np.random.default_rng(2), threads)
        dt, n, _ = time_ref_layer(tp, "i2s", layer, h, i, 0.0, min_steps=args.steps)
        kind = "reference"
        what = ("unmodified reference from baseline/_ref: ternpack.bench._token_pass_int over "
                "one layer (2 quantize_activations + 7 gemv_parallel(I2_S), numba)")
    else:
        for j in range(args.warmup):
            run(*X[j % 4], threads)
        t0 = time.perf_counter()
        for j in range(args.steps):
            run(*X[j % 4], threads)
        dt, n = (time.perf_counter() - t0) / args.steps, args.steps
        kind = "port"
        what = ("C port of the reference byte-table kernels (oracle/c), baseline/_ref absent: "
                "2 quantise + 7 I2_S GEMVs")
    v = round(1.0 / (L * dt), 5)
    sample = (f"{n} timed layers of the cfg4 token pass (M=1) on {threads} threads, "
              f"tokens/s = 1 / (80 x layer time); {what}; {threads} CPUs ({cpu_model()}); "
              f"weights generated on the host in {gen_s:.0f} s")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(L * dt * 1e3, 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "i8",
            "data": "synthetic (seeded N(0,0.02) latent weights -> absmean ternary I2_S; "
                    "N(0,1) activations)",
            "config": headline_config(world),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "cpu_port": {"value": round(port_v, 5), "unit": "tokens/s", "cores": threads,
                         "kind": "port", "sample": f"{np_} layers of the C port (oracle/c)"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------------------

def _spawn(args):
    """--gpus N without a torchrun environment: launch the N ranks ourselves."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={29500 + os.getpid() % 1000}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--collective", default="peer", choices=["peer", "nccl"],
                    help="tp > 1: row-parallel reduction by our peer-memory kernel or NCCL")
    ap.add_argument("--headline-only", action="store_true",
                    help="skip the other BASELINE configs")
    ap.add_argument("--configs", default="cfg0,cfg1,cfg2:i2s,cfg2:tl2,cfg3,cfg4:m8",
                    help="secondary config lines (comma list)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return

    import torch
    if world > 1:
        import torch.distributed as dist
        lr = int(os.environ.get("LOCAL_RANK", 0))
        if os.environ.get("TB_BENCH_SHARE_GPU") == "1":  # functional check only (1-GPU box)
            lr %= torch.cuda.device_count()
        torch.cuda.set_device(lr)
        dist.init_process_group(os.environ.get("TB_BENCH_DIST_BACKEND", "nccl"))
    res = run_headline(args, rank, world)
    if rank == 0 and world == 1 and not args.headline_only:
        import paper_2410_16144_b200 as tb
        res["configs"] = {}
        fns = {"cfg0": lambda: run_cfg0(torch, tb, args),
               "cfg1": lambda: run_cfg1(torch, tb, args),
               "cfg2:i2s": lambda: run_stack_cfg(torch, tb, args, "cfg2", "i2s", 1),
               "cfg2:tl2": lambda: run_stack_cfg(torch, tb, args, "cfg2", "tl2", 1),
               "cfg3": lambda: run_cfg3(torch, tb, args),
               "cfg4:m8": lambda: run_stack_cfg(torch, tb, args, "cfg4", "i2s", 8, passes=4)}
        for name in [c for c in args.configs.split(",") if c]:
            try:
                res["configs"][name] = fns[name]()
            except Exception as e:  # a secondary line must not lose the headline
                import traceback
                res["configs"][name] = {"error": f"{type(e).__name__}: {e}",
                                        "where": traceback.format_exc()[-1500:]}
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
