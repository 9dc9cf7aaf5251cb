"""Benchmark: ternary-linear tokens/s at M=1 decode on BASELINE.json config 1.

Workload (BASELINE.json configs[1]): the TL1 FFN block of a Llama-3-8B-shaped
layer at M=1 -- gate and up (K=4096 -> N=14336) on one freshly quantised
activation vector, down (K=14336 -> N=4096) on another, exactly the per-layer
work of the reference bench's token pass (pkg/src/ternpack/bench.py:138-153):
per-token absmax int8 quantisation + (implicit) TL1 LUT + exact int32 GEMV +
rescale.  One "step" = one token through that block.

  value   device-resident throughput: K steps captured in one CUDA graph,
          inputs already in HBM, weights rotated over 6 distinct copies
          (265 MB > 126 MB L2) so every step streams from HBM.
  e2e     the same steps through the public Python API (quantize_activations
          + gemv_parallel) with pinned HOST inputs and the float64 results
          read back to the host inside the timed region.
  roofline  the TL1 GEMV kernel timed alone (graph of back-to-back launches
          over the rotating copies, CUDA events): algorithmic bytes per
          launch / mean launch time vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the C port of the reference byte-table CPU kernels
          (oracle/c/tern_oracle.c) on this host, bounded sample.

``--impl reference`` times that CPU port alone on the same workload (rank 0).
Multi-GPU (torchrun, N>1): tensor parallel -- gate/up column-parallel, down
row-parallel with an NCCL all-reduce of the int32 partial accumulators.
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

H, I = 4096, 14336
NCOPY = 6
NX = 64
METRIC = "ternary-linear tokens/s (M=1 decode)"


def tl1_bytes(rows, cols):
    return rows * (-(-(-(-cols // 2) * 2 // 2) // 2))


def algo_bytes_gemv(rows, cols, m=1):
    # packed weights (reference TL1 size) + int8 activations + fp32 outputs
    return tl1_bytes(rows, cols) + m * cols + 4 * m * rows


def measured_traffic():
    """DRAM bytes per launch of the step kernel from the committed ncu --set full
    capture (profiles/r1_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as f:
            d = json.load(f)
        return int(d["dram_bytes_read"] + d["dram_bytes_write"])
    except Exception:
        return None


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
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


# ---------------------------------------------------------------------------
# CPU port of the reference (oracle/c) -- baseline and --impl reference
# ---------------------------------------------------------------------------

def cpu_token_runner(gate, up, down):
    """Returns f(xh, xi) running one reference-style TL1 FFN token on the CPU port."""
    from oracle import c_oracle as CO
    g1, g2 = H // 2, I // 2

    def run(xh, xi, threads):
        qh, _ = CO.quantize(xh, 2)
        lut_h = CO.lut_tl1(qh, g1)
        CO.gemv_tl1(gate, lut_h, threads)
        CO.gemv_tl1(up, lut_h, threads)
        qi, _ = CO.quantize(xi, 2)
        lut_i = CO.lut_tl1(qi, g2)
        CO.gemv_tl1(down, lut_i, threads)

    return run


def cpu_baseline(gate, up, down, budget_s=12.0):
    from oracle import c_oracle as CO
    run = cpu_token_runner(gate, up, down)
    rng = np.random.default_rng(7)
    xh = rng.standard_normal(H).astype(np.float32)
    xi = rng.standard_normal(I).astype(np.float32)
    best = None
    ncpu = os.cpu_count() or 1
    for threads in sorted({1, CO.max_threads(), ncpu}):
        run(xh, xi, threads)  # warm
        n, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < budget_s / 2:
            run(xh, xi, threads)
            n += 1
        tps = n / (time.perf_counter() - t0)
        if best is None or tps > best[0]:
            best = (tps, threads, n)
    return {"value": round(best[0], 3), "unit": "tokens/s", "cores": best[1], "kind": "port",
            "sample": f"{best[2]} TL1 FFN tokens (gate+up+down, quantise+LUT+byte-table gather) "
                      f"on {best[1]} thread(s); best of threads in {{1, {ncpu}}}; host has {ncpu} CPUs"}


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

def make_tl1(tb, torch, rows, cols, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = torch.randn(rows, cols, generator=g, device="cuda", dtype=torch.float32) * 0.02
    m = tb.ternarize_weights(w, rows, cols)
    del w
    return tb.encode_tl1(m)


def shard_rows(p, tb, torch, r0, r1):
    """Column-parallel shard: rows [r0, r1) of a packed TL1 matrix (tp.column_shard)."""
    from paper_2410_16144_b200 import tp
    (data,) = tp.column_shard((p.data,), r0, r1)
    return tb.PackedTL1(rows=r1 - r0, cols=p.cols, padded_cols=p.padded_cols,
                        data=data.contiguous(), scale=p.scale, trusted=True)


def shard_cols(p, tb, torch, k0, k1):
    """Row-parallel shard: K-slice [k0, k1) as a byte slice (tp.row_shard)."""
    from paper_2410_16144_b200 import tp
    (data,), cols = tp.row_shard("tl1", (p.data,), p.cols, k0, k1)
    return tb.PackedTL1(rows=p.rows, cols=cols, padded_cols=cols + (cols & 1),
                        data=data.contiguous(), scale=p.scale, trusted=True)


def run_gpu(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2410_16144_b200 as tb

    dev = torch.device("cuda", _local_device(torch))
    torch.cuda.set_device(dev)
    # N > 1: independent decode replicas by default (each GPU holds the block
    # and decodes its own token stream -- no data-path collective, weak
    # scaling); --parallel tp shards the block instead (column-parallel
    # gate/up, row-parallel down + one NCCL int32 all-reduce per token).
    tp = world if args.parallel == "tp" else 1
    # ---- weights: NCOPY distinct seeded copies, TP-sharded
    plans = []
    gate_full_bytes = 0
    for c in range(NCOPY):
        gen = torch.Generator(device="cuda").manual_seed(1000 + c + (rank * 97 if tp == 1 else 0))
        mats = {}
        for name, rows, cols in (("gate", I, H), ("up", I, H), ("down", H, I)):
            w = torch.randn(rows, cols, generator=gen, device="cuda", dtype=torch.float32) * 0.02
            m = tb.ternarize_weights(w, rows, cols)
            del w
            if tp == 1:
                p = tb.encode_tl1(m)
            elif name in ("gate", "up"):
                per = rows // tp
                full = tb.encode_tl1(m)
                p = shard_rows(full, tb, torch, rank * per, (rank + 1) * per)
            else:
                per = cols // tp
                p = shard_cols(tb.encode_tl1(m), tb, torch, rank * per, (rank + 1) * per)
            p.tiled()
            mats[name] = p
        if c == 0:
            gate_full_bytes = mats["gate"].data.numel()
            host_copy = {k: v.data.cpu().numpy() for k, v in mats.items()} if tp == 1 else None
        plans.append({
            "gate": tb.GemvPlan(mats["gate"], out_dtype=torch.float32),
            "up": tb.GemvPlan(mats["up"], out_dtype=torch.float32),
            "down": tb.GemvPlan(mats["down"], out_dtype=(torch.float32 if tp == 1 else None),
                                want_acc=(tp > 1)),
            "mats": mats,
        })
        for p in mats.values():
            p._cache.pop("ref_dropped", None)
    torch.cuda.synchronize()

    gen = torch.Generator(device="cuda").manual_seed(77 + rank)
    XH = torch.randn(NX, H, generator=gen, device="cuda", dtype=torch.float32)
    XI = torch.randn(NX, I, generator=gen, device="cuda", dtype=torch.float32)
    # activation records: quantisation fused with the GEMV input layout; the
    # gate/up pair shares one record buffer (one quantisation per input vector)
    from paper_2410_16144_b200 import _lib as L
    rec_h = tb.ActRecords(L.TL1, 1, H)
    rec_i = tb.ActRecords(L.TL1, 1, I)
    out_down = torch.empty((1, H), dtype=torch.float32, device=dev)
    kloc = I // tp
    # row-parallel down (tp > 1): every rank quantises the full vector (same
    # per-token scale as the reference) and contracts its K-slice
    rec_i_loc = rec_i.chunk_slice(rank * kloc // 64, (rank + 1) * kloc // 64) if tp > 1 else rec_i
    # gate, up and down of one token in ONE grouped launch (independent GEMVs)
    for pl in plans:
        pl["batch"] = tb.GemvBatch([(pl["gate"], rec_h), (pl["up"], rec_h),
                                    (pl["down"], rec_i_loc)])
        if tp == 1:  # fused one-launch step: input 0 = x_h (gate, up), 1 = x_i (down)
            pl["step"] = tb.GemvStep([(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)], [H, I])
    tail = tb.StepGlue([])

    if tp == 1:
        # A decode step is ONE launch (tb_gemv_step_launch): every CTA quantises
        # the token's two input vectors itself, streams gate+up+down, and then
        # finalises the previous step's outputs (scales -> fp32 outputs).
        def step(i, prev):
            pl = plans[i % NCOPY]
            pl["step"].run([XH[i % NX], XI[i % NX]], prev=prev["step"] if prev else None)
            return pl

        def run_steps(n):
            prev = None
            for i in range(n):
                prev = step(i, prev)
            if prev is not None:
                prev["step"].finalize()  # the last step's outputs

        launches_per_step = 1
    else:
        # tp > 1: glue (finalise + quantise) and grouped GEMV launches; the down
        # projection's int32 partials are all-reduced before its rescale.
        glues = [tb.StepGlue([(XH[j:j + 1], rec_h), (XI[j:j + 1], rec_i)]) for j in range(NX)]

        def step(i, prev):
            pl = plans[i % NCOPY]
            glues[i % NX].retarget(prev["batch"] if prev is not None else None).run()
            pl["batch"].run(finalize=True)
            dist.all_reduce(pl["down"].acc, op=dist.ReduceOp.SUM)
            L.check(L.load().tb_scale_outputs(
                pl["down"].acc.data_ptr(), 1, H, float(pl["mats"]["down"].scale),
                rec_i.scales.data_ptr(), None, out_down.data_ptr(), L.stream_ptr()), "scale")
            return None

        def run_steps(n):
            for i in range(n):
                step(i, None)

        launches_per_step = 4  # glue + grouped GEMV + finalize + rescale (+ NCCL)

    # ---- warm-up (eager, also configures kernel attributes before capture)
    run_steps(max(args.warmup, NCOPY))
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps in one CUDA graph (NCCL
    #      collectives are capturable; a gloo functional check runs eagerly)
    capturable = world == 1 or dist.get_backend() == "nccl"
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    if capturable:
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                run_steps(args.steps)
        torch.cuda.synchronize()
        graph.replay()  # untimed replay (first replay uploads the graph)
        torch.cuda.synchronize()

        def timed_region():
            graph.replay()
    else:
        def timed_region():
            run_steps(args.steps)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        e0.record()
        timed_region()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps

    # ---- roofline: the dominant kernel timed alone, back-to-back over the
    #      rotating copies in a graph (tp1: the fused step kernel -- quantise +
    #      gate/up/down GEMV + previous finalize; tp>1: the grouped GEMV)
    R = 4 * NCOPY
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g2, stream=s):
            for i in range(R):
                if tp == 1:
                    plans[i % NCOPY]["step"].run([XH[i % NX], XI[i % NX]],
                                                 prev=plans[(i - 1) % NCOPY]["step"])
                else:
                    plans[i % NCOPY]["batch"].run(finalize=False)
    g2.replay()
    torch.cuda.synchronize()
    e0.record()
    g2.replay()
    e1.record()
    torch.cuda.synchronize()
    chain_ms = e0.elapsed_time(e1) / R
    # tp1: the timed region IS the step kernel chain (K step launches + one
    # trailing finalize), so the kernel's average launch duration over the
    # timed region is ms_per_step (conservative: the finalize is included);
    # the 24-launch chain above is reported beside it
    gemv_ms = ms_per_step if tp == 1 else chain_ms
    for pl in plans:  # finalise what is pending (resets the workspaces)
        if tp == 1:
            pl["step"].finalize()
        else:
            tail.retarget(pl["batch"]).run()
    torch.cuda.synchronize()
    rows_loc = I // tp
    gemv_bytes = (algo_bytes_gemv(rows_loc, H) * 2 + tl1_bytes(H, kloc) + kloc + 4 * H)
    peak, peak_kind = measured_peak()
    achieved = gemv_bytes / (gemv_ms * 1e-3) / 1e9

    replicas = world if tp == 1 else 1
    result = {
        "metric": METRIC, "value": round(replicas * 1000.0 / ms_per_step, 2), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
        "scaling": "weak" if replicas > 1 else "strong", "vs_baseline": None, "dtype": "i8",
        "data": "synthetic (seeded N(0,0.02) latent weights -> absmean ternary, N(0,1) activations)",
        "config": {"workload": "cfg1: TL1 FFN block, gate/up 4096->14336 + down 14336->4096, M=1",
                   "format": "TL1", "tokens_per_step": replicas,
                   "l2": f"{NCOPY} rotating weight copies ({NCOPY * 3 * gate_full_bytes / 1e6:.0f} MB "
                         "packed per rank) > 126 MB L2",
                   "parallelism": (f"dp{world} (independent decode replicas, no collective)"
                                   if replicas > 1 else "tp1") if tp == 1 else
                                  f"tp{tp} (col-parallel gate/up, "
                                  "row-parallel down + NCCL int32 all-reduce)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "frac_vs_nominal_8000": round(achieved / 8000.0, 4),
                     "traffic": measured_traffic() if tp == 1 else None,
                     "kernel": ("tgemv_kernel<TL1,1,fused> one-launch step: quantise x_h, x_i + "
                                "gate/up (14336x4096) + down (4096x14336) + previous finalize")
                               if tp == 1 else "tgemv_kernel<TL1,1> grouped gate+up+down",
                     "bytes_per_launch": gemv_bytes, "launch_us": round(gemv_ms * 1e3, 3),
                     "launch_us_source": ("timed region / K step launches (incl. the one trailing "
                                          "finalize)" if tp == 1 else
                                          f"{R}-launch graph of the grouped GEMV alone"),
                     "launch_us_chain24": round(chain_ms * 1e3, 3),
                     "peak_kind": f"{peak_kind} hbm_gbs (copy)"},
        "gpu_launches": launches_per_step * args.steps + (1 if tp == 1 else 0),
        "clocks": clk.summary(),
    }

    # ---- e2e through the public API with host buffers: every step copies its
    #      two f32 input vectors in from pinned host memory, runs, and copies
    #      its three fp32 output vectors back to pinned host memory
    if rank == 0 and not args.no_e2e and tp == 1:
        n_e2e = max(10, min(args.steps, 200))
        xh_h = torch.randn(NX, H).pin_memory()
        xi_h = torch.randn(NX, I).pin_memory()
        # (a) the serving form: n_e2e independent steps in one HostPipeline
        #     run (H2D / step kernels / D2H overlapped on three streams), the
        #     weights rotating over the NCOPY copies as in `value`
        # 400 steps per run: the first block's copy in and the last block's
        # copy back (not hidden behind kernels) amortise over the run
        n_pipe = 400
        pipe = tb.HostPipeline([[(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)]
                                for pl in plans], [H, I], steps=n_pipe)
        for i in range(n_pipe):
            pipe.inputs[0][i].copy_(xh_h[i % NX])
            pipe.inputs[1][i].copy_(xi_h[i % NX])
        for _ in range(3):
            pipe.run()
        reps = []
        for _ in range(5):
            t0 = time.perf_counter()
            pipe.run()
            reps.append(time.perf_counter() - t0)
        e2e_s = sorted(reps)[len(reps) // 2] / n_pipe
        result["e2e"] = {"value": round(1.0 / e2e_s, 2), "unit": "tokens/s",
                         "h2d_bytes_per_step": (H + I) * 4,
                         "d2h_bytes_per_step": (2 * I + H) * 4,
                         "steps": n_pipe,
                         "path": "tb.HostPipeline.run(): per step, pinned host f32 inputs -> H2D "
                                 "copy -> fused step kernel (PDL chain) -> D2H copy of the fp32 "
                                 "outputs to pinned host memory; copies and kernels on three "
                                 "streams in one CUDA graph; wall clock incl. the final sync "
                                 "(median of 5 runs)"}

        # (b) one token at a time, synchronous (latency-bound): HostStep
        hosts = [tb.HostStep([(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)], [H, I])
                 for pl in plans]

        def e2e_step(i):
            return hosts[i % NCOPY]([xh_h[i % NX], xi_h[i % NX]])

        for i in range(5):
            e2e_step(i)
        t0 = time.perf_counter()
        for i in range(n_e2e):
            e2e_step(i)
        sync_s = (time.perf_counter() - t0) / n_e2e
        result["e2e_sync"] = {"value": round(1.0 / sync_s, 2), "unit": "tokens/s",
                              "us_per_token": round(sync_s * 1e6, 2), "steps": n_e2e,
                              "path": "tb.HostStep: one token per call (H2D, fused step, "
                                      "finalize into mapped pinned memory, stream sync)"}

        # the reference-shaped per-call API (quantize_activations + gemv_parallel
        # per projection, float64 GemvResult.output to host)
        K = tb.KernelKind

        def api_step(i):
            mats = plans[i % NCOPY]["mats"]
            qa_h = tb.quantize_activations(xh_h[i % NX], pad_to=2)
            rg = tb.gemv_parallel(K.TL1, mats["gate"], qa_h)
            ru = tb.gemv_parallel(K.TL1, mats["up"], qa_h)
            qa_i = tb.quantize_activations(xi_h[i % NX], pad_to=2)
            rd = tb.gemv_parallel(K.TL1, mats["down"], qa_i)
            return rg.output.cpu(), ru.output.cpu(), rd.output.cpu()

        for i in range(3):
            api_step(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n_e2e):
            api_step(i)
        torch.cuda.synchronize()
        api_s = (time.perf_counter() - t0) / n_e2e
        result["e2e_reference_api"] = {
            "value": round(1.0 / api_s, 2), "unit": "tokens/s", "steps": n_e2e,
            "h2d_bytes_per_step": (H + I) * 4, "d2h_bytes_per_step": (2 * I + H) * 8,
            "path": "tb.quantize_activations + tb.gemv_parallel(TL1) x3 (reference call "
                    "pattern, bench.py:138-153), float64 outputs to host"}

    if rank == 0 and tp == 1 and not args.no_prefill:
        result["prefill"] = run_prefill(torch, tb)
    if rank == 0 and tp == 1 and args.stacks:
        result["stacks"] = {}
        for spec in args.stacks.split(","):
            if spec == "cfg0":
                result["stacks"][spec] = run_cfg0(torch, tb)
                continue
            name, fmt, m = spec.split(":")
            result["stacks"][spec] = run_stack(torch, tb, name, fmt, int(m))

    if rank == 0 and not args.no_cpu_baseline and tp == 1:
        result["cpu_baseline"] = cpu_baseline(host_copy["gate"], host_copy["up"],
                                              host_copy["down"], budget_s=args.cpu_budget)
    return result


def run_prefill(torch, tb, copies=2, reps=10):
    """BASELINE configs[3]: one Llama-3-8B-shaped layer of prefill GEMMs at
    M=512 (I2_S), q/k/v/o/gate/up on x_h and down on x_i, in ONE grouped
    tcgen05 launch (tb_gemm_batch); int8 TOPS = 2*M*sum(N*K) / time, against
    the cuBLASLt int8 throughput measured here (torch._int_mm, 8192^3)."""
    import ctypes as C

    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    M, KV = 512, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    xh = tb.quantize_tokens(torch.randn(M, H, generator=g, device="cuda"))
    xi = tb.quantize_tokens(torch.randn(M, I, generator=g, device="cuda"))
    tiled = {}
    for qa, k in ((xh, H), (xi, I)):
        t = torch.empty(lib.tb_gemm_act_bytes(M, k), dtype=torch.uint8, device="cuda")
        L.check(lib.tb_gemm_tile_act(qa.data.data_ptr(), M, qa.data.stride(0), k, t.data_ptr(),
                                     L.stream_ptr()), "gemm_tile_act")
        tiled[k] = (qa, t)
    shapes = [(H, H), (KV, H), (KV, H), (H, H), (I, H), (I, H), (H, I)]
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
            qa, t = tiled[k]
            d.tiled, d.rows, d.cols, d.act_tiled = main.data_ptr(), n, k, t.data_ptr()
            d.a_scale, d.w_scale, d.out32 = qa.scales.data_ptr(), float(p.scale), out.data_ptr()
            keep.append((p, main, out))
        layers.append((descs, keep))
    s = L.stream_ptr()

    def run(i):
        L.check(lib.tb_gemm_batch(L.I2S, len(shapes), C.cast(layers[i % copies][0], C.c_void_p),
                                  M, s), "gemm_batch")

    def timed(fn, n):
        fn(0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    ms = timed(run, reps)
    a = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda")
    bt = torch.randint(-127, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
    peak_ms = timed(lambda i: torch._int_mm(a, bt), 5)
    peak = 2 * 8192 ** 3 / (peak_ms * 1e-3) / 1e12
    tops = ops / (ms * 1e-3) / 1e12
    return {"workload": "cfg3: one Llama-3-8B-shaped layer (q,k,v,o,gate,up,down), M=512, I2_S, "
                        "one grouped tcgen05 kind::i8 launch",
            "tops": round(tops, 1), "us_per_layer": round(ms * 1e3, 1), "gop": round(ops / 1e9, 1),
            "peak_tops": round(peak, 1), "peak_kind": "cuBLASLt int8 torch._int_mm 8192^3, measured",
            "frac": round(tops / peak, 4),
            "frac_vs_nominal_4500": round(tops / 4500.0, 4)}


def run_stack(torch, tb, name, fmt, tokens=1, steps=10):
    """BASELINE configs 2 / 4: M-token decode through the whole layer stack,
    one launch per layer (M=1) or glue + grouped GEMV per layer (M > 1)."""
    from paper_2410_16144_b200.stack import STACKS, LayerStack
    cfg = STACKS[name]
    t0 = time.perf_counter()
    st = LayerStack(cfg, fmt=fmt, seed=11, tokens=tokens)
    build_s = time.perf_counter() - t0
    g = torch.Generator(device="cuda").manual_seed(99)
    L = st.nlayers
    if tokens == 1:
        XH = torch.randn(L, cfg["hidden"], generator=g, device="cuda")
        XI = torch.randn(L, cfg["inter"], generator=g, device="cuda")
        xh, xi = list(XH), list(XI)
        glues = None
    else:
        XH = torch.randn(L, tokens, cfg["hidden"], generator=g, device="cuda")
        XI = torch.randn(L, tokens, cfg["inter"], generator=g, device="cuda")
        xh = xi = None
        glues = st.make_glues(XH, XI)
    st.token_pass(xh, xi, glues)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            for _ in range(steps):
                st.token_pass(xh, xi, glues)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    peak, _ = measured_peak()
    gbs = st.algo_bytes / (ms * 1e-3) / 1e9
    out = {"workload": f"{name}: {L} layers, hidden {cfg['hidden']}, {fmt.upper()}, M={tokens}",
           "tokens_per_s": round(tokens * 1000.0 / ms, 1), "ms_per_token_pass": round(ms, 4),
           "algo_bytes_per_pass": int(st.algo_bytes), "hbm_gbs": round(gbs, 1),
           "frac": round(gbs / peak, 4), "launches_per_pass": L + 1 if tokens == 1 else 2 * L + 1,
           "build_s": round(build_s, 1)}
    del graph, st
    torch.cuda.empty_cache()
    return out


def run_cfg0(torch, tb, copies=32, steps=200):
    """BASELINE configs[0]: one I2_S GEMV, M=1, 4096 x 4096 -- one fused
    launch per token (quantise + GEMV + previous finalize), rotating over
    32 weight copies (134 MB > L2) in a CUDA graph."""
    n = k = 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    steps_obj = []
    for _ in range(copies):
        w = torch.randn(n, k, generator=g, device="cuda") * 0.02
        plan = tb.GemvPlan(tb.encode_i2s(tb.ternarize_weights(w, n, k)), out_dtype=torch.float32)
        steps_obj.append(tb.GemvStep([(plan, 0)], [k]))
        del w
    X = torch.randn(16, k, generator=g, device="cuda")

    def run(cnt):
        for i in range(cnt):
            steps_obj[i % copies].run([X[i % 16]], prev=steps_obj[(i - 1) % copies])
        steps_obj[(cnt - 1) % copies].finalize()

    run(copies)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            run(steps)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    algo = n * k // 4 + k + 4 * n
    peak, _ = measured_peak()
    return {"workload": "cfg0: I2_S GEMV M=1, 4096x4096, one fused launch per token",
            "tokens_per_s": round(1e6 / us, 1), "us_per_gemv": round(us, 3),
            "algo_bytes": algo, "hbm_gbs": round(algo / (us * 1e-6) / 1e9, 1),
            "frac": round(algo / (us * 1e-6) / 1e9 / peak, 4),
            "note": "4.2 MB per launch: launch/latency-bound, not bandwidth-bound"}


def run_reference(args):
    """--impl reference: the C port of the reference CPU kernels, all host threads."""
    import torch  # noqa: F401  (weights are generated with the same packer)
    from oracle import c_oracle as CO
    from oracle import ternpack_oracle as O

    rng = np.random.default_rng(1000)
    mats = {}
    for name, rows, cols in (("gate", I, H), ("up", I, H), ("down", H, I)):
        v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)  # ternary draw (bench.py:102)
        mats[name] = O.encode_tl1(v)
    run = cpu_token_runner(mats["gate"], mats["up"], mats["down"])
    threads = os.cpu_count() or 1
    xs = np.random.default_rng(7)
    XH = xs.standard_normal((NX, H)).astype(np.float32)
    XI = xs.standard_normal((NX, I)).astype(np.float32)
    for i in range(args.warmup):
        run(XH[i % NX], XI[i % NX], threads)
    t0 = time.perf_counter()
    for i in range(args.steps):
        run(XH[i % NX], XI[i % NX], threads)
    dt = (time.perf_counter() - t0) / args.steps
    v = round(1.0 / dt, 3)
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "i8",
        "data": "synthetic", "config": {"workload": "cfg1: TL1 FFN block, gate/up 4096->14336 + "
                                                    "down 14336->4096, M=1", "format": "TL1"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} timed TL1 FFN tokens, {threads} OpenMP threads, "
                                   f"C port of the reference byte-table kernels (oracle/c); "
                                   f"reference package itself is not shipped to the box"},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _local_device(torch):
    """LOCAL_RANK's GPU.  TB_BENCH_SHARE_GPU=1 folds ranks onto the visible
    GPUs -- a functional check of the tp > 1 code path on a 1-GPU box (with
    TB_BENCH_DIST_BACKEND=gloo), never a measurement."""
    lr = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("TB_BENCH_SHARE_GPU") == "1":
        lr %= torch.cuda.device_count()
    return lr


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--stacks", default="cfg0,cfg2:i2s:1,cfg2:tl2:1",
                    help="layer-stack decode lines, name:fmt:M comma list ('' = none); "
                         "e.g. cfg4:i2s:1,cfg4:i2s:8")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--parallel", default="dp", choices=["dp", "tp"],
                    help="N > 1: independent replicas (dp, default) or tensor parallel (tp)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(_local_device(torch))
        dist.init_process_group(os.environ.get("TB_BENCH_DIST_BACKEND", "nccl"))
    res = run_gpu(args, rank, world)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
