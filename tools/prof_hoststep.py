"""Attribution of the one-token HostStep latency (bench cfg1 e2e_sync):
the full call, the host-side input copies alone, graph replay + sync alone,
the device time of the replayed graph (events around it), and a trivial
one-kernel graph's replay + sync as the launch/sync floor."""

import time

import numpy as np
import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_16144_b200 as tb  # noqa: E402


def mk(rows, cols, seed):
    rng = np.random.default_rng(seed)
    v = rng.integers(-1, 2, size=(rows, cols), dtype=np.int8)
    return tb.GemvPlan(tb.encode_tl1(tb.TernaryMatrix(rows, cols, v, 0.37)),
                       out_dtype=torch.float32)


def med(f, n=200):
    for _ in range(20):
        f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e6


def main():
    H, I = 4096, 14336
    ncopy = 6
    hosts = []
    for c in range(ncopy):
        g, u, d = mk(I, H, 3 * c), mk(I, H, 3 * c + 1), mk(H, I, 3 * c + 2)
        hosts.append(tb.HostStep([(g, 0), (u, 0), (d, 1)], [H, I]))
    xh = torch.randn(H).pin_memory()
    xi = torch.randn(I).pin_memory()
    k = [0]

    def full():
        hosts[k[0] % ncopy]([xh, xi])
        k[0] += 1

    def copies():
        h = hosts[k[0] % ncopy]
        for d_, s in zip(h.x_host, (xh, xi)):
            d_.copy_(s)
        k[0] += 1

    def replay():
        h = hosts[k[0] % ncopy]
        h._record.replay()
        h._stream.synchronize()
        k[0] += 1

    print(f"full call        {med(full):7.1f} us")
    print(f"input copies     {med(copies):7.1f} us")
    print(f"replay + sync    {med(replay):7.1f} us")
    # device time of the replayed graph
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ds = []
    for j in range(100):
        h = hosts[j % ncopy]
        with torch.cuda.stream(h._stream):
            torch.cuda._sleep(200000)  # keep the GPU busy while the CPU launches
        e0.record(h._stream)
        h._record.replay()
        e1.record(h._stream)
        e1.synchronize()
        ds.append(e0.elapsed_time(e1) * 1e3)
    print(f"graph device (GPU busy before)    {np.median(ds[10:]):7.1f} us")
    # trivial graph floor
    x = torch.zeros(16, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x.add_(1)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            x.add_(1)
    torch.cuda.synchronize()

    def triv():
        g.replay()
        torch.cuda.synchronize()
    print(f"trivial graph    {med(triv):7.1f} us")
    # step alone chained (what the steady-state kernel costs)
    ts = []
    for j in range(100):
        h = hosts[j % ncopy]
        with torch.cuda.stream(h._stream):
            torch.cuda._sleep(200000)
        e0.record(h._stream)
        with torch.cuda.stream(h._stream):
            h.step.run(h.x_dev)
        e1.record(h._stream)
        with torch.cuda.stream(h._stream):
            h.step.finalize()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"step kernel      {np.median(ts[10:]):7.1f} us (eager, isolated, GPU busy before)")


if __name__ == "__main__":
    main()



def chained_vs_isolated():
    """Device time of one step launch (+ finalize) with the GPU kept busy
    while the CPU launches: isolated (big CTAs) vs chain CTAs, and a chain of
    60 steps per launch."""
    H, I = 4096, 14336
    plans = [(mk(I, H, 1), 0), (mk(I, H, 2), 0), (mk(H, I, 3), 1)]
    x = [torch.randn(H, device="cuda"), torch.randn(I, device="cuda")]
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for iso in (True, False):
        st = tb.GemvStep(plans, [H, I], isolated=iso)
        ts = []
        for j in range(60):
            torch.cuda._sleep(200000)
            e0.record(s)
            st.run(x)
            st.finalize()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"isolated={iso}: step + finalize {np.median(ts[5:]):6.1f} us")
    a = tb.GemvStep(plans, [H, I])
    b = tb.GemvStep([(mk(I, H, 4), 0), (mk(I, H, 5), 0), (mk(H, I, 6), 1)], [H, I])
    torch.cuda._sleep(200000)
    e0.record(s)
    prev = None
    for j in range(60):
        cur = (a, b)[j % 2]
        cur.run(x, prev=prev)
        prev = cur
    prev.finalize()
    e1.record(s)
    e1.synchronize()
    print(f"chain of 60: {e0.elapsed_time(e1) * 1e3 / 60:6.1f} us per step (2 weight copies: L2-warm)")


if __name__ == "__main__":
    chained_vs_isolated()


def graph_pieces():
    """Device time of HostStep's pieces, issued eagerly behind a busy GPU
    with events between them: the copy-in kernel alone, the self-finalising
    step alone (inputs already on the device), both (the graph's content),
    and the copy engine's H2D copy for comparison."""
    from paper_2410_16144_b200 import _lib as L
    lib = L.load()
    H, I = 4096, 14336
    h = tb.HostStep([(mk(I, H, 1), 0), (mk(I, H, 2), 0), (mk(H, I, 3), 1)], [H, I])
    solo = tb.GemvStep(h.step.pairs, [H, I], flags=h.flags_host, isolated=True,
                       self_finalize=True)
    s = h._stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nb = h.x_host_all.numel() * 4

    def copy_in():
        L.check(lib.tb_copy_in(h.x_dev_all.data_ptr(), h.x_host_all.data_ptr(), nb,
                               L.stream_ptr()))

    pieces = {
        "copy_in kernel": copy_in,
        "copy engine H2D": lambda: h.x_dev_all.copy_(h.x_host_all, non_blocking=True),
        "step (self-fin, x on device)": lambda: solo.run(h.x_dev),
        "copy_in + step (x after wait)": h._issue,
    }
    with torch.cuda.stream(s):
        for name, f in pieces.items():
            ts = []
            for j in range(40):
                torch.cuda._sleep(300000)
                e0.record(s)
                f()
                e1.record(s)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            print(f"  {name:32s} {np.median(ts[5:]):6.1f} us")
    # replay + sync of graphs holding the pieces (the call's floor per piece)
    dev_pairs = [(mk(I, H, 1), 0), (mk(I, H, 2), 0), (mk(H, I, 3), 1)]
    solo_dev = tb.GemvStep(dev_pairs, [H, I], isolated=True, self_finalize=True)
    pieces["step (self-fin, outputs in HBM)"] = lambda: solo_dev.run(h.x_dev)
    cs = torch.cuda.Stream()
    for name in ("copy_in kernel", "step (self-fin, x on device)",
                 "step (self-fin, outputs in HBM)", "copy_in + step (x after wait)"):
        gr = torch.cuda.CUDAGraph()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            pieces[name]()
            with torch.cuda.graph(gr, stream=cs):
                pieces[name]()
        torch.cuda.synchronize()

        def rep():
            gr.replay()  # (on the CURRENT stream, not the capture stream)
            torch.cuda.synchronize()
        print(f"  graph [{name}] replay + sync {med(rep):6.1f} us")


if __name__ == "__main__":
    graph_pieces()
