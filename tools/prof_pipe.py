"""HostPipeline attribution (cfg1 block): copies on/off, slots, steps per graph.

    python tools/prof_pipe.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_16144_b200 as tb  # noqa: E402

H, I, NCOPY = 4096, 14336, 6


def main():
    plans = []
    for c in range(NCOPY):
        gen = torch.Generator(device="cuda").manual_seed(1000 + c)
        pl = {}
        for name, rows, cols in (("gate", I, H), ("up", I, H), ("down", H, I)):
            w = torch.randn(rows, cols, generator=gen, device="cuda") * 0.02
            pl[name] = tb.GemvPlan(tb.encode_tl1(tb.ternarize_weights(w, rows, cols)))
        plans.append(pl)
    slots = [[(pl["gate"], 0), (pl["up"], 0), (pl["down"], 1)] for pl in plans]
    for T, blk, copies in ((400, 16, (True, True)), (400, 32, (True, True)),
                           (400, 16, (False, False)), (100, 16, (True, True))):
        pipe = tb.HostPipeline(slots, [H, I], steps=T, block=blk, _copies=copies)
        pipe.inputs[0].normal_()
        pipe.inputs[1].normal_()
        pipe._x_dev.normal_()  # copies off: the device inputs stay finite
        for _ in range(3):
            pipe.run()
        reps = []
        for _ in range(7):
            t0 = time.perf_counter()
            pipe.run()
            reps.append(time.perf_counter() - t0)
        # device time of the graph alone
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(pipe._stream):
            e0.record()
            pipe._graph.replay()
            e1.record()
        torch.cuda.synchronize()
        print(f"T={T} block={blk} copies={copies}: wall {sorted(reps)[3] / T * 1e6:.2f} us/step, "
              f"device {e0.elapsed_time(e1) * 1e3 / T:.2f} us/step", flush=True)


if __name__ == "__main__":
    main()
