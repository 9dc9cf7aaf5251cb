"""Where the reference-call-pattern e2e time goes (quantize_activations +
3 x gemv_parallel per token, host numpy in, .cpu() out)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_16144_b200 as tb
KK = tb.KernelKind
H, I = 4096, 14336
g = torch.Generator(device="cuda").manual_seed(1)
m = {}
for nm, r, c in (("gate", I, H), ("up", I, H), ("down", H, I)):
    w = torch.randn(r, c, generator=g, device="cuda") * 0.02
    m[nm] = tb.encode_tl1(tb.ternarize_weights(w, r, c))
rng = np.random.default_rng(0)
xh = [rng.standard_normal(H).astype(np.float32) for _ in range(8)]
xi = [rng.standard_normal(I).astype(np.float32) for _ in range(8)]
def tok(j):
    qh = tb.quantize_activations(xh[j % 8], pad_to=2)
    rg = tb.gemv_parallel(KK.TL1, m["gate"], qh)
    ru = tb.gemv_parallel(KK.TL1, m["up"], qh)
    rd = tb.gemv_parallel(KK.TL1, m["down"], tb.quantize_activations(xi[j % 8], pad_to=2))
    return rg.output.cpu(), ru.output.cpu(), rd.output.cpu()
for j in range(10): tok(j)
torch.cuda.synchronize()
t0 = time.perf_counter()
for j in range(50): tok(j)
print(f"{(time.perf_counter() - t0) / 50 * 1e6:.1f} us per token")
pr = cProfile.Profile(); pr.enable()
for j in range(50): tok(j)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
