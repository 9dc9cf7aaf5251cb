"""Tensor-parallel LayerStack through the CUDA kernels.

One GPU is available, so the multi-rank path is exercised two ways, neither
of which runs kernels that wait on a kernel of another launch:

* ``tp.EmulatedGroup``: all ranks in one process; their steps are
  interleaved layer by layer and each layer's reduction is ONE launch over
  all ranks -- the peer-memory kernel's emulated form (``peer``) or a torch
  sum (``torch``);
* two real processes sharing the GPU over gloo (``TorchAllReduce``: the
  exchange runs on the host, eagerly).

Every tp degree must be bit-identical to tp=1 (integer partial sums are exact;
SPEC.md:333, kernels.py:181-186), and tp=1 is checked against the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import ternpack_oracle as O

pytestmark = pytest.mark.gpu

CFG = {"hidden": 512, "kv": 128, "inter": 1024, "layers": 3}


def _inputs(cfg, seed=8):
    g = torch.Generator(device="cuda").manual_seed(seed)
    L = cfg["layers"]
    return (torch.randn(L, cfg["hidden"], generator=g, device="cuda"),
            torch.randn(L, cfg["inter"], generator=g, device="cuda"))


def _full_outputs(st, li):
    """tp1: every projection's fp32 outputs of layer li (host)."""
    return {k: v.cpu().numpy() for k, v in st.outputs(li).items()}


def _gather(stacks, li):
    """Reassemble the full outputs of layer li from the ranks' shards."""
    res = {}
    for j, (name, rows, cols, src, kind, lo, hi) in enumerate(stacks[0].plan):
        if kind == "row":
            outs = [st.outputs(li)[name].cpu().numpy() for st in stacks]
            for o in outs[1:]:  # every rank holds the full reduced rows
                assert np.array_equal(o, outs[0]), name
            res[name] = outs[0]
        else:
            res[name] = np.concatenate([st.outputs(li)[name].cpu().numpy() for st in stacks])
    return res


@pytest.fixture(scope="module")
def tp1():
    from paper_2410_16144_b200.stack import LayerStack
    st = LayerStack(CFG, fmt="i2s", seed=4, tokens=1)
    XH, XI = _inputs(CFG)
    st.token_pass(list(XH), list(XI))
    torch.cuda.synchronize()
    return st, XH, XI


def test_tp1_stack_matches_oracle(tp1):
    import paper_2410_16144_b200 as tb
    st, XH, XI = tp1
    for li in range(CFG["layers"]):
        outs = _full_outputs(st, li)
        xs = [XH[li].cpu().numpy(), XI[li].cpu().numpy()]
        for plan, (name, rows, cols, src) in zip(st.layers[li], st.shapes):
            v = tb.decode_i2s(plan.p).values.cpu().numpy()
            q, s, _ = O.quantize(xs[src], 1)
            want = O.make_output(O.gemv_ref_int32(v, q), plan.p.scale, s).astype(np.float32)
            assert np.array_equal(outs[name], want), (li, name)


@pytest.mark.parametrize("world,mode", [(2, "peer"), (4, "peer"), (8, "peer"), (2, "torch"),
                                        (3, "peer")])
def test_emulated_tp_bit_identical(tp1, world, mode):
    from paper_2410_16144_b200 import tp as TP
    from paper_2410_16144_b200.stack import LayerStack
    st1, XH, XI = tp1
    grp = TP.EmulatedGroup(world, mode)
    stacks = [LayerStack(CFG, fmt="i2s", seed=4, tokens=1, tp_rank=r, tp_world=world,
                         collective=grp.member(r)) for r in range(world)]
    for rep in range(2):  # a second pass re-uses the epoch counters / flags
        grp.token_pass(list(XH), list(XI))
        torch.cuda.synchronize()
        for li in range(CFG["layers"]):
            got, want = _gather(stacks, li), _full_outputs(st1, li)
            for name in want:
                assert np.array_equal(got[name], want[name]), (world, mode, rep, li, name)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_rank(rank, world, port, q):
    import torch.distributed as dist

    from paper_2410_16144_b200 import tp as TP
    from paper_2410_16144_b200.stack import LayerStack
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = LayerStack(CFG, fmt="i2s", seed=4, tokens=1, tp_rank=rank, tp_world=world,
                        collective=TP.TorchAllReduce())
        XH, XI = _inputs(CFG)
        st.token_pass(list(XH), list(XI))
        torch.cuda.synchronize()
        outs = [{k: v.cpu().numpy() for k, v in st.outputs(li).items()}
                for li in range(CFG["layers"])]
        q.put((rank, outs, [s[4:] for s in st.plan]))
    finally:
        dist.destroy_process_group()


def test_gloo_two_processes_share_gpu(tp1):
    """Two real ranks (processes) on the one GPU, gloo all-reduce of the
    int32 partials (host side), CUDA kernels for everything else."""
    import torch.multiprocessing as mp
    st1 = tp1[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    for li in range(CFG["layers"]):
        want = _full_outputs(st1, li)
        for j, (name, rows, cols, src) in enumerate(st1.shapes):
            kind = res[0][2][j][0]
            if kind == "row":
                assert np.array_equal(res[0][1][li][name], want[name])
                assert np.array_equal(res[1][1][li][name], want[name])
            else:
                cat = np.concatenate([res[0][1][li][name], res[1][1][li][name]])
                assert np.array_equal(cat, want[name]), (li, name)
