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


def test_peer_allreduce_watchdog():
    """A peer that never signals must not hang the GPU: the kernel's wait
    gives up after its 4 s watchdog, records the peer in ctrl[2], and later
    launches do not wait again (the host reads the mask and falls back)."""
    import ctypes as C
    import time

    from paper_2410_16144_b200 import _lib as L
    from paper_2410_16144_b200 import tp as TP
    lib = L.load()
    n = 64
    parts = [torch.arange(n, dtype=torch.int32, device="cuda") * (r + 1) for r in range(2)]
    flags = [torch.zeros(8, dtype=torch.int32, device="cuda") for _ in range(2)]
    ctrl = torch.zeros(4, dtype=torch.int32, device="cuda")
    a_scale = torch.ones(1, dtype=torch.float64, device="cuda")
    out = torch.zeros(n, dtype=torch.float32, device="cuda")
    seg = (L.RowparSeg * 1)()
    seg[0].off, seg[0].n, seg[0].w_scale = 0, n, 1.0
    seg[0].a_scale, seg[0].out32, seg[0].acc_out = a_scale.data_ptr(), out.data_ptr(), None
    pa = (C.c_void_p * 2)(*[p.data_ptr() for p in parts])
    fa = (C.c_void_p * 2)(*[f.data_ptr() for f in flags])

    def launch():
        L.check(lib.tb_rowpar_allreduce(2, 0, pa, fa, ctrl.data_ptr(), 0, 1,
                                        C.cast(seg, C.c_void_p), 0, L.stream_ptr()), "ar")
        torch.cuda.synchronize()

    t0 = time.perf_counter()
    launch()  # rank 1 is silent: rank 0's wait on flags[0][1] times out
    dt = time.perf_counter() - t0
    assert 3.0 < dt < 8.0, dt
    assert int(ctrl[2].item()) == 0b10  # the silent peer
    t0 = time.perf_counter()
    launch()  # sticky: no second wait
    assert time.perf_counter() - t0 < 1.0
    # with the peer's signal present (what rank 1's launch stores) the same
    # launch completes at once and sums both ranks' partials
    ctrl.zero_()
    flags[0][1] = 1  # epoch 1 from rank 1
    launch()
    assert int(ctrl[2].item()) == 0 and int(ctrl[0].item()) == 1
    assert np.array_equal(out.cpu().numpy(), (np.arange(n) * 3).astype(np.float32))
    assert TP is not None


def _ipc_owner(port_q, done_q):
    import ctypes as C

    from paper_2410_16144_b200 import _lib as L
    from paper_2410_16144_b200 import tp as TP
    torch.cuda.set_device(0)
    lib = L.load()
    t = TP.sym_tensor(4096, "i4")
    t.copy_(torch.arange(4096, dtype=torch.int32, device="cuda") * 7 - 3)
    torch.cuda.synchronize()
    h = (C.c_uint8 * lib.tb_ipc_handle_bytes())()
    L.check(lib.tb_ipc_get_handle(t.data_ptr(), h), "get")
    port_q.put(bytes(h))
    assert done_q.get(timeout=120) == "read"
    # the reader wrote through its mapping: visible here
    torch.cuda.synchronize()
    port_q.put(int(t[5].item()))


def test_cuda_ipc_handles_between_processes():
    """tb_sym_alloc / tb_ipc_get_handle / tb_ipc_open / tb_ipc_close: a second
    process maps the owner's buffer (what PeerAllReduce.bind does for every
    peer) and reads / writes it.  No kernel of one process waits on the other."""
    import ctypes as C

    import torch.multiprocessing as mp

    from paper_2410_16144_b200 import _lib as L
    ctx = mp.get_context("spawn")
    hq, dq = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_ipc_owner, args=(hq, dq))
    p.start()
    try:
        h = hq.get(timeout=300)
        lib = L.load()
        torch.cuda.set_device(0)
        torch.zeros(1, device="cuda")
        ptr = C.c_void_p()
        L.check(lib.tb_ipc_open((C.c_uint8 * len(h)).from_buffer_copy(h), C.byref(ptr)), "open")

        class _View:
            __cuda_array_interface__ = {"shape": (4096,), "typestr": "<i4",
                                        "data": (ptr.value, False), "version": 2}
        v = torch.as_tensor(_View(), device="cuda")
        want = np.arange(4096, dtype=np.int32) * 7 - 3
        assert np.array_equal(v.cpu().numpy(), want)
        v[5] = 12345
        torch.cuda.synchronize()
        del v
        L.check(lib.tb_ipc_close(ptr.value), "close")
        dq.put("read")
        assert hq.get(timeout=120) == 12345
    finally:
        p.join(timeout=60)
    assert p.exitcode == 0
