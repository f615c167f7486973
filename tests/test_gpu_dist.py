"""GPU, world size 2 (gloo, both ranks on cuda:0): the batch-sharded hot path of configs[4]
(SURVEY §8(e)).  Rows transformed on a shard are BIT-identical to the same rows of the 1-rank run
(the kernel configuration depends on (n, dtype) only, never on the batch), and the all-reduced
per-shard BCA weight gradient equals the 1-rank dw within the fp32 gate (dw is a sum over tokens,
Eq. 5; only the order of fp32 additions differs)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, TOTAL = 1024, 3 * 4096 + 77          # several tiles per rank and a ragged split
T, D, P = 2 * 1184 + 9, 4096, 1024      # LLaMA-shape BCA: > 1 tile per CTA on every rank


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _work(lo, hi, tlo, thi, dtype):
    from paper_2511_01385_b200 import rdfft as R
    from paper_2511_01385_b200 import synth

    x = synth.randn_rows(TOTAL, (N,), lo, hi, seed=11, dtype=dtype, device="cuda")
    h = synth.randn((1, N), seed=12, dtype=dtype, device="cuda")
    R.rdfft_fwd(x)
    f = x.clone()
    R.rdfft_packed_mul(x, h)
    R.rdfft_inv(x)
    xa = synth.randn_rows(T, (D,), tlo, thi, seed=13, dtype=dtype, device="cuda")
    w = synth.randn((D // P, D // P, P), seed=14, dtype=dtype, device="cuda", std=D ** -0.5)
    g = synth.randn_rows(T, (D,), tlo, thi, seed=15, dtype=dtype, device="cuda")
    y = R.bca_fwd(xa, w)
    dx, dw = R.bca_bwd(xa, w, g)
    torch.cuda.synchronize()
    return f.cpu(), x.cpu(), y.cpu(), dx.cpu(), dw


def _worker(rank, world, port, dtype, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2511_01385_b200 import dist as Dd

        lo, hi = Dd.shard_range(TOTAL, rank, world)
        tlo, thi = Dd.shard_range(T, rank, world)
        f, x, y, dx, dw = _work(lo, hi, tlo, thi, dtype)
        Dd.allreduce_dw(dw)  # gloo all-reduce of the CUDA fp32 dw (NCCL on the 8-GPU box)
        # numpy copies: pickled by value (torch CPU tensors would travel as shared-memory handles
        # that die with this process)
        q.put((rank, lo, hi, tlo, thi, *(t.float().numpy() if t.dtype == torch.bfloat16 else t.numpy()
                                         for t in (f, x, y, dx, dw.cpu()))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_two_rank_shards_bit_identical(cuda_device, dtype):
    from paper_2511_01385_b200 import build

    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    one = _work(0, TOTAL, 0, T, dtype)  # the 1-rank run
    f1, x1, y1, dx1 = (t.float().numpy() for t in one[:4])
    dw1 = one[4].cpu().double().numpy()
    for rank, lo, hi, tlo, thi, f, x, y, dx, dw in res:
        # bf16 values widen exactly to fp32, so equality of the widened arrays is bit-equality
        assert np.array_equal(f, f1[lo:hi])      # forward spectra: bit-identical rows
        assert np.array_equal(x, x1[lo:hi])      # fwd -> packed_mul -> inv: bit-identical rows
        assert np.array_equal(y, y1[tlo:thi])    # BCA forward per token
        assert np.array_equal(dx, dx1[tlo:thi])  # BCA dx per token (shard-local)
        assert np.linalg.norm(dw - dw1) / np.linalg.norm(dw1) <= 1e-5  # all-reduced vs 1-rank dw
    assert res[0][2] == res[1][1] and res[0][4] == res[1][3]  # contiguous, disjoint shards
