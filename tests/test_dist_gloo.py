"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic.

The CUDA kernels need a GPU; here the per-shard work is done by the float64
oracle, which is enough to check what the multi-GPU path adds: the sharding
covers every unit exactly once, max-over-ranks timing, and that all-reducing
the per-shard BCA weight gradients gives the full-batch dw (Eq. 5 is linear
in the tokens), while dx and the transforms stay shard-local.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_01385_b200 import dist as D


def test_shard_range_partitions():
    for total in [0, 1, 7, 16384, 2 ** 20 + 3]:
        for world in [1, 2, 3, 4, 8]:
            spans = [D.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, _) in zip(spans, spans[1:]):
                assert b == c and b >= a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as o
        from paper_2511_01385_b200 import synth

        T, p, qq = 12, 8, 2
        x, w, g = synth.bca_inputs(T, qq * p, qq * p, p, seed=5, dtype="f32")
        lo, hi = D.shard_range(T, rank, world)
        dx, dw = o.bca_bwd(x[lo:hi].double().numpy(), w.double().numpy(), g[lo:hi].double().numpy())
        dw_t = torch.from_numpy(dw).float()
        D.allreduce_dw(dw_t)
        t_max = D.max_over_ranks(float(rank + 1))
        # transforms shard with no collective: each rank's rows equal the full-batch rows
        xs = synth.randn((10, 16), seed=9)
        lo2, hi2 = D.shard_range(10, rank, world)
        fwd_shard = o.rdfft_fwd(xs[lo2:hi2].double().numpy())
        q.put((rank, lo, hi, dx, dw_t.numpy(), t_max, lo2, hi2, fwd_shard))
    finally:
        dist.destroy_process_group()


def test_two_rank_bca_dw_allreduce_and_sharding():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])

    import oracle as o
    from paper_2511_01385_b200 import synth

    T, p, qq = 12, 8, 2
    x, w, g = synth.bca_inputs(T, qq * p, qq * p, p, seed=5, dtype="f32")
    dx_full, dw_full = o.bca_bwd(x.double().numpy(), w.double().numpy(), g.double().numpy())
    for rank, lo, hi, dx, dw, t_max, lo2, hi2, fwd_shard in res:
        np.testing.assert_allclose(dx, dx_full[lo:hi], atol=1e-12)      # dx is shard-local
        np.testing.assert_allclose(dw, dw_full, rtol=1e-5, atol=1e-5)  # all-reduced dw == full-batch dw
        assert t_max == 2.0                                             # max over ranks
        xs = synth.randn((10, 16), seed=9).double().numpy()
        np.testing.assert_allclose(fwd_shard, o.rdfft_fwd(xs)[lo2:hi2], atol=1e-12)
    assert res[0][2] == res[1][1]  # token shards are contiguous and disjoint


def test_chunked_generator_identical_for_any_sharding():
    """configs[4] inputs (SURVEY §8(d) cfg 5): 64 fixed seeded chunks, so the global data a rank's
    shard sees does not depend on how many ranks share the batch."""
    from paper_2511_01385_b200 import synth

    total, row = 1000, (8,)
    full = synth.randn_rows(total, row, 0, total, seed=3, dtype="f32", chunks=64)
    assert full.shape == (total, 8)
    for world in (1, 2, 3, 8):
        parts = [synth.randn_rows(total, row, *D.shard_range(total, r, world), seed=3, dtype="f32", chunks=64)
                 for r in range(world)]
        assert torch.equal(torch.cat(parts), full)
    # pieces are distinct streams (seed + c), not one stream cut up
    lo, hi = synth.chunk_range(total, 1, 64)
    assert torch.equal(full[lo:hi], synth.randn((hi - lo,) + row, seed=4, dtype="f32"))
