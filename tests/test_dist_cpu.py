"""world_size-2 gloo tests of the token-sharding host logic (no GPU): slices tile the batch,
max-over-ranks timing, aggregate throughput, and that gathering per-rank results of a
row-independent computation reproduces the unsharded result bit for bit — here with the
oracle's per-token quantizer standing in for the kernels (same row independence)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2404_00456_b200 import dist as qd


def test_shard_bounds_tile_exactly():
    for total in (1, 7, 131072, 131073):
        for world in (1, 2, 4, 8):
            spans = [qd.shard_bounds(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        qd.shard_bounds(10, 2, 2)


def test_aggregate_throughput():
    assert qd.aggregate_throughput(131072, 100.0, 8) == pytest.approx(8 * 131072 / 0.1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import quant as oquant
        total, k = 37, 64
        rng = np.random.default_rng(0)
        x = rng.standard_normal((total, k)) * 3
        r0, r1 = qd.shard_bounds(total, world, rank)
        codes, scale = oquant.quantize_sym_rows(x[r0:r1])
        packed = torch.from_numpy(oquant.pack_int4(codes))
        gathered = qd.gather_rows(packed, total)
        g_scale = qd.gather_rows(torch.from_numpy(scale), total)
        ms = qd.max_over_ranks(10.0 + rank)
        if rank == 0:
            full_codes, full_scale = oquant.quantize_sym_rows(x)
            out["equal"] = bool(torch.equal(gathered, torch.from_numpy(oquant.pack_int4(full_codes))))
            out["scale_equal"] = bool(torch.equal(g_scale, torch.from_numpy(full_scale)))
            out["ms"] = ms
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_gather_bitwise():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["equal"] and out["scale_equal"]
    assert out["ms"] == 11.0
