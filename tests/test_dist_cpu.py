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


# ---------------------------------------------------------------- bench.py's multi-GPU path

def _bench():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_bench_plan_shard_strong_and_weak():
    b = _bench()
    # strong scaling: config 5 at G = 8 -> 16384 tokens per GPU, 8 sequences each
    spans = [b.plan_shard(131072, 8, r, "strong") for r in range(8)]
    assert all(t == 16384 and job == 131072 for _, _, t, job in spans)
    assert [r0 for r0, _, _, _ in spans] == [16384 * r for r in range(8)]
    assert all(r0 % 2048 == 0 for r0, _, _, _ in spans)  # shards are whole sequences
    # weak scaling: every rank the whole batch
    assert b.plan_shard(131072, 4, 3, "weak") == (0, 131072, 131072, 4 * 131072)


def test_bench_torchrun_cmd():
    b = _bench()
    cmd = b.torchrun_cmd(4, ["--steps", "3"], 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[cmd.index("--master-port") + 1] == "29511"
    assert cmd[-3].endswith("bench.py") and cmd[-2:] == ["--steps", "3"]


def _bench_worker(rank, world, port, out):
    """One rank of bench.py's strong-scaling path on CPU: plan_shard -> make_inputs(rows=...) ->
    a row-independent, position-dependent stand-in step (the oracle's RMSNorm-quantize and RoPE at
    positions (row_offset + t) % seq_len, like DecoderLayerStep) -> dist.gather_and_compare
    against rank 0's unsharded run."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import glue as oglue
        from oracle import quant as oquant
        from synth.inputs import LayerShapes
        b = _bench()
        S = LayerShapes("tiny", 256, 512, 2, 1)
        total, seq_len = 5 * 16, 16
        r0, r1, T, job = b.plan_shard(total, world, rank, "strong")

        def stand_in(inp, row_offset):
            x = inp["x"].numpy().astype(np.float64)
            c, s = oquant.quantize_sym_rows(oglue.rmsnorm(x))
            pos = (row_offset + np.arange(x.shape[0])) % seq_len
            r = oglue.rope(inp["attn_out"].numpy().astype(np.float64).reshape(x.shape[0], 2, 128), pos)
            return {"codes": torch.from_numpy(oquant.pack_int4(c)), "scale": torch.from_numpy(s),
                    "rope": torch.from_numpy(r.astype(np.float16))}

        local = stand_in(b.make_inputs(total, "cpu", rank, "chain", S, rows=(r0, r1)), r0)
        ref = None
        if rank == 0:
            ref = stand_in(b.make_inputs(total, "cpu", 0, "chain", S, rows=(0, total)), 0)
        res = qd.gather_and_compare(local, total, ref)
        if rank == 0:
            out.update(res)
            out["T"] = T
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bench_strong_scaling_gather_bitwise():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bench_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out["T"] == 40
    assert out["codes"] and out["scale"] and out["rope"]


def test_gather_and_compare_detects_a_flipped_bit():
    # world 1 (no process group): gather is the identity; one changed bit is reported
    a = torch.arange(12, dtype=torch.float16).view(4, 3)
    b = a.clone()
    assert qd.gather_and_compare({"y": a}, 4, {"y": b}) == {"y": True}
    b.view(torch.int16)[2, 1] ^= 1
    assert qd.gather_and_compare({"y": a}, 4, {"y": b}) == {"y": False}
