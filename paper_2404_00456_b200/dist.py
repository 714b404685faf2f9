"""Multi-GPU plumbing for token-sharded prefill (one process per GPU, torch.distributed).

The hot path has no collective: every step is row-independent, so each rank
processes its own token slice with the full replicated INT4 weights.  Strong scaling (§8e,
BASELINE config 3/5): the fixed 64 x 2048-token batch is split into contiguous row shards,
GPU g taking sequences [g*64/G, (g+1)*64/G).  The only communication is outside the timed
region:
  * `max_over_ranks` — the step time every rank reports is the max over ranks;
  * `gather_rows` — verification gather of per-rank outputs (NCCL all_gather over
    NVLink on GPUs, gloo in the CPU tests), to check that a sharded run equals the
    unsharded one bit for bit.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced token slice [r0, r1) of `total` rows for `rank` of `world`
    (GPU g takes sequences [g*64/G, (g+1)*64/G))."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return total * rank // world, total * (rank + 1) // world


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. the timed milliseconds) across the job."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(tokens_per_rank: int, ms_per_step: float, world: int) -> float:
    """Whole-job tokens/s: all ranks' tokens divided by the slowest rank's step time."""
    return tokens_per_rank * world / (ms_per_step * 1e-3)


def gather_rows(local: torch.Tensor, total_rows: int) -> torch.Tensor:
    """All-gather row slices produced by `shard_bounds` back into the full [total_rows, ...]
    tensor (verification only; padded to equal sizes for the collective)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    sizes = [shard_bounds(total_rows, world, r) for r in range(world)]
    pad = max(b - a for a, b in sizes)
    buf = torch.zeros((pad,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return torch.cat([o[: b - a] for o, (a, b) in zip(outs, sizes)], 0)


def shard_plan(total: int, world: int) -> list[tuple[int, int]]:
    """Every rank's [r0, r1) (shard_bounds for ranks 0..world-1)."""
    return [shard_bounds(total, world, r) for r in range(world)]


def gather_and_compare(local: dict, total_rows: int, reference=None) -> dict:
    """Verification (outside the timed region): all-gather every per-rank row shard in `local`
    (name -> tensor whose first dim is this rank's rows) into the full batch, then, on the
    ranks holding `reference` (name -> full tensor of an unsharded run, or None), compare
    bitwise.  Returns {name: True/False} on ranks with a reference, {} elsewhere.  Collective:
    every rank must call it with the same names in the same order."""
    result = {}
    for name in sorted(local):
        full = gather_rows(local[name].contiguous(), total_rows)
        if reference is not None:
            ref = reference[name].contiguous()
            result[name] = bool(full.shape == ref.shape and full.dtype == ref.dtype
                                and torch.equal(_bits(full), _bits(ref.to(full.device))))
    return result


def _bits(t: torch.Tensor) -> torch.Tensor:
    """Byte view (bitwise comparison: NaN payloads and signed zeros count)."""
    return t.reshape(-1).view(torch.uint8)
