"""Multi-GPU plumbing of the layer path.

A context created with (rank, world) computes only its contiguous share of a
layer's output words: neurons [r*per, min(M, (r+1)*per)) with per = ceil(M/W)
(the split of run_layer in csrc/scheduler.cpp, so no wire of a neuron's adder
tree crosses ranks).  Between layers the shards are all-gathered over the
process group (NCCL on the GPUs; gloo in the CPU tests).  This module holds
only that host-side bookkeeping; every gate runs in libshe.so.
"""
from __future__ import annotations


def shard(words: int, rank: int, world: int) -> tuple[int, int, int]:
    """(lo, hi, per): the output words rank `rank` of `world` computes."""
    per = -(-words // world)
    lo = min(words, per * rank)
    return lo, min(words, lo + per), per


def padded_words(words: int, world: int) -> int:
    """Rows of a gather buffer: world equal chunks of ceil(words / world)."""
    return -(-words // world) * world


def gather_shards(buf, words: int, rank: int, world: int, group=None):
    """All-gather the per-rank chunks of `buf` (leading dim padded_words(words,
    world); rank r's words in rows [r*per, (r+1)*per)) in place; returns
    buf[:words].  A no-op for world == 1."""
    if world == 1:
        return buf[:words]
    import torch.distributed as dist
    _, _, per = shard(words, rank, world)
    if buf.is_cuda and dist.get_backend(group) == "gloo":  # CPU staging (functional tests)
        host = buf.cpu()
        gather_shards(host, words, rank, world, group)
        buf.copy_(host)
        return buf[:words]
    parts = list(buf.split(per, dim=0))
    mine = parts[rank].clone()
    if buf.is_cuda and buf.is_contiguous():
        # one NCCL all-gather straight into the (contiguous) gather buffer
        dist.all_gather_into_tensor(buf, mine, group=group)
    else:
        dist.all_gather(parts, mine, group=group)
    return buf[:words]


def max_over_ranks(values, world: int):
    """Element-wise max over ranks of a list of floats (device timings are
    reported as the max over ranks).  NCCL reduces on the GPU, gloo on the CPU."""
    if world == 1:
        return list(values)
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]
