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


def gate_batch_sharded(ctx, ops, a, b, c, out, rank: int, world: int, stream=None, group=None):
    """Config-1-style gate batch split across ranks (strong scaling, SURVEY.md
    §8(e)): rank r evaluates gates [r*per, min(count, (r+1)*per)) of the batch
    (per = ceil(count / world)) with she_gate_batch_ops and the output LWEs
    are all-gathered into `out` (device, padded_words(count, world) rows;
    rows [0, count) are the batch's outputs).  a, b, c, ops: the whole batch
    (device; each rank reads only its shard).  Returns out[:count]."""
    from . import she
    count = a.shape[0]
    lo, hi, _ = shard(count, rank, world)
    if hi > lo:
        she.she_gate_batch_ops(ctx, ops[lo:hi], a[lo:hi], b[lo:hi], c[lo:hi], out[lo:hi], stream)
    return gather_shards(out, count, rank, world, group)


def gate_batch_sharded_host(ctx, ops, a, b, c, out, rank: int, world: int, stage, group=None):
    """The end-to-end multi-GPU call: HOST inputs (pinned numpy arrays of the
    whole batch), each rank copies only its shard to the device, evaluates it,
    the shards are all-gathered on the devices, and the full result is copied
    back into the host array `out` (count x stride).  `stage` holds the
    device buffers (dict from make_stage).  Synchronous."""
    import torch
    count = a.shape[0]
    lo, hi, _ = shard(count, rank, world)
    d_ops, d_in, d_out = stage["ops"], stage["in"], stage["out"]
    d_ops[lo:hi].copy_(torch.from_numpy(ops[lo:hi]), non_blocking=True)
    for j, h in enumerate((a, b, c)):
        d_in[j][lo:hi].copy_(torch.from_numpy(h[lo:hi].view("int32")), non_blocking=True)
    gate_batch_sharded(ctx, d_ops, d_in[0], d_in[1], d_in[2], d_out, rank, world, group=group)
    torch.from_numpy(out.view("int32")).copy_(d_out[:count])
    torch.cuda.synchronize()
    return out


def make_stage(count: int, stride: int, world: int, device="cuda"):
    """Device buffers of gate_batch_sharded_host for a batch of `count` gates."""
    import torch
    rows = padded_words(count, world)
    return {"ops": torch.zeros(count, dtype=torch.uint8, device=device),
            "in": [torch.zeros((count, stride), dtype=torch.int32, device=device) for _ in range(3)],
            "out": torch.zeros((rows, stride), dtype=torch.int32, device=device)}


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
