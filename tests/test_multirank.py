"""World-size-2 gloo tests of the multi-GPU layer path.

Each rank builds and evaluates only its neuron shard of every layer (the same
split the GPU contexts use, csrc/scheduler.cpp run_layer) on the clear-bit
backend, then the shards are all-gathered with paper_1906_00148_b200.parallel
(the helper bench.py uses over NCCL) before the next layer.  The gathered
config-3 logits must equal both the world-1 evaluation and the plaintext
network; no rank may write outside its shard.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import she_inputs as si
from oracle import network as net
from paper_1906_00148_b200 import build, parallel, she


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _config3_inputs():
    cfg = 3
    px = si.pixels(cfg, (28, 28, 1)).astype(np.int64)
    w1 = si.log_quant_weights(cfg, (5, 5, 5, 1), layer=0)
    w2 = si.log_quant_weights(cfg, (100, 720), layer=1)
    w3 = si.log_quant_weights(cfg, (10, 100), layer=2)
    return px, w1, w2, w3


def _layer(fn, words, width, rank, world):
    """Run one clear layer on this rank's shard, check it wrote only its shard,
    and all-gather the words (uint8 bits -> int32 tensor for the collective)."""
    out = fn(rank, world)
    lo, hi, _ = parallel.shard(words, rank, world)
    flat = out.reshape(words, width)
    assert not flat[:lo].any() and not flat[hi:].any(), "rank wrote outside its shard"
    buf = torch.zeros((parallel.padded_words(words, world), width), dtype=torch.int32)
    buf[:words] = torch.from_numpy(flat.astype(np.int32))
    return parallel.gather_shards(buf, words, rank, world).numpy().astype(np.uint8)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        px, w1, w2, w3 = _config3_inputs()
        wa = she.conv_width(28, 28, 1, 8, False, w1, 2, 0, 16, relu=True)
        wb = she.fc_width(720, wa, False, w2, 16, relu=True)
        wc = she.fc_width(100, wb, False, w3, 16)
        h1 = _layer(lambda r, w: she.clear_conv_shift_acc(net.bits_of(px, 8), 28, 28, 1, 8, False,
                                                          w1, 2, 0, 16, relu=True, rank=r,
                                                          world=w)[0], 720, wa, rank, world)
        h2 = _layer(lambda r, w: she.clear_fc_shift_acc(h1.reshape(-1), 720, wa, False, w2, 16,
                                                        relu=True, rank=r, world=w)[0],
                    100, wb, rank, world)
        lo = _layer(lambda r, w: she.clear_fc_shift_acc(h2.reshape(-1), 100, wb, False, w3, 16,
                                                        rank=r, world=w)[0], 10, wc, rank, world)
        q.put((rank, net.value_of(lo, signed=True).tolist()))
    finally:
        dist.destroy_process_group()


def test_config3_two_ranks_gloo_equals_plaintext_network():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    px, w1, w2, w3 = _config3_inputs()
    want = net.config3(px, w1, w2, w3).tolist()
    assert res[0] == res[1] == want


def test_shard_split_matches_the_scheduler():
    """parallel.shard is the split csrc/scheduler.cpp run_layer uses: the clear
    backend with (rank, world) writes exactly those words."""
    rng = np.random.default_rng(2)
    x = rng.integers(0, 256, 11)
    wq = si.log_quant_weights(2, (7, 11), layer=7)
    full, w, _ = she.clear_fc_shift_acc(net.bits_of(x, 8).ravel(), 11, 8, False, wq, 16)
    for world in (1, 2, 3, 4, 8):
        got = np.zeros_like(full)
        for rank in range(world):
            part, _, _ = she.clear_fc_shift_acc(net.bits_of(x, 8).ravel(), 11, 8, False, wq, 16,
                                                rank=rank, world=world)
            lo, hi, _ = parallel.shard(7, rank, world)
            assert not part[:lo].any() and not part[hi:].any()
            got[lo:hi] = part[lo:hi]
        assert np.array_equal(got, full), world
