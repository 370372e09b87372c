"""The multi-GPU path on a GPU: world-2 rank processes over gloo on one device
(the NCCL run needs 2 GPUs, which this test box does not
have — gloo stages the all-gathers through the host, the device work and the
sharding are the same).

  * config 1 strong-scaled (parallel.gate_batch_sharded, what bench.py --gpus N
    times): rank r evaluates its 2048 gates, the output LWEs are all-gathered;
    all 4096 gathered ciphertexts == the oracle digests of the world-1 batch;
  * a C0 layer chain (conv + ReLU, max-pool, FC) with neuron-sharded contexts
    and gather_shards between layers: the gathered ciphertexts of every layer
    are bit-identical to the world-1 run's.
"""
import hashlib
import os
import socket

import numpy as np
import pytest

import she_inputs as si
from oracle import network as net

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1906_00148_b200 import parallel, she  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def digest(words: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(words, dtype="<u4").tobytes()).hexdigest()[:32]


def read_digests(cfg):
    rows = []
    for line in open(os.path.join(GOLDEN, f"config{cfg}_oracle_digests.txt")):
        if line.startswith("#") or not line.strip():
            continue
        g, op, d, bit = line.split()
        rows.append((int(g), int(op), d, int(bit)))
    return rows


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _layer_chain(ctx, sk, P, rank, world):
    """C0 chain: conv 3x3 'same' + ReLU -> max-pool -> FC; returns the host
    ciphertexts of the three gathered layer outputs."""
    rng = np.random.default_rng(71)
    px = rng.integers(0, 256, (6, 6, 1))
    w1 = si.log_quant_weights(4, (4, 3, 3, 1), layer=50)
    w2 = si.log_quant_weights(4, (5, 3 * 3 * 4), layer=51)
    bits = net.bits_of(px, 8)
    x = _dev(she.she_encrypt_bits(sk, bits.ravel(), 4545, 0).reshape(bits.shape + (P.stride,)))
    wa = she.conv_width(6, 6, 1, 8, False, w1, 1, 1, 16, relu=True)
    buf = lambda words, w: torch.zeros((parallel.padded_words(words, world), w, P.stride),
                                       dtype=torch.int32, device="cuda")
    h = buf(36 * 4, wa)
    she.she_conv_shift_acc(ctx, x, 6, 6, 1, 8, False, w1, 1, 1, 16, relu=True, out=h[:144])
    h1 = parallel.gather_shards(h, 144, rank, world)
    p = buf(9 * 4, wa)
    she.she_maxpool2x2(ctx, h1.reshape(6, 6, 4, wa, P.stride), 6, 6, 4, wa, False, out=p[:36])
    p1 = parallel.gather_shards(p, 36, rank, world)
    wb = she.fc_width(36, wa, False, w2, 16)
    f = buf(5, wb)
    she.she_fc_shift_acc(ctx, p1.reshape(36, wa, P.stride), 36, wa, False, w2, 16, out=f[:5])
    f1 = parallel.gather_shards(f, 5, rank, world)
    torch.cuda.synchronize()
    return [t.cpu().numpy().view(np.uint32).copy() for t in (h1, p1, f1)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        # config 1, strong-scaled
        P = si.C1
        sk, ck = she.she_keygen(P, si.key_seed(1))
        ctx = she.Context(P, ck, device=0, rank=rank, world=world)
        ops = si.gate_ops(1, 4096)
        bits = si.gate_input_bits(1, 4096)
        cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(1), 0).reshape(4096, 3, -1)
        d_ops = torch.from_numpy(ops.astype(np.uint8)).cuda()
        a, b, c = (_dev(cts[:, j].copy()) for j in range(3))
        out = torch.zeros((parallel.padded_words(4096, world), P.stride), dtype=torch.int32,
                          device="cuda")
        got = parallel.gate_batch_sharded(ctx, d_ops, a, b, c, out, rank, world)
        torch.cuda.synchronize()
        c1 = [digest(row[: P.n + 1]) for row in got.cpu().numpy().view(np.uint32)]
        ctx.close()
        # C0 layer chain, neuron-sharded
        P0 = si.C0
        sk0, ck0 = she.she_keygen(P0, si.key_seed(0))
        ctx0 = she.Context(P0, ck0, device=0, rank=rank, world=world)
        layers = _layer_chain(ctx0, sk0, P0, rank, world)
        ctx0.close()
        q.put((rank, c1, layers))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_strong_scaled_config1_and_sharded_layers(cuda):
    world = 2
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, c1, layers = q.get(timeout=900)
        res[r] = (c1, layers)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rows = read_digests(1)
    for r in range(world):
        c1 = res[r][0]
        bad = [g for g, op, d, bit in rows if c1[g] != d]
        assert not bad, f"rank {r}: {len(bad)} gathered gates differ from the oracle digests"
    # world-1 reference of the layer chain, bit for bit
    P0 = si.C0
    sk0, ck0 = she.she_keygen(P0, si.key_seed(0))
    ctx0 = she.Context(P0, ck0, device=0)
    ref = _layer_chain(ctx0, sk0, P0, 0, 1)
    ctx0.close()
    for r in range(world):
        for name, want, got in zip(("conv+relu", "maxpool", "fc"), ref, res[r][1]):
            n = want.shape[0]
            assert np.array_equal(got[:n], want), f"rank {r}: {name} differs from world 1"
