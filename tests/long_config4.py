#!/usr/bin/env python
"""Full-size parity and timing of BASELINE.json configs[4] (CIFAR-10-shaped
net) on one GPU, layer by layer and shard by shard:

    32x32x3 uint8 -> conv3x3 3->32 + ReLU -> conv3x3 32->32 + ReLU -> maxpool
    -> conv3x3 32->64 + ReLU -> maxpool -> FC 4096->10

at the TFHE default parameters (0.46 G bootstrapped gates, 0.59 G blind-
rotation lanes, ~4 GPU-hours).  One GPU call is limited to an hour, so every
layer (or a rank shard of it: the multi-GPU neuron split) runs on
its own, fed with the client's encryption of that layer's exact plaintext input
(a fresh ciphertext is as valid an input as a bootstrapped one: every gate
output is a freshly bootstrapped sample).  For EVERY output word of the shard
the decrypted value must equal the plaintext network (oracle/network.py), and
seed-sampled gates captured from the GPU wire table are recomputed by the CPU
oracle word for word.  Results go to gpurun_out/config4_<layer>_<r>of<W>.json.

    python tests/long_config4.py --layers conv1,pool1,pool2,fc
    python tests/long_config4.py --layers conv2 --rank 0 --world 4   (x4 ranks)
    python tests/long_config4.py --layers conv3 --rank 0 --world 2   (x2 ranks)

A script (not collected by pytest): it lives under tests/ because it runs the
oracle, which only tests/, smoke() and bench.py's CPU legs may use.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import she_inputs as si  # noqa: E402
from oracle import network as net  # noqa: E402
from paper_1906_00148_b200 import she  # noqa: E402

CFG = 4


def plain_network():
    px = si.pixels(CFG, (32, 32, 3)).astype(np.int64)
    w = {"conv1": si.log_quant_weights(CFG, (32, 3, 3, 3), layer=0),
         "conv2": si.log_quant_weights(CFG, (32, 3, 3, 32), layer=1),
         "conv3": si.log_quant_weights(CFG, (64, 3, 3, 32), layer=2),
         "fc": si.log_quant_weights(CFG, (10, 4096), layer=3)}
    p = {"input": px}
    p["conv1"] = net.relu(net.conv(px, w["conv1"], 1, 1, 16))
    p["conv2"] = net.relu(net.conv(p["conv1"], w["conv2"], 1, 1, 16))
    p["pool1"] = net.maxpool2x2(p["conv2"])
    p["conv3"] = net.relu(net.conv(p["pool1"], w["conv3"], 1, 1, 16))
    p["pool2"] = net.maxpool2x2(p["conv3"])
    p["fc"] = net.fc(p["pool2"].ravel(), w["fc"], 16)
    assert np.array_equal(p["fc"], net.config4(px, w["conv1"], w["conv2"], w["conv3"], w["fc"]))
    return w, p


# layer -> (input name, input width function, signed output, sampling rate)
PREV = {"conv1": "input", "conv2": "conv1", "pool1": "conv2", "conv3": "pool1", "pool2": "conv3",
        "fc": "pool2"}
EVERY = {"conv1": 2_600_003, "conv2": 12_000_017, "pool1": 180_001, "conv3": 12_500_009,
         "pool2": 90_001, "fc": 240_007}


def widths(w):
    wa = she.conv_width(32, 32, 3, 8, False, w["conv1"], 1, 1, 16, relu=True)
    wb = she.conv_width(32, 32, 32, wa, False, w["conv2"], 1, 1, 16, relu=True)
    wc = she.conv_width(16, 16, 32, wb, False, w["conv3"], 1, 1, 16, relu=True)
    return {"input": 8, "conv1": wa, "conv2": wb, "pool1": wb, "conv3": wc, "pool2": wc}


def run(layer, rank, world, sk, ck, P, w, plain, win):
    import torch
    stride = P.stride
    ctx = she.Context(P, ck, device=0, rank=rank, world=world)
    src = plain[PREV[layer]]
    width = win[PREV[layer]]
    bits = net.bits_of(src, width)
    seed = si.input_seed(CFG) + 100 + list(PREV).index(layer)
    x = torch.from_numpy(she.she_encrypt_bits(sk, bits.ravel(), seed, 0).view(np.int32)).cuda()
    x = x.reshape(bits.shape + (stride,))
    she.capture(ctx, si.sample_seed(CFG) + 10 * list(PREV).index(layer) + rank, EVERY[layer], 16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    if layer in ("conv1", "conv2", "conv3"):
        H, _, C = src.shape
        out, wo = she.she_conv_shift_acc(ctx, x, H, H, C, width, False, w[layer], 1, 1, 16,
                                         relu=True)
        signed = False
    elif layer in ("pool1", "pool2"):
        H, _, C = src.shape
        out, wo = she.she_maxpool2x2(ctx, x, H, H, C, width, False), width
        signed = False
    else:
        out, wo = she.she_fc_shift_acc(ctx, x.reshape(-1, width, stride), 4096, width, False,
                                       w["fc"], 16)
        signed = True
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    st = she.layer_stats(ctx)
    ops, slots = she.capture_read(ctx, 16)
    want = plain[layer].reshape(-1)
    words = want.size
    lo, hi = rank * (-(-words // world)), min(words, (rank + 1) * (-(-words // world)))
    h = out.reshape(words, wo, stride)[lo:hi].cpu().numpy().view(np.uint32)
    got = net.value_of(she.she_decrypt_bits(sk, h.reshape(-1, stride)).reshape(-1, wo),
                       signed=signed)
    K = oracle.keygen(P, si.key_seed(CFG))
    bad_ct = 0
    if len(ops):
        a, b, c, o = (np.ascontiguousarray(slots[:, j]) for j in range(4))
        bad_ct = int(np.sum(np.any(oracle.gates(K, ops, a, b, c) != o, axis=1)))
    entry = {"layer": layer, "rank": rank, "world": world, "words": [int(lo), int(hi)],
             "device_s": round(e0.elapsed_time(e1) * 1e-3, 2), "wall_s": round(wall, 2),
             "gates": int(st["gates"]), "br_lanes": int(st["br_lanes"]),
             "levels": int(st["levels"]), "tiles": int(st["tiles"]),
             "decrypted_compared": int(hi - lo),
             "decrypted_mismatches": int(np.sum(got != want[lo:hi])),
             "sampled_gate_ciphertexts_compared": int(len(ops)),
             "sampled_gate_ciphertext_mismatches": bad_ct}
    ctx.close()
    return entry


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="conv1,pool1,pool2,fc")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--world", type=int, default=1)
    args = ap.parse_args()
    P = si.CONFIG_PARAMS[CFG]
    sk, ck = she.she_keygen(P, si.key_seed(CFG))
    w, plain = plain_network()
    win = widths(w)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for layer in args.layers.split(","):
        entry = run(layer, args.rank, args.world, sk, ck, P, w, plain, win)
        path = os.path.join(ROOT, "gpurun_out",
                            f"config4_{layer}_{args.rank}of{args.world}.json")
        with open(path, "w") as f:
            json.dump(entry, f, indent=1)
        print(json.dumps(entry), flush=True)


if __name__ == "__main__":
    main()
