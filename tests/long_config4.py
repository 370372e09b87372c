#!/usr/bin/env python
"""Full encrypted run of BASELINE.json configs[4] (CIFAR-10-shaped net) on one
GPU: 32x32x3 uint8 -> conv3x3 3->32 + ReLU -> conv3x3 32->32 + ReLU ->
maxpool -> conv3x3 32->64 + ReLU -> maxpool -> FC 4096->10, at the TFHE
default parameters (0.46 G bootstrapped gates, 0.59 G blind-rotation lanes).

Every layer's decrypted output is compared with the plaintext network
(oracle/network.py); seed-sampled gates of every layer are captured from the
GPU wire table and recomputed by the CPU oracle word for word at the end.
Results are written to gpurun_out/config4_full.json after every layer, so a
time-out keeps what finished.

    python tests/long_config4.py           (about 4 hours on one B200)

A script (not collected by pytest): it lives under tests/ because it runs the
oracle, which only tests/, smoke() and bench.py's CPU legs may use.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: the parity check only)
import she_inputs as si  # noqa: E402
from oracle import network as net  # noqa: E402
from paper_1906_00148_b200 import she  # noqa: E402


def main():
    import torch
    out_path = os.path.join(ROOT, "gpurun_out", "config4_full.json")
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    cfg = 4
    P = si.CONFIG_PARAMS[cfg]
    stride = P.stride
    sk, ck = she.she_keygen(P, si.key_seed(cfg))
    ctx = she.Context(P, ck, device=0)
    px = si.pixels(cfg, (32, 32, 3)).astype(np.int64)
    w1 = si.log_quant_weights(cfg, (32, 3, 3, 3), layer=0)
    w2 = si.log_quant_weights(cfg, (32, 3, 3, 32), layer=1)
    w3 = si.log_quant_weights(cfg, (64, 3, 3, 32), layer=2)
    w4 = si.log_quant_weights(cfg, (10, 4096), layer=3)
    plain = {}
    plain["conv1"] = net.relu(net.conv(px, w1, 1, 1, 16))
    plain["conv2"] = net.relu(net.conv(plain["conv1"], w2, 1, 1, 16))
    plain["pool1"] = net.maxpool2x2(plain["conv2"])
    plain["conv3"] = net.relu(net.conv(plain["pool1"], w3, 1, 1, 16))
    plain["pool2"] = net.maxpool2x2(plain["conv3"])
    plain["fc"] = net.fc(plain["pool2"].ravel(), w4, 16)
    exact_logits = net.fc_exact(plain["pool2"].ravel(), w4)

    report = {"workload": "config4: CIFAR-10-shaped encrypted net, 32x32x3 uint8 input, "
                          "conv3x3 3->32 + ReLU, conv3x3 32->32 + ReLU, maxpool2x2, conv3x3 "
                          "32->64 + ReLU, maxpool2x2, FC 4096->10; log-quantised weights, 16-bit "
                          "mixed-width accumulators; default TFHE parameters; one B200",
              "layers": [], "wrap16_events_in_logits": int(net.wrap_events(exact_logits, 16))}

    def save():
        with open(out_path, "w") as f:
            json.dump(report, f, indent=1)

    def decrypt(t, width, signed):
        h = t.cpu().numpy().view(np.uint32).reshape(-1, stride)
        return net.value_of(she.she_decrypt_bits(sk, h).reshape(-1, width), signed=signed)

    bits = net.bits_of(px, 8)
    x = torch.from_numpy(she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(cfg), 0)
                         .view(np.int32)).cuda().reshape(32, 32, 3, 8, stride)
    captured = []
    t_all = time.perf_counter()

    def layer(name, fn, every, signed):
        # ~6 seed-sampled gates per layer (every = about gates / 6)
        she.capture(ctx, si.sample_seed(cfg) + len(report["layers"]), every, 8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        out, w = fn()
        e1.record()
        torch.cuda.synchronize()
        st = she.layer_stats(ctx)
        ops, slots = she.capture_read(ctx, 8)
        captured.append((name, ops, slots))
        got = decrypt(out, w, signed)
        want = plain[name].reshape(-1)
        entry = {"layer": name, "device_s": round(e0.elapsed_time(e1) * 1e-3, 2),
                 "wall_s": round(time.perf_counter() - t0, 2), "gates": int(st["gates"]),
                 "br_lanes": int(st["br_lanes"]), "levels": int(st["levels"]),
                 "tiles": int(st["tiles"]), "output_words": int(want.size), "width": int(w),
                 "decrypted_mismatches": int(np.sum(got != want)),
                 "sampled_gates_captured": int(len(ops))}
        report["layers"].append(entry)
        save()
        print(json.dumps(entry), flush=True)
        return out, w

    h1, wa = layer("conv1", lambda: she.she_conv_shift_acc(ctx, x, 32, 32, 3, 8, False, w1, 1, 1,
                                                           16, relu=True), 2_600_003, False)
    h2, wb = layer("conv2", lambda: she.she_conv_shift_acc(ctx, h1, 32, 32, 32, wa, False, w2, 1, 1,
                                                           16, relu=True), 48_000_017, False)
    del h1
    p1, _ = layer("pool1", lambda: (she.she_maxpool2x2(ctx, h2, 32, 32, 32, wb, False), wb),
                  180_001, False)
    del h2
    h3, wc = layer("conv3", lambda: she.she_conv_shift_acc(ctx, p1, 16, 16, 32, wb, False, w3, 1, 1,
                                                           16, relu=True), 25_000_009, False)
    p2, _ = layer("pool2", lambda: (she.she_maxpool2x2(ctx, h3, 16, 16, 64, wc, False), wc),
                  90_001, False)
    lo, wd = layer("fc", lambda: she.she_fc_shift_acc(ctx, p2.reshape(-1, wc, stride), 4096, wc,
                                                      False, w4, 16), 240_007, True)
    report["total_device_s"] = round(sum(e["device_s"] for e in report["layers"]), 1)
    report["total_wall_s"] = round(time.perf_counter() - t_all, 1)
    report["gates"] = int(sum(e["gates"] for e in report["layers"]))
    report["br_lanes"] = int(sum(e["br_lanes"] for e in report["layers"]))
    report["levels"] = int(sum(e["levels"] for e in report["layers"]))
    report["decrypted_mismatches"] = int(sum(e["decrypted_mismatches"] for e in report["layers"]))
    save()

    # seed-sampled ciphertext parity against the oracle (C1 schoolbook, host cores)
    K = oracle.keygen(P, si.key_seed(cfg))
    checked = bad = 0
    for name, ops, slots in captured:
        if not len(ops):
            continue
        a, b, c, out = (np.ascontiguousarray(slots[:, j]) for j in range(4))
        ref = oracle.gates(K, ops, a, b, c)
        bad += int(np.sum(np.any(ref != out, axis=1)))
        checked += len(ops)
    report["sampled_gate_ciphertexts_compared"] = checked
    report["sampled_gate_ciphertext_mismatches"] = bad
    save()
    print(json.dumps({k: v for k, v in report.items() if k != "layers"}), flush=True)


if __name__ == "__main__":
    main()
