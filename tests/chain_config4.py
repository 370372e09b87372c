#!/usr/bin/env python
"""BASELINE.json configs[4] (CIFAR-10-shaped net) END TO END on one GPU, each
layer consuming the previous layer's bootstrapped output ciphertexts:

    32x32x3 uint8 -> conv3x3 3->32 + ReLU -> conv3x3 32->32 + ReLU -> maxpool
    -> conv3x3 32->64 + ReLU -> maxpool -> FC 4096->10

at the TFHE default parameters (0.46 G bootstrapped gates, 0.59 G blind-
rotation lanes).  A GPU call is limited to an hour and the net needs about
1.5 h, so the chain runs as stages that checkpoint the layer-boundary
ciphertexts (SURVEY.md:364-365 checkpoint/resume) under --ckpt on the GPU box:

    A  encrypt the pixels, conv1, conv2 rows [0, 1/2)     -> ckpt conv1, conv2.0
    B  conv2 rows [1/2, 1) (input: ckpt conv1), pool1      -> ckpt pool1
    C  conv3, pool2, fc (input: ckpt pool1)                 -> the encrypted logits

(conv2 is split by output neurons with the multi-GPU shard API, rank r of 2.)
Every checkpoint is recorded in a manifest with its SHA-256; a stage refuses
to start unless the checkpoints it reads match the manifest, so the summary's
digest chain (input digest of layer L == output digest of layer L-1) proves
the layers were chained.  Per layer: device seconds (CUDA events), gates and
lanes, EVERY output word decrypted and compared with the plaintext network
(oracle/network.py), and seed-sampled gate ciphertexts captured from the GPU
wire table recomputed by the CPU oracle word for word (>= 256 over the net).
Results: gpurun_out/config4chain_<stage>.json (+ the manifest).

A script (not collected by pytest): it lives under tests/ because it runs the
oracle, which only tests/, smoke() and bench.py's CPU legs may use.
"""
import argparse
import hashlib
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

sys.path.insert(0, os.path.join(ROOT, "tests"))
from long_config4 import CFG, plain_network, widths  # noqa: E402

STAGES = {"A": ["conv1", "conv2.0"], "B": ["conv2.1", "pool1"], "C": ["conv3", "pool2", "fc"]}
# capture period per layer: ~64 sampled gates each (>= 256 over the net)
EVERY = {"conv1": 160_001, "conv2.0": 1_000_003, "conv2.1": 1_000_003, "pool1": 17_011,
         "conv3": 1_150_007, "pool2": 4_201, "fc": 22_003}
CAP = 80


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


class Ckpt:
    def __init__(self, path):
        self.path = path
        os.makedirs(path, exist_ok=True)
        self.mpath = os.path.join(path, "manifest.json")
        self.m = json.load(open(self.mpath)) if os.path.exists(self.mpath) else {}

    def save(self, name, arr: np.ndarray):
        np.save(os.path.join(self.path, name + ".npy"), arr)
        self.m[name] = {"sha256": sha(arr), "shape": list(arr.shape)}
        json.dump(self.m, open(self.mpath, "w"), indent=1)
        return self.m[name]["sha256"]

    def load(self, name) -> np.ndarray:
        p = os.path.join(self.path, name + ".npy")
        if name not in self.m or not os.path.exists(p):
            raise SystemExit(f"checkpoint {name} missing in {self.path} (box changed?): rerun from stage A")
        a = np.load(p)
        if sha(a) != self.m[name]["sha256"]:
            raise SystemExit(f"checkpoint {name} does not match its manifest digest")
        return a


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stage", required=True, choices=sorted(STAGES))
    ap.add_argument("--ckpt", default="/tmp/she_config4_chain")
    ap.add_argument("--fresh", action="store_true", help="stage A: clear the checkpoint dir")
    args = ap.parse_args()
    import torch

    if args.fresh and os.path.exists(os.path.join(args.ckpt, "manifest.json")):
        os.remove(os.path.join(args.ckpt, "manifest.json"))
    ck = Ckpt(args.ckpt)
    P = si.CONFIG_PARAMS[CFG]
    stride = P.stride
    sk, ckey = she.she_keygen(P, si.key_seed(CFG))
    K = oracle.keygen(P, si.key_seed(CFG))
    w, plain = plain_network()
    win = widths(w)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()
    host = lambda t: t.cpu().numpy().view(np.uint32).copy()
    out_dir = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    report = {"stage": args.stage, "layers": []}

    def run_layer(name, x, ctx, fn, width_in, words, signed, want):
        ops_seed = si.sample_seed(CFG) + 7 * (list(EVERY).index(name) + 1)
        she.capture(ctx, ops_seed, EVERY[name], CAP)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        out, wo = fn(x)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        st = she.layer_stats(ctx)
        ops, slots = she.capture_read(ctx, CAP)
        she.capture(ctx, 0, 0, 0)
        a, b, c, o = (np.ascontiguousarray(slots[:, j]) for j in range(4))
        bad_ct = int(np.sum(np.any(oracle.gates(K, ops, a, b, c) != o, axis=1))) if len(ops) else 0
        return out, wo, {"layer": name, "device_s": round(e0.elapsed_time(e1) * 1e-3, 2),
                         "wall_s": round(wall, 2), "gates": int(st["gates"]),
                         "br_lanes": int(st["br_lanes"]), "levels": int(st["levels"]),
                         "sampled_gate_ciphertexts_compared": int(len(ops)),
                         "sampled_gate_ciphertext_mismatches": bad_ct}

    def decrypt_check(entry, h, lo, hi, wo, signed, want):
        got = net.value_of(she.she_decrypt_bits(sk, h[lo:hi].reshape(-1, stride)).reshape(-1, wo),
                           signed=signed)
        entry["words"] = [int(lo), int(hi)]
        entry["decrypted_compared"] = int(hi - lo)
        entry["decrypted_mismatches"] = int(np.sum(got != want.reshape(-1)[lo:hi]))

    def conv(ctx, name, src_name, x_host, rank=0, world=1):
        src = plain[src_name]
        H, _, C = src.shape
        wi = win[src_name]
        x = dev(x_host).reshape(H, H, C, wi, stride)
        fn = lambda x: she.she_conv_shift_acc(ctx, x, H, H, C, wi, False, w[name.split(".")[0]],
                                              1, 1, 16, relu=True)
        out, wo, e = run_layer(name, x, ctx, fn, wi, None, False, None)
        words = H * H * w[name.split(".")[0]].shape[0]
        per = -(-words // world)
        lo, hi = rank * per, min(words, (rank + 1) * per)
        h = host(out).reshape(words, wo, stride)
        decrypt_check(e, h, lo, hi, wo, False, plain[name.split(".")[0]])
        e["input_sha256"] = sha(x_host)
        return h, wo, lo, hi, e

    def pool(ctx, name, src_name, x_host):
        src = plain[src_name]
        H, _, C = src.shape
        wi = win[src_name]
        x = dev(x_host).reshape(H, H, C, wi, stride)
        fn = lambda x: (she.she_maxpool2x2(ctx, x, H, H, C, wi, False), wi)
        out, wo, e = run_layer(name, x, ctx, fn, wi, None, False, None)
        words = (H // 2) * (H // 2) * C
        h = host(out).reshape(words, wo, stride)
        decrypt_check(e, h, 0, words, wo, False, plain[name])
        e["input_sha256"] = sha(x_host)
        return h, e

    ctx1 = she.Context(P, ckey, device=0)
    if args.stage == "A":
        bits = net.bits_of(plain["input"], 8)
        x0 = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(CFG), 0).reshape(
            bits.shape + (stride,))
        h1, wa, _, _, e = conv(ctx1, "conv1", "input", x0)
        e["output_sha256"] = ck.save("conv1", h1)
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
        ctx2 = she.Context(P, ckey, device=0, rank=0, world=2)
        h2, wb, lo, hi, e = conv(ctx2, "conv2.0", "conv1", h1, rank=0, world=2)
        e["output_sha256"] = ck.save("conv2.0", h2[lo:hi])
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
    elif args.stage == "B":
        h1 = ck.load("conv1")
        ctx2 = she.Context(P, ckey, device=0, rank=1, world=2)
        h2, wb, lo, hi, e = conv(ctx2, "conv2.1", "conv1", h1, rank=1, world=2)
        e["output_sha256"] = sha(h2[lo:hi])
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
        h2[:lo] = ck.load("conv2.0")  # the first half, bootstrapped in stage A
        report["conv2_merged_sha256"] = sha(h2)
        p1, e = pool(ctx1, "pool1", "conv2", h2)
        e["output_sha256"] = ck.save("pool1", p1)
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
    else:
        p1 = ck.load("pool1")
        h3, wc, _, _, e = conv(ctx1, "conv3", "pool1", p1)
        e["output_sha256"] = sha(h3)
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
        p2, e = pool(ctx1, "pool2", "conv3", h3)
        e["output_sha256"] = sha(p2)
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
        x = dev(p2).reshape(4096, win["pool2"], stride)
        fn = lambda x: she.she_fc_shift_acc(ctx1, x, 4096, win["pool2"], False, w["fc"], 16)
        out, wo, e = run_layer("fc", x, ctx1, fn, win["pool2"], 10, True, None)
        lo_h = host(out).reshape(10, wo, stride)
        decrypt_check(e, lo_h, 0, 10, wo, True, plain["fc"])
        e["input_sha256"] = sha(p2)
        e["output_sha256"] = sha(lo_h)
        logits = net.value_of(she.she_decrypt_bits(sk, lo_h.reshape(-1, stride)).reshape(10, wo),
                              signed=True)
        report["logits"] = [int(v) for v in logits]
        report["logits_plain"] = [int(v) for v in plain["fc"]]
        report["layers"].append(e)
        print(json.dumps(e), flush=True)
    report["manifest"] = ck.m
    with open(os.path.join(out_dir, f"config4chain_{args.stage}.json"), "w") as f:
        json.dump(report, f, indent=1)
    print(json.dumps({k: v for k, v in report.items() if k != "layers"}), flush=True)


if __name__ == "__main__":
    main()
