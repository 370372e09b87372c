#!/usr/bin/env python
"""Multiplicative-depth (MD) ledger of the configs' layers (Eq. 1,
:175-180 §3.4; Table 2 :151-162), host only.

For every layer of configs 2-4 (and the DSHE-style net of bench.py --dshe)
two numbers are reported:
  * measured: the depth of the scheduled gate circuit, i.e. the number of
    ASAP levels the library's scheduler emits for the layer (every level is
    one homomorphic gate, NOT/shift/constant are free), from the clear-bit
    backend (csrc/scheduler.cpp; the same circuits the GPU runs);
  * Eq. 1: LMD = IN * log2(KC^2) * (DA[a] + DM[b]) + DR[c] + log2(KP^2) * DM[d]
    read as (reading R-MD): IN input channels, KC the kernel
    size (FC: IN = 1, KC^2 = fan-in), DM[b] = 0 (a log-quantised weight is a
    shift: MD 0), DA[a] = the carry-chain depth of the widest
    a-bit adder of the layer's tree, a + 1 for the FA-B adder (XOR, XOR, MUX;
    the carry passes one MUX per bit after the first XOR), DR[c] = 1 (one AND
    level), DM[d] = d + 2 for the max unit (d + 1 comparator carry levels and
    the output MUX), KP = 2 for a 2x2 pool, 0 otherwise.
Eq. 1 charges every tree level a full carry chain (an upper bound); the
scheduler overlaps the chains of successive tree levels, so measured <= Eq. 1.
The totals are the network MD (Eq. 1 sums the layers) against the paper's
32K AND-depth budget of its leveled TFHE setting.

    python tools/md_ledger.py [--out profiles/r2/md_ledger.json]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import she_inputs as si  # noqa: E402
from paper_1906_00148_b200 import she  # noqa: E402


def bits_of(v, w):
    v = np.asarray(v, dtype=np.int64)
    return ((v[..., None] >> np.arange(w)) & 1).astype(np.uint8)


def depth(st):
    """Circuit depth of a layer: the scheduler levelises each neuron tile on
    its own and runs the tiles one after another, so its level count is the
    sum over tiles; every tile of a layer has the same depth (same fan-in and
    widths), so the depth is levels / tiles."""
    return int(math.ceil(st["levels"] / max(1, st["tiles"])))


def eq1(IN, KC2, a, relu, pool_bits=None):
    lmd = IN * math.log2(KC2) * (a + 1) + (1 if relu else 0)
    if pool_bits is not None:
        lmd += math.log2(4) * (pool_bits + 2)
    return lmd


def conv_layer(name, x, w, wq, stride, pad, relu, signed=False):
    H, W, C = x.shape
    K = wq.shape[1]
    out, wo, st = she.clear_conv_shift_acc(bits_of(x, w), H, W, C, w, signed, wq, stride, pad,
                                           16, relu=relu)
    a = wo + (1 if relu else 0)  # accumulator width before the ReLU drops the sign
    return {"layer": name, "kind": "conv", "IN": C, "KC": K, "a_bits": a,
            "measured_levels": depth(st), "gates": st["gates"], "tiles": st["tiles"],
            "eq1": round(eq1(C, K * K, a, relu), 1)}, out, wo


def fc_layer(name, x, w, wq, relu, signed=False):
    K = x.size
    out, wo, st = she.clear_fc_shift_acc(bits_of(x.ravel(), w), K, w, signed, wq, 16, relu=relu)
    a = wo + (1 if relu else 0)
    return {"layer": name, "kind": "fc", "IN": 1, "KC": f"sqrt({K})", "a_bits": a,
            "measured_levels": depth(st), "gates": st["gates"], "tiles": st["tiles"],
            "eq1": round(eq1(1, K, a, relu), 1)}, out, wo


def pool_layer(name, x, w):
    H, W, C = x.shape
    out, st = she.clear_maxpool2x2(bits_of(x, w), H, W, C, w, False)
    return {"layer": name, "kind": "maxpool2x2", "d_bits": w, "measured_levels": depth(st),
            "gates": st["gates"], "tiles": st["tiles"], "eq1": round(math.log2(4) * (w + 2), 1)}, out


def value(bits, signed=False):
    b = bits.astype(np.int64)
    v = (b << np.arange(b.shape[-1])).sum(axis=-1)
    if signed:
        v = np.where(b[..., -1] == 1, v - (1 << b.shape[-1]), v)
    return v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "md_ledger.json"))
    ap.add_argument("--skip-config4", action="store_true")
    args = ap.parse_args()
    res = {}
    # configs 2-3 (MNIST-shaped)
    px = si.pixels(3, (28, 28, 1)).astype(np.int64)
    w1 = si.log_quant_weights(3, (5, 5, 5, 1), layer=0)
    w2 = si.log_quant_weights(3, (100, 720), layer=1)
    w3 = si.log_quant_weights(3, (10, 100), layer=2)
    L1, h1, wa = conv_layer("conv1 5x5/2 1->5 + ReLU", px, 8, w1, 2, 0, True)
    L2, h2, wb = fc_layer("fc 720->100 + ReLU", value(h1), wa, w2, True)
    L3, _, _ = fc_layer("fc 100->10", value(h2), wb, w3, False)
    res["config2"] = [L1]
    res["config3"] = [L1, L2, L3]
    if not args.skip_config4:
        px4 = si.pixels(4, (32, 32, 3)).astype(np.int64)
        c1 = si.log_quant_weights(4, (32, 3, 3, 3), layer=0)
        c2 = si.log_quant_weights(4, (32, 3, 3, 32), layer=1)
        c3 = si.log_quant_weights(4, (64, 3, 3, 32), layer=2)
        f4 = si.log_quant_weights(4, (10, 4096), layer=3)
        A, o1, wa = conv_layer("conv1 3x3 3->32 + ReLU", px4, 8, c1, 1, 1, True)
        B, o2, wb = conv_layer("conv2 3x3 32->32 + ReLU", value(o1), wa, c2, 1, 1, True)
        P1, p1 = pool_layer("maxpool1", value(o2), wb)
        C, o3, wc = conv_layer("conv3 3x3 32->64 + ReLU", value(p1), wb, c3, 1, 1, True)
        P2, p2 = pool_layer("maxpool2", value(o3), wc)
        D, _, _ = fc_layer("fc 4096->10", value(p2), wc, f4, False)
        res["config4"] = [A, B, P1, C, P2, D]
    out = {"note": __doc__.split("\n\n")[0], "budget_paper_and_depth": 32768, "configs": {}}
    for cfg, layers in res.items():
        out["configs"][cfg] = {"layers": layers,
                               "measured_total": int(sum(L["measured_levels"] for L in layers)),
                               "eq1_total": round(sum(L["eq1"] for L in layers), 1)}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    for cfg, v in out["configs"].items():
        print(cfg, "measured", v["measured_total"], "eq1", v["eq1_total"])
        for L in v["layers"]:
            print("   ", L["layer"], L["measured_levels"], L["eq1"])


if __name__ == "__main__":
    main()
