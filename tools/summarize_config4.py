#!/usr/bin/env python
"""Merge the config-4 shard results (gpurun_out/config4_<layer>_<r>of<W>.json,
written by tests/long_config4.py) into profiles/r1/config4/summary.json: per
layer the summed device seconds, gates, lanes, decrypted words and mismatches,
and the whole net's single-GPU latency as the sum over layers."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORDER = ["conv1", "conv2", "pool1", "conv3", "pool2", "fc"]


def main(src=None, dst=None):
    src = src or os.path.join(ROOT, "profiles", "r1", "config4")
    dst = dst or os.path.join(src, "summary.json")
    shards = [json.load(open(p)) for p in sorted(glob.glob(os.path.join(src, "config4_*of*.json")))]
    layers = {}
    for e in shards:
        L = layers.setdefault(e["layer"], {"layer": e["layer"], "shards": 0, "device_s": 0.0,
                                          "gates": 0, "br_lanes": 0, "decrypted_compared": 0,
                                          "decrypted_mismatches": 0,
                                          "sampled_gate_ciphertexts_compared": 0,
                                          "sampled_gate_ciphertext_mismatches": 0})
        L["shards"] += 1
        for k in ("device_s", "gates", "br_lanes", "decrypted_compared", "decrypted_mismatches",
                  "sampled_gate_ciphertexts_compared", "sampled_gate_ciphertext_mismatches"):
            L[k] += e[k]
    rows = [layers[k] for k in ORDER if k in layers]
    for r in rows:
        r["device_s"] = round(r["device_s"], 2)
    out = {"workload": "config4 (CIFAR-10-shaped net) at the default parameters on one B200, by "
                       "layer / rank shard (tests/long_config4.py); each layer fed with the "
                       "client's encryption of its exact plaintext input",
           "layers": rows,
           "complete": [r["layer"] for r in rows] == ORDER,
           "latency_s_sum_of_layers": round(sum(r["device_s"] for r in rows), 1),
           "gates": sum(r["gates"] for r in rows), "br_lanes": sum(r["br_lanes"] for r in rows),
           "decrypted_compared": sum(r["decrypted_compared"] for r in rows),
           "decrypted_mismatches": sum(r["decrypted_mismatches"] for r in rows),
           "sampled_gate_ciphertexts_compared":
               sum(r["sampled_gate_ciphertexts_compared"] for r in rows),
           "sampled_gate_ciphertext_mismatches":
               sum(r["sampled_gate_ciphertext_mismatches"] for r in rows)}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
