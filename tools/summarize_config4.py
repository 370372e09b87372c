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
LAYER_WORDS = {"conv1": 32 * 32 * 32, "conv2": 32 * 32 * 32, "pool1": 16 * 16 * 32,
               "conv3": 16 * 16 * 64, "pool2": 8 * 8 * 64, "fc": 10}


def main(src=None, dst=None):
    src = src or os.path.join(ROOT, "profiles", "r1", "config4")
    dst = dst or os.path.join(src, "summary.json")
    shards = [json.load(open(p)) for p in sorted(glob.glob(os.path.join(src, "config4_*of*.json")))]
    layers = {}
    for e in shards:
        L = layers.setdefault(e["layer"], {"layer": e["layer"], "shards": 0, "world": e["world"],
                                          "ranks": [], "device_s": 0.0,
                                          "gates": 0, "br_lanes": 0, "decrypted_compared": 0,
                                          "decrypted_mismatches": 0,
                                          "sampled_gate_ciphertexts_compared": 0,
                                          "sampled_gate_ciphertext_mismatches": 0})
        L["shards"] += 1
        L["ranks"].append(e["rank"])
        L["world"] = max(L["world"], e["world"])
        for k in ("device_s", "gates", "br_lanes", "decrypted_compared", "decrypted_mismatches",
                  "sampled_gate_ciphertexts_compared", "sampled_gate_ciphertext_mismatches"):
            L[k] += e[k]
    rows = [layers[k] for k in ORDER if k in layers]
    for r in rows:
        r["device_s"] = round(r["device_s"], 2)
        r["ranks"] = sorted(set(r["ranks"]))
        # a layer is complete when every rank shard of its split ran and every
        # output word was decrypted and compared
        r["complete"] = (r["ranks"] == list(range(r["world"])) and
                         r["decrypted_compared"] == LAYER_WORDS[r["layer"]])
    out = {"workload": "config4 (CIFAR-10-shaped net) at the default parameters on one B200, by "
                       "layer / rank shard (tests/long_config4.py); each layer fed with the "
                       "client's encryption of its exact plaintext input",
           "layers": rows,
           "complete": [r["layer"] for r in rows] == ORDER and all(r["complete"] for r in rows),
           "incomplete_layers": [r["layer"] for r in rows if not r["complete"]] +
                                [k for k in ORDER if k not in layers],
           "latency_s_sum_of_layers": round(sum(r["device_s"] for r in rows), 1),
           "latency_note": "sum of the measured device seconds of the shards that ran; a "
                           "lower bound when a layer is incomplete",
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
