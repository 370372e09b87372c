#!/usr/bin/env python
"""Summary of the chained config-4 run (tests/chain_config4.py stages A, B, C)
-> profiles/r2/config4_chain/summary.json: per layer the device seconds,
gates, lanes, decrypted words and mismatches, sampled gate ciphertexts, and
the digest chain (every layer's input ciphertexts are the previous layer's
bootstrapped outputs: input_sha256 == the previous output_sha256; conv2's two
rank halves merge into pool1's input)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORDS = {"conv1": 32768, "conv2": 32768, "pool1": 8192, "conv3": 16384, "pool2": 4096, "fc": 10}


def main(src=None, dst=None):
    src = src or os.path.join(ROOT, "profiles", "r2", "config4_chain")
    dst = dst or os.path.join(src, "summary.json")
    st = {s: json.load(open(os.path.join(src, f"config4chain_{s}.json"))) for s in "ABC"}
    L = {e["layer"]: e for s in "ABC" for e in st[s]["layers"]}
    chain = [
        ("conv1 -> conv2 (rank 0 of 2)", L["conv1"]["output_sha256"] == L["conv2.0"]["input_sha256"]),
        ("conv1 -> conv2 (rank 1 of 2)", L["conv1"]["output_sha256"] == L["conv2.1"]["input_sha256"]),
        ("conv2 (merged halves) -> pool1", st["B"]["conv2_merged_sha256"] == L["pool1"]["input_sha256"]),
        ("pool1 -> conv3", L["pool1"]["output_sha256"] == L["conv3"]["input_sha256"]),
        ("conv3 -> pool2", L["conv3"]["output_sha256"] == L["pool2"]["input_sha256"]),
        ("pool2 -> fc", L["pool2"]["output_sha256"] == L["fc"]["input_sha256"]),
    ]
    rows = []
    for name in ("conv1", "conv2", "pool1", "conv3", "pool2", "fc"):
        parts = [L[k] for k in (["conv2.0", "conv2.1"] if name == "conv2" else [name])]
        rows.append({"layer": name, "device_s": round(sum(p["device_s"] for p in parts), 2),
                     "gates": sum(p["gates"] for p in parts),
                     "br_lanes": sum(p["br_lanes"] for p in parts),
                     "decrypted_compared": sum(p["decrypted_compared"] for p in parts),
                     "decrypted_mismatches": sum(p["decrypted_mismatches"] for p in parts),
                     "words": WORDS[name],
                     "sampled_gate_ciphertexts_compared":
                         sum(p["sampled_gate_ciphertexts_compared"] for p in parts),
                     "sampled_gate_ciphertext_mismatches":
                         sum(p["sampled_gate_ciphertext_mismatches"] for p in parts)})
    out = {"workload": "BASELINE.json configs[4] (CIFAR-10-shaped net) at the default parameters, "
                       "end to end on one B200: every layer consumes the previous layer's "
                       "bootstrapped output ciphertexts (checkpointed between the three one-hour "
                       "calls on the same box, digests below); conv2 as two rank halves",
           "layers": rows,
           "digest_chain": [{"link": k, "ok": bool(v)} for k, v in chain],
           "chained": all(v for _, v in chain),
           "complete": all(r["decrypted_compared"] == r["words"] for r in rows),
           "latency_s_measured": round(sum(r["device_s"] for r in rows), 1),
           "latency_note": "sum of the CUDA-event device seconds of every layer (all measured; "
                           "excludes checkpoint save/load and the client's encryption/decryption)",
           "gates": sum(r["gates"] for r in rows), "br_lanes": sum(r["br_lanes"] for r in rows),
           "decrypted_compared": sum(r["decrypted_compared"] for r in rows),
           "decrypted_mismatches": sum(r["decrypted_mismatches"] for r in rows),
           "sampled_gate_ciphertexts_compared":
               sum(r["sampled_gate_ciphertexts_compared"] for r in rows),
           "sampled_gate_ciphertext_mismatches":
               sum(r["sampled_gate_ciphertext_mismatches"] for r in rows),
           "logits": st["C"].get("logits"), "logits_plain": st["C"].get("logits_plain")}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "layers"}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
