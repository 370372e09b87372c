"""Write the oracle's output digests for a gate-batch config (calls only oracle/).

    python tests/golden/make_oracle_digests.py 1      # config 1: 4096 gates, C1

Workload: keys seed 1000+cfg; per gate g: op = gate_ops(cfg)[g];
input bits = gate_input_bits(cfg)[g, slot], encrypted with seed 2000+cfg as
ciphertext number 3g+slot.  Output: one line per gate,
    <g> <op> <sha256(out[g][0..n] as little-endian uint32)[:32]> <decrypted bit>
The GPU parity test (tests/test_gpu_gates.py) compares every gate of the CUDA
path against these digests (full ciphertext comparison, config 1).
"""
import hashlib
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import she_inputs as si  # noqa: E402


def workload_oracle(cfg: int, count: int):
    P = si.CONFIG_PARAMS[cfg]
    K = oracle.keygen(P, si.key_seed(cfg))
    ops = si.gate_ops(cfg, count)
    bits = si.gate_input_bits(cfg, count)
    cts = oracle.encrypt(P, K.s, bits.ravel(), si.input_seed(cfg), 0).reshape(count, 3, -1)
    return P, K, ops, bits, cts


def digest(words: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(words, dtype="<u4").tobytes()).hexdigest()[:32]


def main(cfg: int) -> None:
    count = si.CONFIG_GATES[cfg]
    P, K, ops, bits, cts = workload_oracle(cfg, count)
    t0 = time.time()
    out = oracle.gates(K, ops, cts[:, 0].copy(), cts[:, 1].copy(), cts[:, 2].copy())
    dt = time.time() - t0
    dec = oracle.decrypt(P, K.s, out)
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    assert np.array_equal(dec, want), "oracle decrypts a gate wrongly"
    path = os.path.join(HERE, f"config{cfg}_oracle_digests.txt")
    with open(path, "w") as f:
        f.write(f"# config {cfg}: {count} gates, params {P}; oracle {dt:.1f} s on "
                f"{oracle.threads()} threads; written by tests/golden/make_oracle_digests.py\n")
        for g in range(count):
            f.write(f"{g} {int(ops[g])} {digest(out[g, : P.n + 1])} {int(dec[g])}\n")
    print(path, f"{dt:.1f}s")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
