#!/usr/bin/env python
"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
16 config-0 gates, 64 config-1 gates on the default FFT engine (and the NTT
engine), the tensor-core key switch, a C0 conv + ReLU layer, and 8 leveled
CMuxes.  Exits non-zero on a parity mismatch (the parity itself is the GPU
tests' job; this only drives every kernel once under the tool)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import she_inputs as si  # noqa: E402
from paper_1906_00148_b200 import she  # noqa: E402


def gates(cfg, count, **opts):
    P = si.CONFIG_PARAMS[cfg]
    sk, ck = she.she_keygen(P, si.key_seed(cfg))
    ctx = she.Context(P, ck, device=0, **opts)
    ops = si.gate_ops(cfg, count)
    bits = si.gate_input_bits(cfg, count)
    cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(cfg), 0).reshape(count, 3, -1)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).cuda()
    out = torch.zeros((count, P.stride), dtype=torch.int32, device="cuda")
    she.she_gate_batch_ops(ctx, torch.from_numpy(ops.astype(np.uint8)).cuda(), dev(cts[:, 0]),
                           dev(cts[:, 1]), dev(cts[:, 2]), out)
    torch.cuda.synchronize()
    dec = she.she_decrypt_bits(sk, out.cpu().numpy().view(np.uint32))
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    assert np.array_equal(dec, want), (cfg, opts)
    return ctx, sk, P


ctx0, sk0, P0 = gates(0, 16)
gates(0, 16, ks_kernel="imma")
ctx1, sk1, P1 = gates(1, 64)
gates(1, 64, engine="ntt")
gates(1, 64, ks_kernel="imma")
# a C0 layer through the scheduler
px = np.random.default_rng(1).integers(0, 256, (5, 5, 1))
wq = si.log_quant_weights(2, (2, 3, 3, 1), layer=5)
bits = ((px[..., None] >> np.arange(8)) & 1).astype(np.uint8)
x = torch.from_numpy(she.she_encrypt_bits(sk0, bits.ravel(), 7, 0).view(np.int32)).cuda()
h, w = she.she_conv_shift_acc(ctx0, x.reshape(5, 5, 1, 8, P0.stride), 5, 5, 1, 8, False, wq, 1, 1,
                              16, relu=True)
torch.cuda.synchronize()
# leveled CMuxes
sel = she.lvl_encrypt_selectors(sk1, np.array([0, 1, 1, 0], np.uint8), 3, 0)
sd = she.lvl_selectors_to_device(ctx1, sel)
d = torch.zeros((8, 2, P1.N), dtype=torch.int32, device="cuda")
out = she.lvl_cmux_batch(ctx1, sd, torch.tensor([0, 1, 2, 3, 3, 2, 1, 0], dtype=torch.int32,
                                                device="cuda"), d, d.clone())
torch.cuda.synchronize()
print("sanitize workload done")
