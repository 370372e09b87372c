#!/usr/bin/env python
"""Benchmark: bootstrapped TFHE gates/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl she|reference]

A step is one pass of the whole hot path (gate prologue,
blind rotation, sample extract, MUX combine, key switch) over one batch of
config 1: 4096 independent gates at the TFHE default parameters (N=1024,
n=500, Bg=2^10, l=2, key switching 2^2 x 8), ops uniform over
NAND/AND/OR/XOR/XNOR/MUX, input bits uniform (she_inputs).
Inputs are resident in HBM when the timed region starts; L2 is flushed
(256 MiB write) between timed steps, outside the per-step CUDA-event pairs.

N > 1 (torchrun, or `--gpus N` alone: bench.py then launches the N ranks
itself): the 4096 gates are split across the ranks (4096/N each) and the
output LWEs are all-gathered (NCCL) inside the step — strong scaling, value =
4096 / max-over-ranks device time; the weak-scaled figure (every rank its own
4096-gate batch, no collective) is reported beside it as "weak_scaled".

--impl reference: the CPU oracle (oracle/, schoolbook TFHE) timed on this
box's host cores on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import she_inputs as si  # noqa: E402

METRIC = "bootstrapped gates/s"
UNIT = "gates/s"
CFG = 1
COUNT = 4096
# FP64 engine (N = 1024): FP64 instructions (DADD, DMUL, DFMA
# one each) per CMux of one lane: 4 forward + 4 inverse 512-point FFTs x 17920
# (passes A and B, folding twist, int<->double conversions) + pointwise
# 512 x 4 x 16 = 176,128; ncu's DADD + DMUL + DFMA count: 176,129
FP64_OPS_PER_CMUX = 8 * 17_920 + 512 * 4 * 16
# The work unit above is fixed (the round-1 transform's count, DESIGN.md
# §4.2b), so the fraction measures useful work per second whichever transform
# runs.  FP64 instructions the default transform (v2, §4.2c) actually executes
# per CMux and lane, from ncu (profiles/r2/: DADD + DMUL + DFMA / lanes / n):
FP64_EXECUTED_PER_CMUX = {1: 176_129, 2: 183_875, 8: 171_074}  # 8: the TMEM engine, transform 3 (ncu, r2 tm10)
# A lower bound on the FP64 instructions of one CMux of one lane, for scale:
# 8 complex 512-point transforms at the best known real-flop count (split
# radix, 4 M log2 M - 6 M + 8 = 15,368 flops) with every instruction a fused
# multiply-add (2 flops), plus the pointwise sum (4 DFMA per complex
# multiply-add, 512 x 4 outputs x 4 rows) = 8 x 7,684 + 32,768 = 94,240.
TM_DEFAULT_CHUNK = 32  # include/she.h she_ctx_options.fft_chunk default
FP64_LOWER_BOUND_PER_CMUX = 8 * (4 * 512 * 9 - 6 * 512 + 8) // 2 + 512 * 4 * 4 * 4
MODMUL_PER_LANE = {1024: 19_456_000, 256: 1_048_576}  # n[(k+1)l+(k+1)](N/2)log2N + n(k+1)l(k+1)N
WORKLOAD = ("config1: 4096 independent bootstrapped gates, ops uniform over "
            "NAND/AND/OR/XOR/XNOR/MUX, uniform input bits; TFHE N=1024 k=1 n=500 "
            "Bg=2^10 l=2 ks 2^2x8 alpha_lwe=2.44e-5 alpha_bk=3.73e-9 (torus32)")


def set_count(n: int) -> None:
    global COUNT
    COUNT = n


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# roofline peak: Goldilocks modmuls per second the ALUs can issue
# ---------------------------------------------------------------------------
def modmul_sass_instructions(lib_path: str) -> float | None:
    """SASS instructions per gl::mul_le (the kernel's general multiply), from
    the K6 loop body of libshe.so (non-uniform-datapath instructions of the
    one-iteration loop / 8 independent chains)."""
    try:
        sass = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True,
                              timeout=120).stdout
    except (OSError, subprocess.TimeoutExpired):
        return None
    m = re.search(r"Function : \S*modmul_peak_kernel\S*\n(.*?)(?:\n\s*Function :|\Z)", sass, re.S)
    if not m:
        return None
    lines = re.findall(r"/\*([0-9a-f]{4,6})\*/\s+([^;]+);", m.group(1))
    ins = [(int(a, 16), t.strip()) for a, t in lines]
    back = [(a, t) for a, t in ins if t.split()[0].endswith("BRA.U") and not t.startswith("@")]
    for a, t in back:
        tgt = int(t.split(",")[-1].strip(), 16)
        if tgt < a:
            body = [x for addr, x in ins if tgt <= addr < a]
            vec = [x for x in body if not re.match(r"^(@!?U?P\d+\s+)?U", x) and not x.startswith("NOP")]
            return len(vec) / 8.0
    return None


def roofline_peak(device: int, lib_path: str, sm_max_mhz: float | None):
    import torch
    from paper_1906_00148_b200 import she
    props = torch.cuda.get_device_properties(device)
    sms = props.multi_processor_count
    f = (sm_max_mhz or 1965.0) * 1e6
    measured, _ = she.modmul_peak(device)
    ipm = modmul_sass_instructions(lib_path)
    # 4 SMSPs x 32 lanes issue one instruction per clock each (B300_MICROARCH.md)
    derived = sms * 4 * 32 * f / ipm if ipm else None
    peak = max(x for x in (derived, measured) if x)
    src = (f"max(derived {derived / 1e9:.0f} = {sms} SM x 128 lanes/clk x {f / 1e6:.0f} MHz / "
           f"{ipm:.1f} SASS instr per modmul, K6 measured {measured / 1e9:.0f}) Gmodmul/s"
           if derived else f"K6 measured {measured / 1e9:.0f} Gmodmul/s")
    return peak, measured, derived, ipm, src


def read_ncu_summary(kernel: str = "br_kernel"):
    """Instruction-level evidence of the dominant kernel from the committed ncu
    capture (profiles/ncu_summary.json): issue-slot and pipe utilisation."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            br = json.load(f)[kernel]
        return {k: v for k, v in br.items() if k.endswith("_pct") or k.endswith("_per_launch")}
    except (OSError, ValueError, KeyError):
        return None


def read_profile_traffic(kernel: str = "br_kernel"):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(f"{kernel}_dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# the product arm
# ---------------------------------------------------------------------------
def _bits_of(v, width: int) -> np.ndarray:
    """Client-side word encoding: two's-complement bits, LSB first."""
    v = np.asarray(v, dtype=np.int64)
    return ((v[..., None] >> np.arange(width)) & 1).astype(np.uint8)


def _value_of(bits, signed: bool) -> np.ndarray:
    """Client-side word decoding (inverse of _bits_of)."""
    bits = np.asarray(bits, dtype=np.int64)
    w = bits.shape[-1]
    v = (bits << np.arange(w)).sum(axis=-1)
    return np.where(bits[..., -1] == 1, v - (1 << w), v) if signed else v


def net_latency(ctx, sk, P, world: int, rank: int, tcn: bool = False):
    """BASELINE.json's second metric: latency of the encrypted MNIST-shaped net
    (configs[3]: conv 5x5/2 1->5 + ReLU, FC 720->100 + ReLU, FC 100->10) at the
    default parameters, device-resident input ciphertexts -> device-resident
    encrypted logits.  Host scheduling of each layer (circuit build from the
    plaintext weights, levelisation) runs inside the timed region (not
    precompiled).  N > 1: every layer's output words are split across ranks
    (neuron-affine) and all-gathered over NCCL before the next
    layer.  The decrypted logits are reported (client decryption); their
    equality with the plaintext network is a GPU test
    (tests/test_gpu_layers.py::test_config3_full_at_default_params)."""
    import torch
    import torch.distributed as dist
    from paper_1906_00148_b200 import she

    cfg = 3
    px = si.pixels(cfg, (28, 28, 1)).astype(np.int64)
    # SHE: log-quantised codes; TCN (--tcn): 8-bit
    # fixed-point multipliers by shift-and-add on the same engine
    gen = si.tcn_weights if tcn else si.log_quant_weights
    w1 = gen(cfg, (5, 5, 5, 1), layer=0)
    w2 = gen(cfg, (100, 720), layer=1)
    w3 = gen(cfg, (10, 100), layer=2)
    conv_call, fc_call = ((she.she_conv_mul_acc, she.she_fc_mul_acc) if tcn
                          else (she.she_conv_shift_acc, she.she_fc_shift_acc))
    conv_w, fc_w = (she.conv_mul_width, she.fc_mul_width) if tcn else (she.conv_width, she.fc_width)
    stride = P.stride
    bits = _bits_of(px, 8)
    t_enc = time.perf_counter()  # client side (host): the paper's EDL column
    cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(cfg), 0)
    t_enc = time.perf_counter() - t_enc
    t_ser = time.perf_counter()  # the message the client sends (MSize)
    wire = she.serialize(P, cts)
    cts = she.deserialize(P, wire)
    t_ser = time.perf_counter() - t_ser
    x = torch.from_numpy(cts.view(np.int32)).cuda().reshape(28, 28, 1, 8, stride)

    from paper_1906_00148_b200.parallel import gather_shards, max_over_ranks, padded_words

    def sharded(words, width):
        return torch.zeros((padded_words(words, world), width, stride), dtype=torch.int32,
                           device="cuda"), words

    def gather(buf, words):
        return gather_shards(buf, words, rank, world)

    wa = conv_w(28, 28, 1, 8, False, w1, 2, 0, 16, relu=True)
    wb = fc_w(720, wa, False, w2, 16, relu=True)
    wc = fc_w(100, wb, False, w3, 16)
    h1, p1 = sharded(720, wa)
    h2, p2 = sharded(100, wb)
    lo, p3 = sharded(10, wc)
    stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    conv_call(ctx, x, 28, 28, 1, 8, False, w1, 2, 0, 16, relu=True, out=h1[:720])
    s1 = she.layer_stats(ctx)
    gather(h1, p1)
    fc_call(ctx, h1[:720], 720, wa, False, w2, 16, relu=True, out=h2[:100])
    s2 = she.layer_stats(ctx)
    gather(h2, p2)
    fc_call(ctx, h2[:100], 100, wb, False, w3, 16, out=lo[:10])
    s3 = she.layer_stats(ctx)
    gather(lo, p3)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev_s = e0.elapsed_time(e1) * 1e-3
    dev_s, wall = max_over_ranks([dev_s, wall], world)
    lanes_total = sum(s["br_lanes"] for s in (s1, s2, s3))
    if world > 1:  # every rank's share, for the oracle projection of the whole net
        t = torch.tensor([float(lanes_total)], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t)
        lanes_total = int(t.item())
    out_cts = lo[:10].cpu().numpy().view(np.uint32).reshape(-1, stride)
    t_dec = time.perf_counter()
    dec_bits = she.she_decrypt_bits(sk, out_cts)
    t_dec = time.perf_counter() - t_dec
    # the same client steps on the GPU (NEXT-4): host noise + device masks,
    # bit-identical ciphertexts; device decryption of the logits
    torch.cuda.synchronize()
    g0 = time.perf_counter()
    noise = she.she_encrypt_noise(sk, bits.size, si.input_seed(cfg), 0)
    g_ct = she.she_encrypt_bits_gpu(sk, torch.from_numpy(bits.ravel().astype(np.uint8)).cuda(),
                                    torch.from_numpy(noise.view(np.int32)).cuda(),
                                    si.input_seed(cfg), 0)
    torch.cuda.synchronize()
    g_enc = time.perf_counter() - g0
    g0 = time.perf_counter()
    g_bits = she.she_decrypt_bits_gpu(sk, lo[:10].reshape(-1, stride)).cpu().numpy()
    g_dec = time.perf_counter() - g0
    gpu_client = {"encrypt_s": round(g_enc, 4), "decrypt_s": round(g_dec, 5),
                  "edl_s": round(g_enc + g_dec, 4),
                  "bit_exact_with_host_client": bool(
                      np.array_equal(g_ct.cpu().numpy().view(np.uint32), cts)
                      and np.array_equal(g_bits, dec_bits))}
    logits = _value_of(dec_bits.reshape(10, wc), signed=True)
    stats = [s1, s2, s3]
    kind = ("TCN baseline: 8-bit fixed-point multipliers (shift-and-add)" if tcn
            else "log-quantised weights")
    return {"workload": "config3: MNIST-shaped encrypted net, 28x28x1 uint8 input, conv 5x5/2 1->5 "
                        f"+ ReLU, FC 720->100 + ReLU, FC 100->10, {kind}, 16-bit "
                        "mixed-width accumulators; default TFHE parameters",
            "latency_s": round(dev_s, 3), "wall_s": round(wall, 3), "unit": "s",
            "higher_is_better": False, "host_scheduling": "inside the timed region",
            "gates_per_rank": int(sum(s["gates"] for s in stats)),
            "br_lanes_per_rank": int(sum(s["br_lanes"] for s in stats)),
            "levels": int(sum(s["levels"] for s in stats)),
            "br_lanes_total": int(lanes_total),
            "logits": [int(v) for v in logits],
            "client": {"encrypt_s": round(t_enc, 4), "decrypt_s": round(t_dec, 5),
                       "edl_s": round(t_enc + t_dec, 4),
                       "msize_bytes": len(wire), "serialize_roundtrip_s": round(t_ser, 4),
                       "note": "host client (she_encrypt_bits / she_decrypt_bits): 784 pixels x 8 "
                               "bit-wise LWE ciphertexts of n+1 = 501 words (PAPER.md:256 MSize)",
                       "gpu": gpu_client},
            "parallelism": f"neuron-sharded x{world}, {dist.get_backend()} all-gather between "
                           "layers" if world > 1 else "1 GPU"}


def dshe_latency(ctx, sk, P, world: int, rank: int, H=28, ch=4, k=4):
    """a DSHE-style deeper net (PAPER.md T3 :202-203,
    [C-B-A-C-B-A-P] x k - F - F) at the default parameters: 28x28x1 uint8
    input, 3x3 'same' convs with `ch` channels, BN lowered to shift + constant
    (she_bn_shift_add), ReLU, max-pool; FC -> 8 + ReLU, FC -> 10.  Device-
    resident input to device-resident logits, host scheduling included; the
    decrypted logits are reported (their plaintext check at this size is a
    run recorded in profiles/r1/bench_dshe_net.json; the same chain at C0 is
    a GPU test)."""
    import torch
    from paper_1906_00148_b200 import she
    from paper_1906_00148_b200.parallel import gather_shards, max_over_ranks, padded_words

    cfg, stride = 5, P.stride
    px = si.pixels(cfg, (H, H, 1)).astype(np.int64)
    blocks, cin = [], 1
    for b in range(k):
        wa = si.log_quant_weights(cfg, (ch, 3, 3, cin), layer=10 * b)
        wb = si.log_quant_weights(cfg, (ch, 3, 3, ch), layer=10 * b + 1)
        blocks.append((wa, si.bn_params(cfg, ch, 10 * b), wb, si.bn_params(cfg, ch, 10 * b + 1)))
        cin = ch
    side = H >> k
    fc1 = si.log_quant_weights(cfg, (8, side * side * ch), layer=90)
    fc2 = si.log_quant_weights(cfg, (10, 8), layer=91)
    cts = she.she_encrypt_bits(sk, _bits_of(px, 8).ravel(), si.input_seed(cfg), 0)
    x = torch.from_numpy(cts.view(np.int32)).cuda().reshape(H, H, 1, 8, stride)

    def buf(words, width):
        return torch.zeros((padded_words(words, world), width, stride), dtype=torch.int32,
                           device="cuda")

    lanes = levels = 0

    def tally():
        nonlocal lanes, levels
        st = she.layer_stats(ctx)
        lanes += st["br_lanes"]
        levels += st["levels"]

    stream = torch.cuda.current_stream()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h, Hc, C, w, signed = x, H, 1, 8, False
    for wa, bna, wb, bnb in blocks:
        for wq, bn in ((wa, bna), (wb, bnb)):
            co = wq.shape[0]
            words = Hc * Hc * co
            wc = she.conv_width(Hc, Hc, C, w, signed, wq, 1, 1, 16)
            o = buf(words, wc)
            she.she_conv_shift_acc(ctx, h, Hc, Hc, C, w, signed, wq, 1, 1, 16, out=o[:words])
            tally()
            gather_shards(o, words, rank, world)
            wbn = she.bn_width(words, co, wc, True, *bn, cap=16, relu=True)
            o2 = buf(words, wbn)
            she.she_bn_shift_add(ctx, o[:words], words, co, wc, True, *bn, cap=16, relu=True,
                                 out=o2[:words])
            tally()
            h, C, w, signed = gather_shards(o2, words, rank, world), co, wbn, False
        words = (Hc // 2) * (Hc // 2) * C
        o3 = buf(words, w)
        she.she_maxpool2x2(ctx, h, Hc, Hc, C, w, False, out=o3[:words])
        tally()
        h, Hc = gather_shards(o3, words, rank, world), Hc // 2
    w1 = she.fc_width(Hc * Hc * C, w, False, fc1, 16, relu=True)
    o4 = buf(8, w1)
    she.she_fc_shift_acc(ctx, h, Hc * Hc * C, w, False, fc1, 16, relu=True, out=o4[:8])
    tally()
    h = gather_shards(o4, 8, rank, world)
    w2 = she.fc_width(8, w1, False, fc2, 16)
    o5 = buf(10, w2)
    she.she_fc_shift_acc(ctx, h, 8, w1, False, fc2, 16, out=o5[:10])
    tally()
    lo = gather_shards(o5, 10, rank, world)
    e1.record(stream)
    torch.cuda.synchronize()
    dev_s = max_over_ranks([e0.elapsed_time(e1) * 1e-3], world)[0]
    logits = _value_of(she.she_decrypt_bits(sk, lo.cpu().numpy().view(np.uint32)
                                            .reshape(-1, stride)).reshape(10, w2), signed=True)
    return {"workload": f"DSHE-style net (NEXT-3): {H}x{H}x1 uint8, [conv3x3 {ch}ch + BN(shift+const) "
                        f"+ ReLU] x2 + maxpool, x{k} blocks, FC->8 + ReLU, FC->10; default TFHE "
                        "parameters",
            "latency_s": round(dev_s, 3), "unit": "s", "higher_is_better": False,
            "br_lanes_per_rank": int(lanes), "levels": int(levels),
            "logits": [int(v) for v in logits]}


def leveled_units(ctx, sk, P, words=720, width=16):
    """NEXT-2 leveled mode (reading R-LV): ADD, MAX and ReLU units on
    `words` client word pairs of `width` bits (the 720 accumulators of config
    2's conv layer), each a CMux program on TRGSW selectors with no
    bootstrapping; device time per unit (CUDA events), CMuxes, depth, and the
    decrypted outputs against the plaintext."""
    import torch
    from paper_1906_00148_b200 import she
    rng = np.random.default_rng(si.input_seed(2) + 77)
    lo, hi = -(1 << (width - 1)), 1 << (width - 1)
    x, y = rng.integers(lo, hi, words), rng.integers(lo, hi, words)
    bits = lambda v: ((v[:, None] >> np.arange(width)) & 1).astype(np.uint8)
    t0 = time.perf_counter()
    sel = she.lvl_encrypt_selectors(sk, np.concatenate([bits(x).ravel(), bits(y).ravel()]),
                                    si.input_seed(2) + 78, 0)
    t_enc = time.perf_counter() - t0
    sel_dev = she.lvl_selectors_to_device(ctx, sel)
    xs = np.arange(words * width, dtype=np.uint32).reshape(words, width)
    ys = xs + words * width
    res = {"workload": f"{words} client word pairs of {width} bits (config 2's conv outputs), "
                       "TRGSW selectors (N=1024, Bg=2^10, l=2, alpha_bk), TRLWE data",
           "client_selector_encrypt_s": round(t_enc, 3),
           "selector_bytes_each": int(sel[0].nbytes)}
    for name, op, ref in (("add", she.SHE_LVL_ADD, lambda: (x + y) & ((1 << width) - 1)),
                          ("max", she.SHE_LVL_MAX, lambda: np.maximum(x, y)),
                          ("relu", she.SHE_LVL_RELU, lambda: np.maximum(x, 0))):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out, n_cmux, depth = she.lvl_unit(ctx, op, sel_dev, xs, None if op == she.SHE_LVL_RELU
                                          else ys, width, True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        got = she.lvl_decrypt(sk, out.cpu().numpy().view(np.uint32)).astype(np.int64)
        v = (got << np.arange(got.shape[-1])).sum(axis=-1)
        if name == "max":
            v = np.where(got[:, -1] == 1, v - (1 << width), v)
        res[name] = {"ms": round(ms, 2), "cmux": n_cmux, "depth": depth,
                     "cmux_per_s": round(n_cmux / (ms * 1e-3), 1),
                     "decrypted_mismatches": int(np.sum(v != ref()))}
    return res


def batch_sweep(ctx, sk, P, sizes=(40, 148, 300, 512, 740, 1024, 1480, 2048, 4096, 8192, 16384, 32768)):
    """Gates/s against the batch size (config-1 gates): where the persistent
    kernel's pipelines fill the 148 SMs and how narrow levels of a circuit run
    (`--sweep`); 512 / 1024 / 2048 gates are one rank's shard of config 1 on
    8 / 4 / 2 GPUs."""
    import torch
    from paper_1906_00148_b200 import she
    res = []
    big = max(sizes)
    ops = si.gate_ops(CFG, big)
    bits = si.gate_input_bits(CFG, big)
    cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(CFG), 0).reshape(big, 3, -1)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).cuda()
    d_ops = dev(np.pad(ops, (0, (-big) % 4)))
    d_a, d_b, d_c = (dev(cts[:, j].copy()) for j in range(3))
    out = torch.empty((big, P.stride), dtype=torch.int32, device="cuda")
    for n in sizes:
        run = lambda: she.she_gate_batch_ops(ctx, d_ops[: (n + 3) // 4].view(torch.uint8)[:n],
                                             d_a[:n], d_b[:n], d_c[:n], out[:n])
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(1, 8192 // n)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res.append({"gates": n, "br_lanes": si.br_lanes(ops[:n]), "ms": round(ms, 3),
                    "gates_per_s": round(n / (ms * 1e-3), 1)})
    return res


def engine_options(args) -> dict:
    """she_ctx_options from the command line (all engines are exact; A/B only)."""
    opts = {}
    if args.engine != "default":
        opts["engine"] = args.engine
    if args.fft_lanes:
        opts["fft_lanes"] = args.fft_lanes
    if args.fft_variant:
        opts["fft_variant"] = args.fft_variant
    if args.fft_groups:
        opts["fft_groups"] = args.fft_groups
    if args.fft_prefetch:
        opts["fft_prefetch"] = args.fft_prefetch
    if args.fft_streams:
        opts["fft_streams"] = args.fft_streams
    if args.fft_store != "default":
        opts["fft_store"] = args.fft_store
    if args.fft_stagger_ns:
        opts["fft_stagger_ns"] = args.fft_stagger_ns
    if args.fft_chunk:
        opts["fft_chunk"] = args.fft_chunk
    if args.ks_kernel != "default":
        opts["ks_kernel"] = args.ks_kernel
    return opts


def run_she(args):
    import torch
    import torch.distributed as dist
    from paper_1906_00148_b200 import she
    from paper_1906_00148_b200 import parallel
    from paper_1906_00148_b200.parallel import max_over_ranks

    world, rank, local = dist_env()
    # SHE_BENCH_BACKEND=gloo runs the N ranks with gloo collectives (CPU
    # staging), e.g. several ranks on one GPU: a functional check of the N > 1
    # code path (its timings say nothing about NVLink).
    backend = os.environ.get("SHE_BENCH_BACKEND", "nccl")
    ndev = max(1, torch.cuda.device_count())
    local = int(os.environ.get("SHE_BENCH_DEVICE", local % ndev))
    if world > 1:
        if backend == "nccl":
            # communicator set-up lines on stderr (the JSON line stays alone on stdout)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    P = si.CONFIG_PARAMS[CFG]
    sk, ck = she.she_keygen(P, si.key_seed(CFG))
    ctx = she.Context(P, ck, device=local, rank=rank, world=world, **engine_options(args))
    ops = si.gate_ops(CFG, COUNT)
    bits = si.gate_input_bits(CFG, COUNT)
    stride = P.stride
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).cuda()
    # the config-1 batch, identical on every rank; rank r evaluates its shard
    # [r*per, (r+1)*per) and the output LWEs are all-gathered (strong scaling)
    cts = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(CFG), 0).reshape(COUNT, 3, -1)
    lo, hi, per = parallel.shard(COUNT, rank, world)
    lanes = si.br_lanes(ops)
    lanes_rank = si.br_lanes(ops[lo:hi])
    d_ops = torch.from_numpy(ops.astype(np.uint8)).cuda()
    d_a, d_b, d_c = (dev(cts[:, j].copy()) for j in range(3))
    d_out = torch.zeros((parallel.padded_words(COUNT, world), stride), dtype=torch.int32,
                        device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        parallel.gate_batch_sharded(ctx, d_ops, d_a, d_b, d_c, d_out, rank, world, stream)

    peak, k6, derived, ipm, peak_src = roofline_peak(local, she.LIB_PATH, None)
    engine = she.br_engine(ctx)
    fp64_peak = she.fp64_peak(local)[0] if engine else None

    def timed(fn, steps, kernel_timing=False):
        """K steps bracketed by a barrier + synchronize, one CUDA-event pair per
        step on the launch stream, L2 flushed between steps (outside the pairs);
        returns the max over ranks of the summed device time (ms)."""
        if kernel_timing:
            ctx.enable_timing(True)
            ctx.timing(reset=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(steps)]
        for k in range(steps):
            flush.zero_()
            evs[k][0].record(stream)
            fn()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = None
        if kernel_timing:
            ctx.enable_timing(False)
            t = ctx.timing(reset=True)
        return max_over_ranks([sum(a.elapsed_time(b) for a, b in evs)], world)[0], t

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: the strong-scaled config-1 step ----
    clocks = ClockSampler(local)
    clocks.start()
    ctx.kernel_launches(reset=True)
    dev_ms, t = timed(step, args.steps, kernel_timing=True)
    launches = ctx.kernel_launches(reset=True)
    clk = clocks.stop()
    ms_per_step = dev_ms / args.steps
    value = COUNT * args.steps / (dev_ms * 1e-3)
    gpu_out = d_out[:COUNT].cpu().numpy().view(np.uint32).copy()

    # ---- weak scaling beside it: every rank its own 4096-gate batch ----
    weak = None
    if world > 1:
        cts_w = she.she_encrypt_bits(sk, bits.ravel(), si.input_seed(CFG),
                                     3 * COUNT * rank).reshape(COUNT, 3, -1)
        w_a, w_b, w_c = (dev(cts_w[:, j].copy()) for j in range(3))
        w_out = torch.zeros((COUNT, stride), dtype=torch.int32, device="cuda")
        step_w = lambda: she.she_gate_batch_ops(ctx, d_ops, w_a, w_b, w_c, w_out, stream)
        step_w()
        w_ms, _ = timed(step_w, args.steps)
        weak = {"value": round(world * COUNT * args.steps / (w_ms * 1e-3), 2), "unit": UNIT,
                "gates_per_rank": COUNT, "ms_per_step": round(w_ms / args.steps, 3),
                "note": "every rank evaluates its own 4096-gate batch (inputs encrypted at a "
                        "rank-offset ordinal), no collective; value = all ranks' gates / "
                        "max-over-ranks device time"}

    # dominant kernel: the blind rotation (K2+K3), this rank's shard
    br_ms_per_launch = t["br_ms"] / max(1, t["br_launches"])
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    common = {"kernel_ms_per_launch": round(br_ms_per_launch, 3),
              "kernel_share_of_step": round(t["br_ms"] / dev_ms, 4) if dev_ms else None,
              "ks_kernel_ms_per_launch": round(t["ks_ms"] / max(1, t["ks_launches"]), 3),
              "lanes_per_launch": lanes_rank}
    if engine:  # FP64 FFT engine: bound by the FP64 pipe
        fp64_ops = lanes_rank * P.n * FP64_OPS_PER_CMUX
        achieved = fp64_ops / (br_ms_per_launch * 1e-3)
        # lanes resident per round: the TMEM engine 8 per SM (4 pipelines x 2),
        # fft2x2 2 CTAs of 2 lanes, else G lanes per CTA, one CTA per SM
        slots = sms * engine * (2 if engine == 2 else 1)
        kname = "br_fft_tm_kernel" if engine == 8 else "br_fft_kernel"
        rounds = -(-lanes_rank // slots)
        wave = {"lanes": lanes_rank, "slots_per_round": slots, "rounds": rounds,
                "last_round_fill": round(lanes_rank / slots - (rounds - 1), 3)}
        if engine == 8 and args.fft_chunk != -1 and lanes_rank > 4 * sms:
            # the TMEM engine splits units (lane pairs; single lanes up to 1.65 per pipeline)
            # in time (she_ctx_options.fft_chunk, csrc/tm_queue.h)
            singles = lanes_rank * 100 <= 4 * sms * 165
            units = lanes_rank if singles else -(-lanes_rank // 2)
            if singles or lanes_rank > 2 * 4 * sms:
                wave = {"lanes": lanes_rank, "unit": "lane" if singles else "lane pair", "units": units,
                        "pipelines": 4 * sms}
                if args.fft_chunk == -2:
                    wave["wrap_around_schedule"] = {
                        "iterations_per_pipeline": round(units * P.n / (4 * sms), 1),
                        "handovers": 4 * sms}
                else:
                    chunk = args.fft_chunk or TM_DEFAULT_CHUNK
                    items = units * -(-P.n // chunk)
                    wave["chunk_queue"] = {"chunk_cmux": chunk, "items": items,
                                           "item_rounds": round(items / (4 * sms), 2)}
        roof = {"bound": "fp64", "achieved": round(achieved / 1e12, 3),
                "peak": round(fp64_peak / 1e12, 3), "unit": "T FP64-instr/s",
                "frac": round(achieved / fp64_peak, 4), "traffic": read_profile_traffic(kname),
                "kernel": (("br_fft_tm_kernel (four two-lane pipelines per SM, spectra in TMEM)"
                            if engine == 8 else f"br_fft_kernel<{engine}>")
                           + ": gate prologue + blind rotation by exact FP64 FFT + sample extract"),
                "algorithmic_per_launch": f"{lanes_rank} BR lanes x {P.n} CMux x {FP64_OPS_PER_CMUX} "
                                          "FP64 instr (DESIGN.md §4.2b)",
                "fp64_executed_per_cmux_default_transform": FP64_EXECUTED_PER_CMUX[8 if engine == 8 else 2],
                "frac_of_executed": round(lanes_rank * P.n * FP64_EXECUTED_PER_CMUX[8 if engine == 8 else 2]
                                          / (br_ms_per_launch * 1e-3) / fp64_peak, 4),
                "fp64_lower_bound_per_cmux": FP64_LOWER_BOUND_PER_CMUX,
                "frac_of_lower_bound": round(lanes_rank * P.n * FP64_LOWER_BOUND_PER_CMUX
                                             / (br_ms_per_launch * 1e-3) / fp64_peak, 4),
                **common,
                "wave_rounds": wave,
                "peak_source": f"K7 measured {fp64_peak / 1e12:.2f} T DFMA/s on {sms} SMs "
                               "(nominal 64 FP64 lanes/SM/clk)",
                "ntt_engine_equivalent": {"achieved_gmodmul_s": round(lanes_rank * MODMUL_PER_LANE[P.N] / (br_ms_per_launch * 1e-3) / 1e9, 1),
                                          "ntt_peak_gmodmul_s": round(peak / 1e9, 1)},
                "ncu_profile": read_ncu_summary(kname)}
    else:
        achieved = lanes_rank * MODMUL_PER_LANE[P.N] / (br_ms_per_launch * 1e-3)
        roof = {"bound": "alu", "achieved": round(achieved / 1e9, 2), "peak": round(peak / 1e9, 2),
                "unit": "Gmodmul/s", "frac": round(achieved / peak, 4), "traffic": read_profile_traffic(),
                "kernel": "br_kernel (gate prologue + blind rotation + sample extract)",
                "algorithmic_per_launch": f"{lanes_rank} BR lanes x {MODMUL_PER_LANE[P.N]} modmul",
                **common,
                "peak_source": peak_src, "ncu_profile": read_ncu_summary()}

    # the key switch's own roofline: the tcgen05 kind::i8 product (DESIGN.md
    # §4.3) of a (gates padded to 128) x 24N one-hot matrix and the key's
    # (stride x 4 planes) columns, against the int8 dense tensor peak = the
    # measured bf16 peak x 2 (the nominal int8 / bf16 ratio, 4.5 / 2.25 PF)
    ks_ms = t["ks_ms"] / max(1, t["ks_launches"])
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bf16 = float(json.load(f)["bf16_tflops"])
        src = "MEASURED_PEAKS.json bf16_tflops (burst) x 2"
    except (OSError, ValueError, KeyError):
        bf16, src = 1590.0, "B200_PROFILING.md fallback 1.59 PF bf16 x 2"
    gemm_ops = 2.0 * (-(-(hi - lo) // 128) * 128) * (stride * 4) * (24 * P.N)
    roof["key_switch"] = {"bound": "tensor", "kernel": "ksi_gemm_tc (tcgen05.mma kind::i8, TMEM)",
                          "ms_per_launch": round(ks_ms, 4),
                          "achieved": round(gemm_ops / (ks_ms * 1e-3) / 1e12, 1),
                          "peak": round(2 * bf16, 1), "unit": "T int8-op/s",
                          "frac": round(gemm_ops / (ks_ms * 1e-3) / 1e12 / (2 * bf16), 4),
                          "peak_source": src,
                          "note": "ks_ms spans the prep, GEMM and combine launches"}

    # ---- end to end through the public host-buffer API (H2D + D2H inside) ----
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
    h_ops = pin((COUNT,), torch.uint8)
    h_ops[:] = ops
    h_in = [pin((COUNT, stride), torch.int32).view(np.uint32) for _ in range(3)]
    for j in range(3):
        h_in[j][:] = cts[:, j]
    h_out = pin((COUNT, stride), torch.int32).view(np.uint32)
    if world == 1:  # the library's own host-buffer call
        e2e_call = lambda: she.she_gate_batch_ops_host(ctx, h_ops, *h_in, h_out, stream)
        h2d = COUNT + 3 * COUNT * stride * 4
        api = "she_gate_batch_ops_host (libshe.so): H2D, gates, D2H, stream sync"
    else:  # each rank copies its shard in, all-gather on the devices, full result out
        stage = parallel.make_stage(COUNT, stride, world)
        e2e_call = lambda: parallel.gate_batch_sharded_host(ctx, h_ops, *h_in, h_out, rank, world,
                                                            stage)
        h2d = (hi - lo) * (1 + 3 * stride * 4)
        api = ("parallel.gate_batch_sharded_host: per-rank shard H2D, she_gate_batch_ops, "
               f"{backend} all-gather, full result D2H")
    e2e_call()  # warm
    e2e_s = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_call()
        e2e_s.append(time.perf_counter() - t0)
    e2e_total = max_over_ranks([sum(e2e_s)], world)[0]
    # correctness of this run: the e2e output equals the device path's, and
    # every gate decrypts to its truth-table value
    assert np.array_equal(h_out, gpu_out), "e2e output differs"
    dec = she.she_decrypt_bits(sk, h_out)
    want = np.array([si.truth(o, *b) for o, b in zip(ops, bits)])
    assert np.array_equal(dec, want), "decryption mismatch"
    decrypted = {"decrypted_compared": int(COUNT), "decrypted_mismatches": int(np.sum(dec != want))}
    e2e = {"value": round(COUNT * args.steps / e2e_total, 2), "unit": UNIT,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(COUNT * stride * 4),
           "api": api}

    line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if engine else "u64",
            "data": "synthetic (seeded she_inputs; keys 1001, inputs 2001, ops 4001)",
            "config": {"workload": WORKLOAD, "gates": COUNT, "br_lanes": lanes,
                       "gates_per_rank": hi - lo, "br_lanes_per_rank": lanes_rank,
                       "parallelism": (f"gate-sharded x{world}: {per} gates per rank, output LWEs "
                                       f"all-gathered over {backend} inside the step"
                                       if world > 1 else "1 GPU"),
                       "l2": "flushed between timed steps (256 MiB write), outside the event pairs"},
            "br_lanes_per_s": round(lanes * args.steps / (dev_ms * 1e-3), 1),
            "parity": decrypted,
            "roofline": roof, "clocks": clk, "e2e": e2e,
            "gpu_launches": int(launches),  # this library's kernels in the timed region
            "k6_modmul_peak_per_s": round(k6, 1)}
    if weak:
        line["weak_scaled"] = weak
    if not args.no_net:
        line["net_latency"] = net_latency(ctx, sk, P, world, rank)
        if engine:
            line["leveled_units"] = leveled_units(ctx, sk, P)
    if args.tcn:
        line["tcn_net_latency"] = net_latency(ctx, sk, P, world, rank, tcn=True)
    if args.dshe:
        line["dshe_net_latency"] = dshe_latency(ctx, sk, P, world, rank)
    if args.sweep:
        line["batch_sweep"] = batch_sweep(ctx, sk, P)
    if rank == 0 and world == 1:  # the CPU baseline is reported at N = 1 only
        line["cpu_baseline"] = cpu_baseline(args, h_out)
        if "net_latency" in line:  # the paper's FIL-style projection of the oracle
            cb = line["cpu_baseline"]
            lanes_s = cb["value"] * si.br_lanes(ops[:12 * cb["cores"]]) / min(COUNT, 12 * cb["cores"])
            line["net_latency"]["oracle_projected_s"] = round(
                line["net_latency"]["br_lanes_total"] / lanes_s, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# the CPU oracle: cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------
def _oracle_workload():
    import oracle
    P = si.CONFIG_PARAMS[CFG]
    K = oracle.keygen(P, si.key_seed(CFG))
    ops = si.gate_ops(CFG, COUNT)
    bits = si.gate_input_bits(CFG, COUNT)
    return oracle, P, K, ops, bits


def _oracle_sample(oracle, P, K, ops, bits, start: int, size: int):
    sel = np.arange(start, start + size) % COUNT
    cts = oracle.encrypt(P, K.s, bits[sel].ravel(), si.input_seed(CFG), 0).reshape(size, 3, -1)
    t0 = time.perf_counter()
    out = oracle.gates(K, ops[sel], cts[:, 0].copy(), cts[:, 1].copy(), cts[:, 2].copy())
    dt = time.perf_counter() - t0
    return out, dt


def cpu_baseline(args, gpu_out=None):
    """The oracle timed on the host cores on the first gates of the batch; when
    the GPU outputs of rank 0 are given, the same oracle outputs double as a
    word-for-word parity check of this very run."""
    oracle, P, K, ops, bits = _oracle_workload()
    cores = oracle.threads()
    size = min(COUNT, 12 * cores)
    ref, dt = _oracle_sample(oracle, P, K, ops, bits, 0, size)
    out = {"value": round(size / dt, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"first {size} gates of config 1 ({si.br_lanes(ops[:size])} BR lanes), "
                     f"{dt:.1f} s wall, schoolbook negacyclic products, OpenMP over gates, "
                     f"gcc {oracle.COMPILER_FLAGS} {oracle.lib().variant}"}
    if gpu_out is not None:
        bad = int(np.sum(np.any(gpu_out[:size] != ref, axis=1)))
        out["parity"] = {"ciphertexts_compared": size, "ciphertext_mismatches": bad}
    import platform
    try:
        model = [ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo")
                 if ln.startswith("model name")][0]
    except (OSError, IndexError):
        model = platform.processor()
    out["cpu_model"] = model
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    oracle, P, K, ops, bits = _oracle_workload()
    cores = oracle.threads()
    per_step_s = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    size = max(cores, int(per_step_s * cores / 0.8))
    size = min(size, COUNT)
    for w in range(args.warmup):
        _oracle_sample(oracle, P, K, ops, bits, w * size, size)
    times = []
    for k in range(args.steps):
        _, dt = _oracle_sample(oracle, P, K, ops, bits, (args.warmup + k) * size, size)
        times.append(dt)
    total = sum(times)
    value = size * args.steps / total
    sample = f"{size} gates of config 1 per step ({size} of the 4096-gate batch), host cores"
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * total / args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "gates_per_step": size}, "impl": "reference",
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="she", choices=["she", "reference"])
    ap.add_argument("--no-net", action="store_true",
                    help="skip the encrypted MNIST-shaped net latency (config 3, ~1.5 min)")
    ap.add_argument("--tcn", action="store_true",
                    help="also time the TCN baseline of the same net (fixed-point multipliers)")
    ap.add_argument("--dshe", action="store_true",
                    help="also time a DSHE-style deeper net with batch norm (NEXT-3)")
    ap.add_argument("--sweep", action="store_true",
                    help="also report gates/s against the batch size")
    ap.add_argument("--engine", default="default", choices=["default", "fft", "ntt"],
                    help="blind-rotation engine (she_ctx_options; A/B measurements only)")
    ap.add_argument("--fft-lanes", type=int, default=0,
                    help="FFT engine lanes per CTA (she_ctx_options.fft_lanes)")
    ap.add_argument("--fft-variant", type=int, default=0,
                    help="FFT engine transform (she_ctx_options.fft_variant: 1 round-1, 2 v2)")
    ap.add_argument("--fft-groups", type=int, default=0,
                    help="FFT engine independent lane groups per CTA (she_ctx_options.fft_groups)")
    ap.add_argument("--fft-prefetch", type=int, default=0,
                    help="BK planes prefetched before the pointwise barrier (she_ctx_options)")
    ap.add_argument("--fft-streams", type=int, default=0,
                    help="FFT engine lanes per warp (she_ctx_options.fft_streams: 1 or 2)")
    ap.add_argument("--fft-store", default="default", choices=["default", "smem", "tmem"],
                    help="FFT engine spectra store (she_ctx_options.fft_store): shared or tensor memory")
    ap.add_argument("--fft-stagger-ns", type=int, default=0,
                    help="TMEM engine: start delay per quarter pipeline (ns)")
    ap.add_argument("--fft-chunk", type=int, default=0,
                    help="TMEM engine: 0 chunk queue of 32 CMux iterations per item (default), N > 0 that "
                         "queue with N, -1 static lane split, -2 wrap-around schedule")
    ap.add_argument("--ks-kernel", default="default", choices=["default", "general", "cuda", "imma", "tcgen05"],
                    help="key-switch kernel (she_ctx_options.ks_kernel)")
    ap.add_argument("--count", type=int, default=COUNT,
                    help="gates per step (default: config 1's 4096; other values are A/B only)")
    args = ap.parse_args()
    set_count(args.count)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # no external launcher: run the N ranks ourselves (one process per GPU)
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}\n")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_she(args)


if __name__ == "__main__":
    main()
