/*
 * she.h — C-ABI of the B200-native batched TFHE gate-bootstrapping engine for
 * SHE (arxiv 1906.00148): "Shift-accumulation-based LHE-enabled deep neural
 * network", whose ReLU units, max-pool units, shifts and mixed-bitwidth
 * accumulators are circuits of bootstrapped TFHE Boolean gates.
 *
 * Paper passages the calls follow (PAPER.md line, section):
 *   client encrypts / server computes blind / client decrypts  :17, :29 (§1, §2)
 *   epsilon(x, k) / delta(c, k), homomorphic gates, bootstrapping  :31 (§2)
 *   TFHE over the torus; TLWE / TRLWE / TRGSW                   :35, :188 (§2, §4)
 *   any 2-input gate (AND, OR, NOT, MUX); >2 inputs split        :110 (§3.1)
 *   ReLU and max-pool units                                     :92, :110 (F2)
 *   log-quantised weights; shift = ciphertext rewiring           :118, :142 (§3.2)
 *   mixed-bitwidth accumulator (b+n bits at level n)             :147, :149 (§3.3)
 * TFHE internals are not in the paper; conventions R1-R10 are listed in
 * DESIGN.md §2.
 *
 * Conventions shared by every call
 * --------------------------------
 *  - Torus32: a torus element x in R/Z is the uint32 round(x * 2^32).
 *  - LWE slot: uint32[she_lwe_stride(p)] = a[0..n-1], b at [n], zero padding.
 *    A bit m is encrypted with phase b - <a,s> = (m ? +1/8 : -1/8) + noise.
 *  - Encrypted word: [width][stride] slots, LSB first, two's complement.
 *  - Host pointers ("host") are ordinary CPU memory; device pointers
 *    ("device") are CUDA global memory on the context's device (e.g. torch
 *    tensors); every device call is asynchronous on the given stream.
 *  - Ownership: the caller owns every buffer passed in; the library owns its
 *    keys, contexts and scratch, released by the matching *_free / _destroy.
 *  - Errors: every call returns she_status; no exception crosses the ABI;
 *    she_last_error() gives a thread-local message for the last failure.
 *    Asynchronous device faults surface at the next call that synchronises.
 *  - count == 0 is a no-op returning SHE_OK.
 */
#ifndef SHE_H_
#define SHE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SHE_OK = 0,
  SHE_ERR_ARG = -1,    /* null pointer, bad op, overlap, out-of-range value */
  SHE_ERR_PARAMS = -2, /* unsupported parameter set (see she_params)        */
  SHE_ERR_SHAPE = -3,  /* inconsistent shapes in a layer call               */
  SHE_ERR_CUDA = -4,   /* CUDA runtime error (message in she_last_error)    */
  SHE_ERR_NCCL = -5,   /* collective failure                                */
  SHE_ERR_OOM = -6,    /* device or host allocation failed                  */
  SHE_ERR_STATE = -7   /* call not valid in the current context state       */
} she_status;

/* Gate codes.  MUX(a, b, c) = a ? b : c (SPEC.md:128 argument order). */
typedef enum {
  SHE_AND = 0, SHE_NAND = 1, SHE_OR = 2, SHE_NOR = 3, SHE_XOR = 4, SHE_XNOR = 5,
  SHE_MUX = 6, /* 2 blind rotations + 1 key switch (R6)          */
  SHE_NOT = 7, /* -a, no bootstrapping                                     */
  SHE_COPY = 8 /* a, no bootstrapping                                      */
} she_op;

/* TFHE gate-bootstrapping parameters (BASELINE.json configs).  Supported:
 * k = 1; N in {256, 1024}; 1 <= n <= 511 (an LWE slot of n + 1 words padded
 * to 32 fits the key-switch kernels); l = 2; l * bg_bits < 32; ks_base_bits =
 * 2, ks_t * ks_base_bits < 32; exactness (k+1) l N (Bg/2) 2^31 < (p-1)/2 for
 * p = 2^64 - 2^32 + 1.  Anything else is SHE_ERR_PARAMS. */
typedef struct {
  uint32_t N, k, n, bg_bits, l, ks_base_bits, ks_t;
  double alpha_lwe, alpha_bk;
} she_params;

typedef struct she_secret_key she_secret_key;
typedef struct she_cloud_key she_cloud_key;
typedef struct she_ctx she_ctx;

/* Words per LWE slot: n+1 rounded up to a multiple of 32 (C0: 160, C1: 512). */
size_t she_lwe_stride(const she_params* p);

const char* she_last_error(void);

/* ---- client side (host only) -------------------------------------------- */

/* Keygen from a seed (DESIGN.md §3 random-stream layout; R1-R3).  Secret key
 * s in {0,1}^n, TRLWE key S in {0,1}^N; cloud key = bootstrapping key
 * BK_i = TRGSW_S(s_i) (uint32[n][2l][2][N], row r = c*l + j) and key-switching
 * key KSK[i][j][v] = LWE_s(v S_i 2^{32-(j+1)basebits}) (uint32[N][t][base][n+1],
 * v = 0 rows zero).  Both outputs are library-owned. */
she_status she_keygen(const she_params* p, uint64_t seed, she_secret_key** sk,
                      she_cloud_key** ck);
void she_secret_key_free(she_secret_key* sk);
void she_cloud_key_free(she_cloud_key* ck);

/* Export the documented layouts into caller buffers (host).  Pass buf = NULL
 * to query the size in bytes through *len.
 *   secret key: uint8 s[n] then uint8 S[N]
 *   cloud key : uint32 bk[n][2l][2][N] then uint32 ksk[N][t][base][n+1]      */
she_status she_secret_key_export(const she_secret_key* sk, void* buf, size_t* len);
she_status she_cloud_key_export(const she_cloud_key* ck, void* buf, size_t* len);
/* Build a cloud key from the exported layout (e.g. received from a client). */
she_status she_cloud_key_import(const she_params* p, const void* buf, size_t len,
                                she_cloud_key** ck);

/* epsilon(bits): ciphertext idx draws mask/noise number first_index + idx
 * (host buffers; out = count * stride uint32, padding zeroed). */
she_status she_encrypt_bits(const she_secret_key* sk, const uint8_t* bits, size_t count,
                            uint64_t seed, uint64_t first_index, uint32_t* out);
/* delta(c): bit = [(int32)(b - <a,s>) >= 0]  (R5). */
she_status she_decrypt_bits(const she_secret_key* sk, const uint32_t* in, size_t count,
                            uint8_t* bits);

/* Ciphertext batches on the wire (NEXT-4; the paper's MSize, PAPER.md:232,
 * :256): a 16-byte header {u32 magic "SHEC", u32 n, u64 count} followed by
 * count x (n + 1) little-endian uint32 words (a[0..n-1], b), slot padding not
 * sent: she_serialized_bytes(p, count) = 16 + 4 count (n + 1).
 * she_serialize_ciphertexts: in = count slots (host, stride words each); buf =
 * NULL queries *len; else *len is the capacity in, the size written out.
 * she_deserialize_ciphertexts: *count = the batch's count; out (host, cap
 * slots, padding zeroed) may be NULL to query.  A wrong magic or length is
 * SHE_ERR_SHAPE, another n SHE_ERR_PARAMS. */
size_t she_serialized_bytes(const she_params* p, size_t count);
she_status she_serialize_ciphertexts(const she_params* p, const uint32_t* in, size_t count,
                                     void* buf, size_t* len);
she_status she_deserialize_ciphertexts(const she_params* p, const void* buf, size_t len,
                                       uint32_t* out, size_t cap, size_t* count);

/* ---- client side on the GPU --------------------- */
/* Host: the rounded-Gaussian noise words that fresh ciphertexts first_index ..
 * first_index + count - 1 draw (stream 8 of she_rng.h), i.e. exactly what
 * she_encrypt_bits adds, so that the device encryption below reproduces the
 * host client bit for bit (the Gaussian uses libm, which differs between host
 * and device; the integer masks do not).  noise: host uint32[count]. */
she_status she_encrypt_noise(const she_secret_key* sk, size_t count, uint64_t seed,
                             uint64_t first_index, uint32_t* noise);
/* Device: encrypt count bits (device uint8[count]); masks drawn on the device
 * from stream 7, noise given (device uint32[count], from she_encrypt_noise);
 * out: device count x stride words, padding zeroed.  One warp per ciphertext,
 * asynchronous on `stream` (a cudaStream_t on CUDA `device`). */
she_status she_encrypt_bits_gpu(const she_secret_key* sk, const uint8_t* bits,
                                const uint32_t* noise, size_t count, uint64_t seed,
                                uint64_t first_index, uint32_t* out, int device, void* stream);
/* Device: decrypt count ciphertexts (device count x stride) into bits (device
 * uint8[count]), R5 rule as she_decrypt_bits.  Asynchronous on `stream`. */
she_status she_decrypt_bits_gpu(const she_secret_key* sk, const uint32_t* in, size_t count,
                                uint8_t* bits, int device, void* stream);

/* ---- server side (device) ------------------------------------------------ */

/* Engine selection of a context (she_ctx_create_ex).  Every engine and shape
 * computes the same ciphertexts bit for bit (all are exact); they differ only
 * in speed.  Zero-initialised = the defaults. */
typedef struct {
  int br_engine;  /* 0 = default: the FP64 FFT engine for N = 1024 and bg_bits
                     <= 12, else the Goldilocks NTT engine;
                     1 = FFT (SHE_ERR_ARG where it does not apply); 2 = NTT */
  int fft_lanes;  /* FFT engine: blind-rotation lanes per CTA, 0 = default (4);
                     2 (two CTAs per SM), 3, 4 or 5 */
  int ntt_lanes;  /* NTT engine: lanes per CTA x CTAs per SM, 0 = default 5 x 1; */
  int ntt_ctas;   /*   the instantiated shapes are 5x1, 4x1, 3x1, 2x2, 1x4      */
  int ks_kernel;  /* 0 = default; 1 = the general ks_kernel (any base-4
                     decomposition); 2 = ks2_kernel (CUDA cores, base 4, t = 8);
                     3 = the tensor-core key switch (ks_imma.cuh: 0/1 digit
                     matrix x key byte planes on mma.sync u8, base 4, t = 8),
                     4 = the same product on tcgen05 (kind::i8, TMEM) */
  int fft_variant;/* FFT engine transform: 0 = default (3 on the TMEM engine,
                     2 on the shared-memory engine), 1 = the round-1
                     transform (16-entry twiddle tables, select-based pair
                     exchange; 4 lanes per CTA only), 2 = v2,
                     3 = v2 with DIT/FMA 16-point DFTs (4 lanes, or 5 lanes
                     with fft_prefetch = 3; with fft_store = 2 the TMEM
                     engine with FMA butterflies in both directions) */
  int fft_groups; /* FFT engine: independent lane groups per CTA, 0 = default
                     (1); 2 = two groups of 2 lanes with their own pointwise
                     step and barriers (4 lanes per CTA, variant 2) */
  int fft_prefetch;/* FFT engine: BK_i planes prefetched into registers before
                     the pointwise barrier: 0 = default (16), 1 = 16, 2 = 8
                     (4 or 5 lanes), 3 = none (5 lanes) */
  int fft_streams;/* FFT engine: 0 = default; 1 = one lane per warp
                     (br_fft_kernel); 2 = two lanes per warp with one lane a
                     step behind the other (br_fft2s_kernel, 4 lanes per CTA
                     on 8 warps, variant 2) */
  int fft_store;  /* FFT engine: where the digit spectra and products live
                     between the transforms: 0 = default (1); 1 = shared
                     memory (br_fft_kernel, CTA-wide pointwise step; the
                     default when any shape option above is given); 2 =
                     tensor memory (the default; br_fft_tm_kernel: four independent
                     two-lane pipelines per SM, one per sub-partition, spectra
                     in TMEM, the inverse on the forward's register layout;
                     DESIGN.md §4.2e; no other shape option applies) */
  int fft_stagger_ns;/* TMEM engine: start delay of quarter q = q x this (ns),
                     0..100000 (phase offset between the pipelines) */
  int fft_chunk;  /* TMEM engine, how batches of more than one blind-rotation
                     lane per pipeline are balanced (DESIGN.md §4.2e,
                     csrc/tm_queue.h): 0 = default, a device-wide queue of
                     (lane pair | lane, chunk of 32 CMux iterations) items;
                     1..1024 = that queue with chunks of this many iterations;
                     -1 = the static contiguous lane split only; -2 = the
                     wrap-around schedule (every pipeline the same number of
                     iterations, one accumulator hand-over per pipeline) */
  int reserved[1];/* must be 0 */
} she_ctx_options;

/* Create a context on CUDA `device`: uploads BK and KSK and transforms BK for
 * the blind-rotation engine that `opt` selects (NULL = defaults): for the FFT
 * engine into the FP64 FFT domain (each torus32 coefficient split into 16-bit
 * halves, 1/512 folded in; 65.5 MB at the default parameters; the product is
 * exact), for the NTT engine into the Goldilocks NTT domain
 * (N^-1 folded in; 32.8 MB).  Only the selected engine's BK is built.  The
 * BK of the NTT engine and of the shared-memory FFT engine gets an L2
 * persisting access-policy window on the blind-rotation launches when the
 * device allows one (cudaLimitPersistingL2CacheSize); the TMEM engine keeps
 * the part of BK in use L2-resident by its schedule instead.
 * Unknown or inapplicable option values are SHE_ERR_ARG.  rank/world describe
 * the multi-GPU group this context belongs to (world = 1 for single GPU; the
 * exchange between ranks is done by the caller's process group).
 *
 * Threading and streams: a context's scratch (extracted samples, lane list,
 * wire table, host staging) is shared by all its calls, which are serialised
 * by a mutex on the host but ordered only on the stream each call is given.
 * Use one context from one stream at a time (or synchronise between streams);
 * calls on two streams that overlap on the device race on the scratch. */
she_status she_ctx_create_ex(const she_params* p, const she_cloud_key* ck, int device, int rank,
                             int world, const she_ctx_options* opt, she_ctx** ctx);
/* she_ctx_create_ex with the default options. */
she_status she_ctx_create(const she_params* p, const she_cloud_key* ck, int device, int rank,
                          int world, she_ctx** ctx);
she_status she_ctx_destroy(she_ctx* ctx);
/* Block until all work the context enqueued has finished; reports async faults. */
she_status she_ctx_synchronize(she_ctx* ctx);

/* Per-kernel device timing for measurement (bench.py): when enabled, CUDA
 * events are recorded on the launch stream around every blind-rotation (K3)
 * and key-switch (K4) launch; she_ctx_timing synchronises on them and returns
 * the accumulated milliseconds and launch counts (reset != 0 clears them). */
she_status she_ctx_enable_timing(she_ctx* ctx, int on);
she_status she_ctx_timing(she_ctx* ctx, int reset, double* br_ms, double* ks_ms,
                          uint64_t* br_launches, uint64_t* ks_launches);

/* Kernels this library launched for the context's gate passes since the last
 * reset (lane list, blind rotation, key switch: 4 or 6 per pass; bench.py's
 * gpu_launches).  reset != 0 zeroes the counter after reading. */
she_status she_ctx_kernel_launches(she_ctx* ctx, int reset, uint64_t* count);

/* K6: peak Goldilocks modmul throughput of `device` (independent chains of the
 * kernel's own field multiplication on every SM; the roofline denominator). */
she_status she_bench_modmul_peak(int device, double* modmul_per_s, double* ms);

/* K7: peak FP64 instruction throughput of `device` (independent DFMA chains on
 * every SM, one DFMA = one op; the roofline denominator of the FFT engine). */
she_status she_bench_fp64_peak(int device, double* ops_per_s, double* ms);

/* Blind-rotation engine of a context: *fft_lanes = 8 for the FP64 FFT engine
 * with the spectra in tensor memory (br_fft_tm_kernel: 4 two-lane pipelines
 * per SM; the default for N = 1024), G = 2..5 for the shared-memory FFT engine
 * (br_fft_kernel, G lanes per CTA), 0 for the Goldilocks NTT engine
 * (br_kernel; N = 256, or br_engine = 2).  All are exact, so the outputs are
 * bit-identical. */
she_status she_ctx_br_engine(const she_ctx* ctx, int* fft_lanes);

/* Test instrumentation: evaluate the device Goldilocks primitives (hand-written
 * PTX carry chains) on n input triples (HOST buffers a, b: uint64[n]; c:
 * uint32[n]) and return out[n][104]: add, sub, add_le, sub_le (y = b), mul,
 * mul_le, reduce128_le(lo = a, hi = b), reduce_acc_le(a, b, top = c & 3),
 * shl_le(a, s) for s = 0..95.  Results are lazy residues (the *_le ones <= p). */
she_status she_field_selftest(int device, const uint64_t* a, const uint64_t* b, const uint32_t* c,
                              size_t n, uint64_t* out);

/* Test instrumentation: the FP64 engine's CMux product on caller-given inputs,
 * through the exact device code of br_fft_kernel (BK split into 16-bit halves
 * and transformed by the engine's setup kernel; forward FFT of the digit rows,
 * pointwise sum, inverse FFT, rounding, hi/lo recombination),
 * so that the exactness reading is pinned on the kernel that runs, not on a
 * model of it.  variant: the transform (she_ctx_options.fft_variant; 0 =
 * the default); 4 = the TMEM engine (fft_store = 2: bk_tm_kernel's setup, the
 * digit spectra and products in tensor memory, the register-layout inverse
 * inverse_tr; br_tmem.cuh), 5 = the TMEM engine with transform 3's FMA
 * butterflies (fft_store = 2, fft_variant = 3).  N = 1024 only.  HOST buffers:
 *   digits int32[count][4][1024]      digit rows r = c*l + j, |d| <= 2^11
 *   bk     uint32[count][4][2][1024]  torus32 BK rows (r, output o)
 *   out    uint32[count][2][1024]     out[c][o] = sum_r digits[c][r] * bk[c][r][o]
 *                                     mod (X^1024 + 1), mod 2^32
 * *worst_distance (may be NULL) = max over all cases of |v - rint(v)| for every
 * value before rounding (exactness needs < 1/2).  count <= 65535. */
she_status she_fft_product_selftest(int device, int variant, const int32_t* digits,
                                    const uint32_t* bk, size_t count, uint32_t* out,
                                    double* worst_distance);

/* Bootstrapped gates, all with the same op (north_star signature).  a, b, c,
 * out: device, count slots each (c read only for MUX, b not read for
 * NOT/COPY; unused pointers may be NULL).  out must not overlap any input.
 * stream: a cudaStream_t (NULL = legacy default stream). */
she_status she_gate_batch(she_ctx* ctx, int op, const uint32_t* a, const uint32_t* b,
                          const uint32_t* c, uint32_t* out, size_t count, void* stream);

/* Mixed-op batch: ops is a DEVICE array of count she_op codes. */
she_status she_gate_batch_ops(she_ctx* ctx, const uint8_t* ops, const uint32_t* a,
                              const uint32_t* b, const uint32_t* c, uint32_t* out,
                              size_t count, void* stream);

/* Same as she_gate_batch_ops with HOST buffers (ops, a, b, c, out): copies in,
 * evaluates, copies out and synchronises the stream (the end-to-end call). */
she_status she_gate_batch_ops_host(she_ctx* ctx, const uint8_t* ops, const uint32_t* a,
                                   const uint32_t* b, const uint32_t* c, uint32_t* out,
                                   size_t count, void* stream);

/* Wire-table level (the scheduler's unit of work): gate g reads slots
 * wires[in[3g+j] & 0x7fffffff], negated when bit 31 of in[3g+j] is set, and
 * writes slot wires[out_idx[g]].  ops, in, out_idx: DEVICE arrays. */
she_status she_gate_level(she_ctx* ctx, uint32_t* wires, const uint8_t* ops,
                          const uint32_t* in, const uint32_t* out_idx, size_t count,
                          void* stream);

/* ---- leveled mode (reading R-LV) -------
 * PAPER.md:188 evaluates its networks "in the LHE mode" with "all 3 levels of
 * TFHE": here the client's bits are TRGSW selectors (the BK_i layout,
 * uint32[2l][2][N]), the data are TRLWE (uint32[2][N], a bit = +-1/8 on the
 * constant coefficient), and a gate is a CMux with no bootstrapping, so the
 * noise grows by one external product per CMux on a data path (the depth
 * budget).  Only client-supplied bits can select, which is why
 * the leveled units below take client words.  The FFT engine (N = 1024) only. */
typedef enum { SHE_LVL_ADD = 0, SHE_LVL_MAX = 1, SHE_LVL_RELU = 2 } she_lvl_op;
/* Host, client: selectors q = first_index + idx as TRGSW_S(bits[idx]) (masks
 * stream 9, noise stream 10 of she_rng.h with alpha_bk); out: count x
 * [2l][2][N] uint32. */
she_status she_lvl_encrypt_selectors(const she_secret_key* sk, const uint8_t* bits, size_t count,
                                     uint64_t seed, uint64_t first_index, uint32_t* out);
/* Host, client: bits of count TRLWE data ciphertexts ([2][N] each). */
she_status she_lvl_decrypt(const she_secret_key* sk, const uint32_t* in, size_t count,
                           uint8_t* bits);
/* Bytes of one selector in the FFT domain (device layout of she_lvl_*). */
size_t she_lvl_selector_bytes(void);
/* Upload + transform count selectors (HOST [count][2l][2][N]) into `out`
 * (DEVICE, count * she_lvl_selector_bytes(), caller-owned). */
she_status she_lvl_selectors_to_device(she_ctx* ctx, const uint32_t* sel, size_t count,
                                       void* out, void* stream);
/* count CMuxes out[i] = d0[i] + sel[sel_idx[i]] [x] (d1[i] - d0[i]) (= sel ? d1 :
 * d0); all DEVICE: sel from she_lvl_selectors_to_device, sel_idx uint32[count],
 * d1, d0, out uint32[count][2][N] (out must not overlap d1, d0). */
she_status she_lvl_cmux_batch(she_ctx* ctx, const void* sel, const uint32_t* sel_idx,
                              const uint32_t* d1, const uint32_t* d0, uint32_t* out, size_t count,
                              void* stream);
/* Leveled units on client words (F2 circuits of the paper, PAPER.md:92, :110,
 * and its adder) as CMux programs levelised on the host: x_sel / y_sel (HOST
 * uint32[count][width]) give each bit's selector index, LSB first.
 *   SHE_LVL_ADD   out = x + y mod 2^width (ripple carry: MAJ and XOR3 as CMux
 *                 trees, 6 CMux per bit)
 *   SHE_LVL_MAX   out = max(x, y) (signed when is_signed; the comparator's
 *                 x < y flag is TRLWE data driving 3 CMux per output bit)
 *   SHE_LVL_RELU  out = relu(x) of a signed word, width - 1 bits (y unused)
 * out: DEVICE uint32[count][width or width - 1][2][N] TRLWE bits.
 * *cmux_count / *depth (may be NULL): CMuxes run and CMux levels (the
 * multiplicative depth of the unit).  Synchronous. */
she_status she_lvl_unit(she_ctx* ctx, int op, const void* sel, const uint32_t* x_sel,
                        const uint32_t* y_sel, size_t count, int width, int is_signed,
                        uint32_t* out, uint64_t* cmux_count, uint32_t* depth, void* stream);

/* ---- layer calls (§3; scheduled by the library) ------------------ */
/* Each call builds the layer's gate circuit on the host from the PLAINTEXT
 * weights (shifts = rewiring, negations = literal flags, constants folded),
 * levelises it ASAP and runs one she_gate_level per level on the device.
 *
 * Weight codes (host int8): 0 = zero weight; w = +-(e+1) means sign * 2^-e,
 * e in 0..7 (PAPER.md:118 weightQ); a term is sign * (x >> e) (R12).
 * Words: [..][width][stride] device slot arrays, LSB first.  in_signed = 0:
 * unsigned words of w_in value bits (e.g. 8-bit pixels, ReLU outputs; the
 * constant-0 sign bit is implicit); in_signed = 1: two's complement words.
 * Accumulators widen one bit per tree level up to acc_cap bits and wrap at
 * the cap (R13).
 * Output width: *w_out (in: capacity of `out` per word; out: width used).
 * Call with out == NULL to query *w_out only (host only, no device work).
 * relu != 0 fuses the sign-bit ReLU: outputs are UNSIGNED words of width w-1.
 * Multi-GPU: a context with world > 1 computes only its rank's contiguous
 * share of the output words (neurons [r*ceil(M/W), ...)); the caller
 * all-gathers `out` across ranks. */
typedef struct {
  uint64_t gates, br_lanes, levels, max_level_width, min_level_width, tiles;
} she_circuit_stats;

/* conv (no bias): in [H][W][C][w_in][stride], wq [Co][K][K][C],
 * out [Ho][Wo][Co][*w_out][stride], Ho = (H + 2 pad - K)/stride + 1 ("same"
 * zero padding when pad > 0, R14/R15). */
she_status she_conv_shift_acc(she_ctx* ctx, const uint32_t* in, int H, int W, int C, int w_in,
                              int in_signed, const int8_t* wq, int Co, int K, int stride, int pad,
                              int acc_cap, int relu, uint32_t* out, int* w_out, void* stream);
/* fully connected: in [K][w_in][stride] (HWC-flattened, R16), wq [M][K],
 * out [M][*w_out][stride]. */
she_status she_fc_shift_acc(she_ctx* ctx, const uint32_t* in, int K, int w_in, int in_signed,
                            const int8_t* wq, int M, int acc_cap, int relu, uint32_t* out,
                            int* w_out, void* stream);
/* TCN baseline (SURVEY.md §8(f) NEXT-1; PAPER.md:115, :254 the TFHE version
 * of FCN with plaintext x ciphertext multiplications): the same layers with
 * fixed-point multipliers wm (int16, c in [-255, 255], value c / 2^7) in place
 * of log-quantised codes.  A product is the shift-and-add over the set bits of
 * |c|: sign(c) * sum_{b : bit b of |c|} (x >> (7 - b)), one
 * adder-tree term per set bit, so a single-bit c = 2^(7-e) is SHE's code e+1.
 * Layouts, widths, sharding and errors as she_conv_shift_acc / she_fc_shift_acc. */
she_status she_conv_mul_acc(she_ctx* ctx, const uint32_t* in, int H, int W, int C, int w_in,
                            int in_signed, const int16_t* wm, int Co, int K, int stride, int pad,
                            int acc_cap, int relu, uint32_t* out, int* w_out, void* stream);
she_status she_fc_mul_acc(she_ctx* ctx, const uint32_t* in, int K, int w_in, int in_signed,
                          const int16_t* wm, int M, int acc_cap, int relu, uint32_t* out,
                          int* w_out, void* stream);
/* ReLU on `words` signed words of `width` bits: R_i = AND(X_i, NOT sign)
 * (SPEC.md:193-201 reading of PAPER.md F2); out: words x (width-1) unsigned. */
she_status she_relu(she_ctx* ctx, const uint32_t* in, size_t words, int width, uint32_t* out,
                    void* stream);
/* Batch normalisation lowered to shift + constant (the
 * B layers of PAPER.md T3 :202-203): on `words` words of w_in bits laid out
 * HWC (channel = word index mod C),
 *   y = wrap_acc_cap(sign_c * scale(x, shift_c) + bias_c)
 * with scale(x, s) = x 2^s for s >= 0, floor(x / 2^-s) for s < 0 (shift in
 * [-8, 8], host int8[C]), sign_c = -1 where neg[c] != 0 (host uint8[C], NULL =
 * all +1), bias host int32[C] in [-2^20, 2^20].  The scale is rewiring, the
 * sign NOT flags + a carry-in, the bias an adder against constant bits.  relu
 * != 0 fuses the ReLU (unsigned outputs of width w-1).  *w_out as in the conv
 * call; words % C == 0. */
she_status she_bn_shift_add(she_ctx* ctx, const uint32_t* in, size_t words, int C, int w_in,
                            int in_signed, const int8_t* shift, const uint8_t* neg,
                            const int32_t* bias, int acc_cap, int relu, uint32_t* out,
                            int* w_out, void* stream);
/* 2x2 stride-2 max-pool on [H][W][C][w][stride]: max = subtract-comparator
 * sign driving per-bit MUXes (PAPER.md F2); out [H/2][W/2][C][w][stride],
 * same signedness as the input. */
she_status she_maxpool2x2(she_ctx* ctx, const uint32_t* in, int H, int W, int C, int w,
                          int in_signed, uint32_t* out, void* stream);
/* Gate / lane / level counters of the context's last layer call. */
she_status she_ctx_layer_stats(she_ctx* ctx, she_circuit_stats* stats);

/* Gate capture, for the seed-sampled ciphertext parity of the layer calls
 * ("the oracle recomputes sampled gates from the exact input
 * ciphertexts captured from the GPU's wire table").  While enabled (every > 0)
 * each bootstrapped layer gate whose ordinal o (counted over every level of
 * every layer call since this call) satisfies mix64(seed + o) % every == 0 is
 * recorded, up to max_gates: its op, its three input slots exactly as the gate
 * reads them (negation flags applied to the n+1 live words) and its output
 * slot.  every == 0 disables capture and frees the buffer.  Capture makes the
 * layer calls synchronous.  Test instrumentation, not part of the hot path. */
she_status she_ctx_capture(she_ctx* ctx, uint64_t seed, uint32_t every, size_t max_gates);
/* Copy the captured gates out (HOST buffers): ops[cap], slots[cap][4][stride]
 * (a, b, c, out); *count = number recorded (<= cap copied). */
she_status she_ctx_capture_read(she_ctx* ctx, uint8_t* ops, uint32_t* slots, size_t cap,
                                size_t* count);

/* Clear-bit backend: the same circuits evaluated on plaintext bits (uint8 per
 * bit, layouts as above without the stride axis), host only.  For testing the
 * scheduler and counting gates; stats may be NULL.  rank/world select the
 * same output shard a context with that rank/world computes (only those
 * output words are written). */
she_status she_clear_conv_shift_acc(const uint8_t* in, int H, int W, int C, int w_in,
                                    int in_signed, const int8_t* wq, int Co, int K, int stride,
                                    int pad, int acc_cap, int relu, uint8_t* out, int* w_out,
                                    int rank, int world, she_circuit_stats* stats);
she_status she_clear_fc_shift_acc(const uint8_t* in, int K, int w_in, int in_signed,
                                  const int8_t* wq, int M, int acc_cap, int relu, uint8_t* out,
                                  int* w_out, int rank, int world, she_circuit_stats* stats);
she_status she_clear_conv_mul_acc(const uint8_t* in, int H, int W, int C, int w_in,
                                  int in_signed, const int16_t* wm, int Co, int K, int stride,
                                  int pad, int acc_cap, int relu, uint8_t* out, int* w_out,
                                  int rank, int world, she_circuit_stats* stats);
she_status she_clear_fc_mul_acc(const uint8_t* in, int K, int w_in, int in_signed,
                                const int16_t* wm, int M, int acc_cap, int relu, uint8_t* out,
                                int* w_out, int rank, int world, she_circuit_stats* stats);
she_status she_clear_relu(const uint8_t* in, size_t words, int width, uint8_t* out, int rank,
                          int world, she_circuit_stats* stats);
she_status she_clear_bn_shift_add(const uint8_t* in, size_t words, int C, int w_in,
                                  int in_signed, const int8_t* shift, const uint8_t* neg,
                                  const int32_t* bias, int acc_cap, int relu, uint8_t* out,
                                  int* w_out, int rank, int world, she_circuit_stats* stats);
she_status she_clear_maxpool2x2(const uint8_t* in, int H, int W, int C, int w, int in_signed,
                                uint8_t* out, int rank, int world, she_circuit_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* SHE_H_ */
