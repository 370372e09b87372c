// ks_imma.cuh — K4 on the tensor cores: the key switch N -> n of a batch of
// gates as an exact 8-bit integer matrix product (
// PAPER.md:188 "key-switching").
//
// For base 4 and t = 8 (every config) the key switch of gate g is
//   out_g = (0, b'_g) - sum_{i<N, j<t} KSK[i][j][d_gij],   d = 2 b1 + b0
// and KSK[i][j][d] = b0 K1 + b1 K2 + b0 b1 K3'   (K3' = K3 - K1 - K2 mod 2^32)
// (the ks2 identity).  With the 0/1 matrix
//   A[g][(i, j, v)] = (b0, b1, b0 b1)[v]                 (gates x 24 N)
// and the key's four byte planes
//   B_p[(i, j, v)][w] = byte p of (K1, K2, K3')[v][i][j][w]
// the sum is  sum_p 2^(8p) (A B_p)[g][w]  mod 2^32, each A B_p an exact
// integer product (<= 24 N * 255 < 2^31).  Three kernels:
//   ksi_prep    extracted samples (+ MUX combine, rounding R10) -> A (u8), b'
//   ksi_gemm    C = A B with mma.sync m16n8k32 u8 x u8 -> s32 (IMMA), B's
//               columns ordered (word, plane); cp.async 3-stage pipeline,
//               XOR-swizzled shared tiles (conflict-free fragment loads)
//   ksi_combine out = (0, b') - sum_p C_p << 8p; NOT / COPY gates copy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ksi {

constexpr int BM = 128, BN = 128, BK = 128;  // CTA tile (gates, columns, k bytes)
constexpr int kStages = 3;
constexpr int kThreads = 256;                // 8 warps: 2 (M) x 4 (N), warp tile 64 x 32
constexpr size_t kStageBytes = (size_t)(BM + BN) * BK;
constexpr size_t kSmem = kStages * kStageBytes;  // 96 KB

// 16-byte chunk c of tile row r lives at chunk c ^ (r & 7) (8 chunks per row)
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * BK + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void mma_u8(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// C[M][Ncols] (s32) = A[M][K] (u8, row-major) x Bt[Ncols][K] (u8, K contiguous).
// M % BM == 0, Ncols % BN == 0, K % BK == 0 (the caller pads).
__global__ void __launch_bounds__(kThreads, 2) ksi_gemm(const uint8_t* A, const uint8_t* Bt,
                                                        int32_t* C, int K, int ncols) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile origin: (64 wm, 32 wn)
  const int g = lane >> 2, t = lane & 3;
  const size_t m0 = (size_t)blockIdx.y * BM, n0 = (size_t)blockIdx.x * BN;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  const int ktiles = K / BK;

  auto load_stage = [&](int s, int kt) {
    const uint32_t sa = sbase + (uint32_t)(s * kStageBytes), sb = sa + BM * BK;
    const size_t k0 = (size_t)kt * BK;
#pragma unroll
    for (int q = 0; q < (BM * BK / 16) / kThreads; ++q) {  // 4 chunks of A, 4 of B per thread
      const int idx = tid + q * kThreads, r = idx >> 3, c = idx & 7;
      cp_async16(sa + swz(r, c), A + (m0 + r) * (size_t)K + k0 + c * 16);
      cp_async16(sb + swz(r, c), Bt + (n0 + r) * (size_t)K + k0 + c * 16);
    }
  };

  int acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<kStages - 2>();
    __syncthreads();
    {  // refill the stage consumed last iteration
      const int nk = kt + kStages - 1;
      if (nk < ktiles) load_stage(nk % kStages, nk);
      cp_commit();
    }
    const uint8_t* sa = sm + (size_t)(kt % kStages) * kStageBytes;
    const uint8_t* sb = sa + BM * BK;
#pragma unroll
    for (int kk = 0; kk < BK / 32; ++kk) {
      uint32_t af[4][4], bf[4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r0 = wm * 64 + mi * 16 + g, r1 = r0 + 8;
        af[mi][0] = *reinterpret_cast<const uint32_t*>(sa + swz(r0, 2 * kk) + 4 * t);
        af[mi][1] = *reinterpret_cast<const uint32_t*>(sa + swz(r1, 2 * kk) + 4 * t);
        af[mi][2] = *reinterpret_cast<const uint32_t*>(sa + swz(r0, 2 * kk + 1) + 4 * t);
        af[mi][3] = *reinterpret_cast<const uint32_t*>(sa + swz(r1, 2 * kk + 1) + 4 * t);
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int c0 = wn * 32 + ni * 8 + g;
        bf[ni][0] = *reinterpret_cast<const uint32_t*>(sb + swz(c0, 2 * kk) + 4 * t);
        bf[ni][1] = *reinterpret_cast<const uint32_t*>(sb + swz(c0, 2 * kk + 1) + 4 * t);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) mma_u8(acc[mi][ni], af[mi], bf[ni]);
    }
  }
  cp_wait<0>();
  // epilogue: C fragment (row g / g + 8, columns 2t, 2t + 1)
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const size_t r = m0 + wm * 64 + mi * 16 + g, c = n0 + wn * 32 + ni * 8 + 2 * t;
      *reinterpret_cast<int2*>(C + r * ncols + c) = make_int2(acc[mi][ni][0], acc[mi][ni][1]);
      *reinterpret_cast<int2*>(C + (r + 8) * ncols + c) = make_int2(acc[mi][ni][2], acc[mi][ni][3]);
    }
}

}  // namespace ksi

// ---------------------------------------------------------------------------
// The same product on the 5th-generation tensor cores (tcgen05, kind::i8):
// the shared tiles above are already the canonical K-major SWIZZLE_128B layout
// (rows of 128 bytes, 16-byte chunk c of row r at chunk c ^ (r & 7), tiles
// 1024-byte aligned), so the cp.async pipeline feeds tcgen05.mma directly.
// One elected thread issues 4 MMAs (M = 128, N = 128, K = 32) per stage into a
// 128 x 128 s32 accumulator in TMEM and commits them to the stage's mbarrier;
// a stage is refilled once its MMAs have drained.  Epilogue: tcgen05.ld of the
// accumulator (warp w reads TMEM lanes 32 (w & 3) .. + 31, columns 64 (w >> 2)
// .. + 63) -> global.
// ---------------------------------------------------------------------------
namespace ksi {

constexpr size_t kSmemTc = kSmem + 1024;  // + alignment of the tiles to 1024 B

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  // start >> 4 | LBO 1 (unused for swizzled K-major) | SBO 1024 B | version 1 | SWIZZLE_128B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// kind::i8 instruction descriptor: D = s32 (c_format 2), A = B = u8, both
// K-major, N = 128 (n_dim = N >> 3), M = 128 (m_dim = M >> 4).
constexpr uint32_t kIdescU8 = (2u << 4) | (0u << 7) | (0u << 10) | ((128u >> 3) << 17) |
                              ((128u >> 4) << 24);

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0; !done; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (spin > (1u << 26)) __trap();  // a lost commit must fail, not hang the device
  }
}

__global__ void __launch_bounds__(kThreads, 1) ksi_gemm_tc(const uint8_t* A, const uint8_t* Bt,
                                                           int32_t* C, int K, int ncols) {
  extern __shared__ __align__(128) uint8_t sm_raw[];
  __shared__ __align__(8) uint64_t mbar[kStages];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const size_t m0 = (size_t)blockIdx.y * BM, n0 = (size_t)blockIdx.x * BN;
  const uint32_t raw = (uint32_t)__cvta_generic_to_shared(sm_raw);
  const uint32_t sbase = (raw + 1023u) & ~1023u;
  const int ktiles = K / BK;
  const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);

  if (warp == 0) {
    const uint32_t slot = (uint32_t)__cvta_generic_to_shared(&tmem_slot);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(slot)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(mb0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  auto load_stage = [&](int s, int kt) {
    const uint32_t sa = sbase + (uint32_t)(s * kStageBytes), sb = sa + BM * BK;
    const size_t k0 = (size_t)kt * BK;
#pragma unroll
    for (int q = 0; q < (BM * BK / 16) / kThreads; ++q) {
      const int idx = tid + q * kThreads, r = idx >> 3, c = idx & 7;
      cp_async16(sa + swz(r, c), A + (m0 + r) * (size_t)K + k0 + c * 16);
      cp_async16(sb + swz(r, c), Bt + (n0 + r) * (size_t)K + k0 + c * 16);
    }
  };
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_wait<kStages - 2>();
    // the cp.async writes (generic proxy) must be visible to the tensor
    // core's reads (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int s = kt % kStages;
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sa = sbase + (uint32_t)(s * kStageBytes), sb = sa + BM * BK;
#pragma unroll
      for (int kk = 0; kk < BK / 32; ++kk) {
        const uint64_t ad = umma_desc_sw128(sa + 32 * kk), bd = umma_desc_sw128(sb + 32 * kk);
        const uint32_t acc = (kt | kk) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(kIdescU8), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       mb0 + 8 * s)
                   : "memory");
    }
    const int nk = kt + kStages - 1;
    if (nk < ktiles) {
      if (kt >= 1)  // the stage to refill was read by the MMAs of iteration kt - 1
        mbar_wait(mb0 + 8 * ((kt - 1) % kStages), (uint32_t)(((kt - 1) / kStages) & 1));
      load_stage(nk % kStages, nk);
    }
    cp_commit();
  }
  cp_wait<0>();
  {  // all MMAs done: the last commit
    const int last = ktiles - 1;
    mbar_wait(mb0 + 8 * (last % kStages), (uint32_t)((last / kStages) & 1));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int q = warp & 3, half = warp >> 2;
  const size_t row = m0 + 32 * q + lane;
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    const uint32_t col = 64 * half + 32 * part;
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + ((uint32_t)(32 * q) << 16) + col));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int4* dst = reinterpret_cast<int4*>(C + row * ncols + n0 + col);
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4)
      dst[c4] = make_int4((int)v[4 * c4], (int)v[4 * c4 + 1], (int)v[4 * c4 + 2], (int)v[4 * c4 + 3]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

}  // namespace ksi
