// TMEM as a per-thread-row scratch store: tcgen05.st / tcgen05.ld
// (32x32b shapes) throughput per SM with 16 warps, alone and beside 16-byte
// shared-memory loads (does TMEM traffic use the L1/shared-memory data path?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tmem_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void tst16(uint32_t addr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr)
      : "memory");
}

// MODE 0: st only, 1: ld only, 2: LDS.128 only, 3: ld + LDS.128 (same bytes each)
template <int MODE>
__global__ void __launch_bounds__(512, 1) tmem_kernel(uint32_t* out, int iters) {
  __shared__ uint32_t tslot;
  __shared__ __align__(16) uint4 sm[512 * 4];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int i = tid; i < 512 * 4; i += 512) sm[i] = make_uint4(i, i + 1, i + 2, i + 3);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // warp w: TMEM lanes 32 (w % 4) .. +31, its own 128-column band (w / 4)
  const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * (warp >> 2);
  uint32_t v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = tid * 16 + k;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // 8 x 16 columns = 128 columns (512 B per thread)
      if (MODE == 0) {
        tst16(base + 16 * c, v);
        v[c] += 1;
      } else if (MODE == 1 || MODE == 3) {
        tld16(base + 16 * c, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += v[c] ^ v[15 - c];
      }
      if (MODE == 2 || MODE == 3) {
        const int o = tid + it + c * 64;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 x = sm[(o + q * 512) & 2047];
          acc += x.x ^ x.w;
        }
      }
    }
    if (MODE == 0) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  uint32_t s = acc;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += v[k];
  out[blockIdx.x * 512 + tid] = s;
}

template <int MODE>
void run(const char* name, int sms, int clk, uint32_t* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  tmem_kernel<MODE><<<sms, 512>>>(d, 8);
  cudaEventRecord(e0);
  tmem_kernel<MODE><<<sms, 512>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cyc = ms * 1e-3 * clk * 1e3;
  const double tbytes = (MODE == 0 || MODE == 1 || MODE == 3) ? 512.0 * iters * 8 * 64 : 0;
  const double sbytes = (MODE >= 2) ? 512.0 * iters * 8 * 64 : 0;
  printf("%-22s %8.3f ms  TMEM %7.1f B/clk/SM  SMEM %7.1f B/clk/SM\n", name, ms, tbytes / cyc,
         sbytes / cyc);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* d;
  cudaMalloc(&d, 4 * sms * 512);
  run<0>("tcgen05.st x16", sms, clk, d);
  run<1>("tcgen05.ld x16 + wait", sms, clk, d);
  run<2>("LDS.128", sms, clk, d);
  run<3>("ld x16 + LDS.128", sms, clk, d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
