// tm_queue.h — unit numbering of the TMEM engine's work distribution
// (br_tmem.cuh): which lanes and which CMux iterations a
// pipeline runs next.  Plain integer functions, shared by the kernel and the
// host emulation library (tests/test_tm_queue.py checks on the CPU that every
// (lane, iteration) is run exactly once and in dependency order).
#pragma once
#include <stdint.h>
#ifdef __CUDACC__
#define TMQ_HD __host__ __device__ __forceinline__
#else
#define TMQ_HD inline
#endif

namespace tmq {

// Lanes base .. base + nsl - 1 (nsl = 0: no more work), iterations [i0, i1).
struct Unit {
  uint32_t base, nsl, i0, i1;
};

// The queue serves batches of more than two lanes per pipeline; chunk >= n
// (or fewer lanes) means the static contiguous split.
TMQ_HD bool queued(uint32_t total, uint32_t n, uint32_t chunk, uint32_t pipelines) {
  return chunk < n && total > 2 * pipelines;
}

// total / 2 lane pairs x ceil(n / chunk) chunks, + an odd last lane (whole).
TMQ_HD uint32_t units(uint32_t total, uint32_t n, uint32_t chunk) {
  return (total >> 1) * ((n + chunk - 1) / chunk) + (total & 1);
}

// Unit u of the queue, chunk-major: an odd lane is unit 0 and runs all n
// iterations (the longest unit first); then chunk 0 of every pair, chunk 1 of
// every pair, ...  Chunk k of a pair depends on its chunk k - 1, which is a
// smaller unit number.
TMQ_HD Unit unit(uint32_t u, uint32_t total, uint32_t n, uint32_t chunk) {
  const uint32_t npairs = total >> 1, odd = total & 1;
  if (u >= units(total, n, chunk)) return {0, 0, 0, n};
  if (odd && u == 0) return {total - 1, 1, 0, n};
  u -= odd;
  const uint32_t k = u / npairs, pair = u - k * npairs, i0 = k * chunk;
  return {2 * pair, 2, i0, n < i0 + chunk ? n : i0 + chunk};
}

// Static split: pipeline gq of nq runs the contiguous lanes [first(gq),
// first(gq + 1)) as pairs, an odd last lane alone, each for all n iterations.
TMQ_HD uint32_t first(uint32_t gq, uint32_t total, uint32_t nq) {
  return (uint32_t)(((uint64_t)gq * total) / nq);
}
TMQ_HD Unit next_static(uint32_t cursor, uint32_t gq, uint32_t total, uint32_t nq, uint32_t n) {
  const uint32_t last = first(gq + 1, total, nq);
  const uint32_t left = cursor < last ? last - cursor : 0;
  return {cursor, left < 2 ? left : 2, 0, n};
}

}  // namespace tmq
