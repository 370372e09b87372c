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

// Lanes base .. base + nsl - 1 (nsl = 0: no more work), iterations [i0, i1);
// slot = where the unit's accumulators wait between chunks (acc_save, progress
// word): the pair index (pair queue) or the lane index (single-lane queue).
struct Unit {
  uint32_t base, nsl, i0, i1, slot;
};

// How a batch of `total` lanes is spread over `pipelines` two-lane pipelines.
//  kStatic   the contiguous split, every lane for all n iterations: up to one
//            lane per pipeline (a lane alone runs on all four warps of its
//            pipeline, the shortest latency), or chunk >= n;
//  kSingles  a queue of (lane, chunk) units, each lane alone on a pipeline:
//            batches a little wider than the pipelines.  A pair takes ~1.75x
//            as long as a single lane, so up to ~1.65 lanes per pipeline the
//            single-lane chunks, spread evenly, finish before one pair would;
//  kPairs    a queue of (lane pair, chunk) units (+ an odd lane, whole): the
//            highest throughput per pipeline, for everything wider.
enum Mode { kStatic = 0, kPairs = 1, kSingles = 2 };
TMQ_HD int mode(uint32_t total, uint32_t n, uint32_t chunk, uint32_t pipelines) {
  if (chunk >= n || total <= pipelines) return kStatic;
  if ((uint64_t)total * 100 <= (uint64_t)pipelines * 165) return kSingles;
  return total > 2 * pipelines ? kPairs : kStatic;
}

TMQ_HD uint32_t units(uint32_t total, uint32_t n, uint32_t chunk, int m) {
  const uint32_t nchunks = (n + chunk - 1) / chunk;
  return m == kSingles ? total * nchunks : (total >> 1) * nchunks + (total & 1);
}

// Unit u of the queue, chunk-major: chunk 0 of every pair (lane), then chunk 1
// of every pair (lane), ...  Chunk k depends on chunk k - 1 of the same slot,
// which is a smaller unit number.  Pair queue: an odd last lane is unit 0 and
// runs all n iterations (the longest unit first).
TMQ_HD Unit unit(uint32_t u, uint32_t total, uint32_t n, uint32_t chunk, int m) {
  if (u >= units(total, n, chunk, m)) return {0, 0, 0, n, 0};
  const uint32_t odd = m == kPairs ? (total & 1) : 0;
  if (odd && u == 0) return {total - 1, 1, 0, n, 0};
  u -= odd;
  const uint32_t per = m == kSingles ? total : total >> 1;  // slots
  const uint32_t k = u / per, slot = u - k * per, i0 = k * chunk;
  const uint32_t i1 = n < i0 + chunk ? n : i0 + chunk;
  return m == kSingles ? Unit{slot, 1, i0, i1, slot} : Unit{2 * slot, 2, i0, i1, slot};
}
// ---- the wrap-around schedule (the default for kPairs / kSingles) -----------
// McNaughton's rule for identical machines with preemption: lay the units'
// n iterations end to end (unit p = lane pair p, or lane p; an odd last lane
// is a unit of one lane) and cut the line into `pipelines` equal ranges.
// With at least n iterations per pipeline a unit is cut at most once, into a
// first part [0, x) that ends one pipeline's range and a last part [x, n) that
// starts the next pipeline's range.  A pipeline runs the END of its range
// first (a first part: no dependency), then its whole units, and the START of
// its range last (a last part: it waits for the first part, which its
// neighbour ran first, tens of milliseconds earlier).  Every pipeline gets the
// same number of iterations (+- 1) and there is one hand-over per pipeline,
// instead of one per (unit, chunk) as in the queue.
TMQ_HD uint32_t wrap_units(uint32_t total, int m) { return m == kSingles ? total : (total + 1) >> 1; }
TMQ_HD Unit wrap_make(uint32_t p, uint32_t i0, uint32_t i1, uint32_t total, int m) {
  if (m == kSingles) return {p, 1, i0, i1, p};
  return {2 * p, 2 * p + 1 < total ? 2u : 1u, i0, i1, p};
}
// The step-th unit, in execution order, of pipeline gq (nsl = 0: done).
TMQ_HD Unit wrap_unit(uint32_t gq, uint32_t step, uint32_t total, uint32_t n, uint32_t nq, int m) {
  const uint64_t W = (uint64_t)wrap_units(total, m) * n;
  const uint64_t s0 = W * gq / nq, s1 = W * (gq + 1) / nq;
  if (s1 <= s0) return {0, 0, 0, n, 0};
  const uint32_t a = (uint32_t)(s0 / n), b = (uint32_t)((s1 - 1) / n);
  const uint32_t a0 = (uint32_t)(s0 - (uint64_t)a * n);  // unit a from iteration a0
  const uint32_t b1 = (uint32_t)(s1 - (uint64_t)b * n);  // unit b up to iteration b1 (1 .. n)
  const bool first_part = b > a && b1 < n, last_part = a0 > 0;
  uint32_t k = step;
  if (first_part) {
    if (k == 0) return wrap_make(b, 0, b1, total, m);
    --k;
  }
  const uint32_t lo = a + (last_part ? 1 : 0), hi = first_part ? b : b + 1;  // units [lo, hi) from their start
  if (lo < hi) {
    if (k < hi - lo) return wrap_make(lo + k, 0, lo + k == b ? b1 : n, total, m);
    k -= hi - lo;
  }
  if (last_part && k == 0) return wrap_make(a, a0, a == b ? b1 : n, total, m);
  return {0, 0, 0, n, 0};
}

// Save slots a batch of up to max_lanes lanes can need on `pipelines` pipelines.
TMQ_HD uint32_t slots(uint32_t max_lanes, uint32_t pipelines) {
  const uint32_t singles = max_lanes < 2 * pipelines ? max_lanes : 2 * pipelines;
  const uint32_t pairs = (max_lanes + 1) >> 1;
  return pairs > singles ? pairs : singles;
}

// Static split: pipeline gq of nq runs the contiguous lanes [first(gq),
// first(gq + 1)) as pairs, an odd last lane alone, each for all n iterations.
TMQ_HD uint32_t first(uint32_t gq, uint32_t total, uint32_t nq) {
  return (uint32_t)(((uint64_t)gq * total) / nq);
}
TMQ_HD Unit next_static(uint32_t cursor, uint32_t gq, uint32_t total, uint32_t nq, uint32_t n) {
  const uint32_t last = first(gq + 1, total, nq);
  const uint32_t left = cursor < last ? last - cursor : 0;
  return {cursor, left < 2 ? left : 2, 0, n, 0};
}

}  // namespace tmq
