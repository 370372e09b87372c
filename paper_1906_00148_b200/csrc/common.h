// common.h — shared host-side plumbing of libshe: status/errors, params checks.
#pragma once
#include <stdarg.h>
#include <stdio.h>

#include <string>

#include "../../include/she.h"

namespace she {

void set_error(const char* fmt, ...);

inline she_status fail(she_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error("%s", buf);
  return s;
}

inline size_t lwe_stride(const she_params& p) { return (p.n + 1 + 31) / 32 * 32; }

// Parameter sets this build supports (include/she.h she_params).
inline she_status check_params(const she_params* p) {
  if (!p) return fail(SHE_ERR_ARG, "params is NULL");
  if (p->k != 1) return fail(SHE_ERR_PARAMS, "k=%u unsupported (k=1 only)", p->k);
  if (p->N != 256 && p->N != 1024) return fail(SHE_ERR_PARAMS, "N=%u unsupported", p->N);
  // an LWE slot (n + 1 words padded to 32) must fit the key-switch kernels'
  // 512 threads / 2 x 256 words per gate: n <= 511
  if (p->n == 0 || p->n > 511) return fail(SHE_ERR_PARAMS, "n=%u unsupported (1..511)", p->n);
  if (p->l != 2) return fail(SHE_ERR_PARAMS, "l=%u unsupported (l=2: 4 rows = 4 warps)", p->l);
  if (p->bg_bits == 0 || p->l * p->bg_bits >= 32)
    return fail(SHE_ERR_PARAMS, "l*bg_bits=%u must be < 32", p->l * p->bg_bits);
  if (p->ks_base_bits != 2 || p->ks_t == 0 || p->ks_t * p->ks_base_bits >= 32)
    return fail(SHE_ERR_PARAMS, "key switching base 2^%u x %u unsupported", p->ks_base_bits,
                p->ks_t);
  // exactness of the Goldilocks NTT product: (k+1) l N (Bg/2) 2^31 < (p-1)/2 ~ 2^63
  double bound = 2.0 * p->l * p->N * (double)(1u << (p->bg_bits - 1)) * 2147483648.0;
  if (bound >= 9.2e18) return fail(SHE_ERR_PARAMS, "NTT exactness bound violated");
  return SHE_OK;
}

}  // namespace she
