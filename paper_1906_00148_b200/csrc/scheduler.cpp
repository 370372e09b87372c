// scheduler.cpp — layer calls (placeholder until the circuit scheduler lands).
#include "common.h"

extern "C" {
she_status she_conv_shift_acc(she_ctx*, const uint32_t*, int, int, int, int, const int8_t*, int,
                              int, int, int, int, int, uint32_t*, int*, void*) {
  return she::fail(SHE_ERR_STATE, "she_conv_shift_acc: not implemented yet");
}
she_status she_fc_shift_acc(she_ctx*, const uint32_t*, int, int, const int8_t*, int, int, int,
                            uint32_t*, int*, void*) {
  return she::fail(SHE_ERR_STATE, "she_fc_shift_acc: not implemented yet");
}
she_status she_relu(she_ctx*, const uint32_t*, size_t, int, uint32_t*, void*) {
  return she::fail(SHE_ERR_STATE, "she_relu: not implemented yet");
}
she_status she_maxpool2x2(she_ctx*, const uint32_t*, int, int, int, int, uint32_t*, void*) {
  return she::fail(SHE_ERR_STATE, "she_maxpool2x2: not implemented yet");
}
}
