// engine.h — internal interface between the host scheduler and the device engine.
#pragma once
#include <stdint.h>

#include <vector>

#include "../../include/she.h"
#include "scheduler.h"

namespace she {

// Run a compiled circuit tile on the GPU: gather its inputs (layer-input slots
// input_bits[k] of `in`) into the wire table, launch one gate level at a time
// (K2-K4 per level), then gather the requested outputs into
// out[out_first + o] (slots, negation applied).  Stream-ordered.
she_status engine_run_program(she_ctx* ctx, const sched::Program& p, const uint32_t* in,
                              const std::vector<uint32_t>& input_bits, uint32_t* out,
                              size_t out_first, void* stream);
// Circuit counters of the last layer call (reset = start a new call).
she_circuit_stats* engine_stats(she_ctx* ctx, bool reset);
int engine_rank(const she_ctx* ctx);
int engine_world(const she_ctx* ctx);

}  // namespace she
