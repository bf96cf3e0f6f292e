// Internal accessors of the readiness negotiator (hvd_negotiate.cpp) for the runtime.
#pragma once
#include <cstdint>

struct hvd_negotiator;

namespace hvd_neg {
// i-th id agreed by the last cycle, with the count / dtype every rank reported for it
bool agreed_meta(const hvd_negotiator* g, uint32_t i, uint32_t* id, uint64_t* count, int* dtype);
int size_of(const hvd_negotiator* g);
int nlocal_of(const hvd_negotiator* g);
uint32_t max_of(const hvd_negotiator* g);
// The newest min(m, available) negotiation records of local rank `local`, oldest first:
// out[3i..3i+2] = {id, ns reported ready, ns agreed} (CLOCK_REALTIME).  Records stay
// for hvd_negotiator_trace.  Returns the number copied.
uint32_t trace_recent(const hvd_negotiator* g, int local, uint32_t m, uint64_t* out);
}  // namespace hvd_neg
