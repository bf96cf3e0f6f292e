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
}  // namespace hvd_neg
