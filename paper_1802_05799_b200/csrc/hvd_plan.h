#pragma once
#include <cstdint>
#include <vector>

#include "../../include/hvd.h"

namespace hvd {
int build_plan(const uint64_t* counts, const int32_t* dtypes, int n, uint64_t threshold,
               uint64_t capacity, std::vector<hvd_plan_entry>* entries,
               std::vector<hvd_plan_buffer>* buffers);
uint64_t chunk_len(uint64_t length, int size, int dtype);
}  // namespace hvd
