// Tensor Fusion plan (host): PAPER.md §7 step 1 "Select the first
// few tensors that fit in the buffer and have the same data type", step 6
// "Repeat until there are no more tensors to reduce in the cycle".
//
// Readings: R6 "fits" is inclusive (padded bytes + bytes <= limit);
// R7 a tensor larger than the limit is split into limit-sized segments, each a
// buffer of its own; R8 threshold 0 turns fusion off; members start on 16 B.
// Also hosts the chunk partition (R2).
#include <cstdint>
#include <vector>

#include "../../include/hvd.h"
#include "hvd_internal.h"
#include "hvd_plan.h"

namespace hvd {

static uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

int build_plan(const uint64_t* counts, const int32_t* dtypes, int n, uint64_t threshold,
               uint64_t capacity, std::vector<hvd_plan_entry>* entries,
               std::vector<hvd_plan_buffer>* buffers) {
  entries->clear();
  buffers->clear();
  if (n < 0 || capacity == 0) return HVD_ERR_INVALID;
  const uint64_t limit = threshold == 0 ? capacity : (threshold < capacity ? threshold : capacity);
  bool open = false;
  uint64_t open_bytes = 0;  // end of the last member, bytes
  int open_dtype = 0;
  auto close = [&]() {
    if (open) {
      hvd_plan_buffer& b = buffers->back();
      b.length = open_bytes / elem_size(open_dtype);
      open = false;
    }
  };
  auto start = [&](int dtype) {
    hvd_plan_buffer b = {};
    b.dtype = dtype;
    b.first_entry = (int32_t)entries->size();
    buffers->push_back(b);
  };
  for (int k = 0; k < n; ++k) {
    const int esz = elem_size(dtypes[k]);
    if (esz == 0) return HVD_ERR_UNSUPPORTED;
    const uint64_t count = counts[k];
    if (count == 0) continue;
    if (count > UINT64_MAX / (uint64_t)esz) return HVD_ERR_INVALID;
    const uint64_t nbytes = count * esz;
    if (nbytes > limit) {  // R7: oversize -> singleton segments
      close();
      const uint64_t seg = limit / esz;
      if (seg == 0) return HVD_ERR_INVALID;
      for (uint64_t s0 = 0; s0 < count; s0 += seg) {
        const uint64_t c = count - s0 < seg ? count - s0 : seg;
        start(dtypes[k]);
        entries->push_back({k, (int32_t)buffers->size() - 1, s0, 0, c});
        buffers->back().n_entries = 1;
        buffers->back().length = c;
      }
      continue;
    }
    if (threshold == 0) {  // R8: fusion off
      close();
      start(dtypes[k]);
      entries->push_back({k, (int32_t)buffers->size() - 1, 0, 0, count});
      buffers->back().n_entries = 1;
      buffers->back().length = count;
      continue;
    }
    if (open && open_dtype == dtypes[k]) {
      const uint64_t off = align_up(open_bytes, kMemberAlign);
      if (off + nbytes <= limit) {  // R6: inclusive
        entries->push_back({k, (int32_t)buffers->size() - 1, 0, off / esz, count});
        buffers->back().n_entries += 1;
        open_bytes = off + nbytes;
        continue;
      }
    }
    close();
    start(dtypes[k]);
    entries->push_back({k, (int32_t)buffers->size() - 1, 0, 0, count});
    buffers->back().n_entries = 1;
    open = true;
    open_bytes = nbytes;
    open_dtype = dtypes[k];
  }
  close();
  return HVD_OK;
}

// R2: q = ceil(L / (N * g)) * g elements, g = 256 B; chunk c = [min(cq, L), min((c+1)q, L)).
uint64_t chunk_len(uint64_t length, int size, int dtype) {
  const uint64_t g = kChunkQuantum / elem_size(dtype);
  const uint64_t per = (uint64_t)size * g;
  return (length + per - 1) / per * g;
}

}  // namespace hvd

extern "C" int hvd_plan(const uint64_t* counts, const int32_t* dtypes, int n, uint64_t fusion_threshold,
                        uint64_t capacity, hvd_plan_entry* entries, int* n_entries, hvd_plan_buffer* buffers,
                        int* n_buffers) {
  if (n < 0 || (n > 0 && (!counts || !dtypes)) || !n_entries || !n_buffers) return HVD_ERR_INVALID;
  std::vector<hvd_plan_entry> e;
  std::vector<hvd_plan_buffer> b;
  const int st = hvd::build_plan(counts, dtypes, n, fusion_threshold, capacity, &e, &b);
  if (st != HVD_OK) return st;
  const int cap_e = *n_entries, cap_b = *n_buffers;
  *n_entries = (int)e.size();
  *n_buffers = (int)b.size();
  if ((int)e.size() > cap_e || (int)b.size() > cap_b) return HVD_ERR_INVALID;
  for (size_t i = 0; i < e.size(); ++i) entries[i] = e[i];
  for (size_t i = 0; i < b.size(); ++i) buffers[i] = b[i];
  return HVD_OK;
}

extern "C" int hvd_chunk_bounds(uint64_t length, int size, int dtype, uint64_t* out) {
  if (size < 1 || !out || hvd::elem_size(dtype) == 0) return size < 1 || !out ? HVD_ERR_INVALID : HVD_ERR_UNSUPPORTED;
  const uint64_t q = hvd::chunk_len(length, size, dtype);
  for (int c = 0; c < size; ++c) out[c] = (uint64_t)c * q < length ? (uint64_t)c * q : length;
  out[size] = length;
  return HVD_OK;
}
