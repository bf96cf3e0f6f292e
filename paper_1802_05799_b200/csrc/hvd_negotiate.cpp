// Readiness negotiation: Tensor Fusion steps 1 and 6 ("Determine which
// tensors are ready to be reduced", "Repeat until there are no more
// tensors to reduce in the cycle"), R15.
//
// Host-only.  Ranks of one node share a POSIX shared-memory segment:
//   [header 64 B][rank 0 parity 0 slot][rank 0 parity 1 slot][rank 1 ...] ...
//   slot = {u64 seq, u64 n, Entry e[max_tensors]}, Entry = {u32 id, i32 dtype, u64 count}
// Cycle k: every process writes its ranks' pending lists into parity k&1, then
// release-stores seq = k; it waits (acquire) until every rank's parity-k&1 seq
// reaches k and intersects the lists itself, so all ranks compute the same
// agreed list without a coordinator round trip.  A rank reuses parity k&1 at
// cycle k+2, which it reaches only after seeing every rank publish cycle k+1 —
// i.e. after every rank has finished reading cycle k.
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <time.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hvd.h"
#include "hvd_negotiate.h"

namespace {

constexpr uint64_t kMagic = 0x4856444e45474f31ull;  // "HVDNEGO1"

struct Header {
  uint64_t magic;  // written last by the creator (release)
  uint32_t size;
  uint32_t max_tensors;
  uint32_t creator_pid;    // rank 0's process: a segment whose creator is gone is stale
  uint32_t pad0;
  uint64_t creator_start;  // its start time (/proc/<pid>/stat field 22): pid reuse
  uint64_t pad[4];
};
static_assert(sizeof(Header) == 64, "header");

struct Entry {
  uint32_t id;
  int32_t dtype;
  uint64_t count;
};

struct SlotHead {
  uint64_t seq;
  uint64_t n;
};

bool valid_dtype(int d) { return d >= 1 && d <= 4; }

// Start time of a process in clock ticks since boot (/proc/<pid>/stat field 22); 0 if
// the process does not exist.
uint64_t proc_start(int pid) {
  char path[64];
  std::snprintf(path, sizeof path, "/proc/%d/stat", pid);
  FILE* f = std::fopen(path, "r");
  if (!f) return 0;
  char buf[1024];
  const size_t n = std::fread(buf, 1, sizeof buf - 1, f);
  std::fclose(f);
  buf[n] = 0;
  const char* p = std::strrchr(buf, ')');  // the command name may contain spaces
  if (!p) return 0;
  int field = 2;
  for (; *p && field < 22; ++p)
    if (*p == ' ') ++field;
  return std::strtoull(p, nullptr, 10);
}

// A segment left by a crashed run has a valid magic but a creator that no longer runs:
// a rank attaching before rank 0 replaced it must not use it.
bool creator_alive(const Header* h) {
  const uint64_t st = proc_start((int)h->creator_pid);
  return st != 0 && st == h->creator_start;
}

uint64_t now_ns() {  // CLOCK_REALTIME: comparable across the processes of one node
  timespec ts;
  clock_gettime(CLOCK_REALTIME, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

constexpr size_t kTraceCap = 8192;  // negotiation records kept per local rank

struct TraceRec {
  uint64_t id, t_ready, t_agreed;
};

}  // namespace

struct hvd_negotiator {
  std::string name;        // shm object ("" = process-private)
  int rank = 0, size = 1, nlocal = 1;
  uint32_t max = 0;
  uint64_t timeout_ms = 0;
  char* base = nullptr;    // mapped segment
  size_t bytes = 0;
  bool owner = false;      // created the shm object (unlinks it)
  bool priv = false;       // malloc'd (virtual communicator)
  uint64_t cycle = 0;
  std::vector<std::vector<Entry>> pending;     // [nlocal], submission order
  std::vector<std::vector<uint8_t>> is_pending;  // [nlocal][max]
  // scratch of the intersection, indexed by id
  std::vector<uint64_t> stamp;
  std::vector<uint32_t> nranks;
  std::vector<Entry> meta;
  std::vector<Entry> agreed;  // last cycle's agreed entries, in order
  std::vector<std::vector<uint64_t>> t_ready;   // [nlocal][max] when each pending id was reported
  std::vector<std::vector<TraceRec>> trace;     // [nlocal] (id, reported, agreed) since the last read

  size_t slot_bytes() const { return sizeof(SlotHead) + (size_t)max * sizeof(Entry); }
  char* slot(int r, int par) const { return base + sizeof(Header) + ((size_t)r * 2 + par) * slot_bytes(); }
};

namespace hvd_neg {
bool agreed_meta(const hvd_negotiator* g, uint32_t i, uint32_t* id, uint64_t* count, int* dtype) {
  if (!g || i >= g->agreed.size()) return false;
  *id = g->agreed[i].id;
  *count = g->agreed[i].count;
  *dtype = g->agreed[i].dtype;
  return true;
}
int size_of(const hvd_negotiator* g) { return g ? g->size : 0; }
int nlocal_of(const hvd_negotiator* g) { return g ? g->nlocal : 0; }
uint32_t max_of(const hvd_negotiator* g) { return g ? g->max : 0; }
uint32_t trace_recent(const hvd_negotiator* g, int local, uint32_t m, uint64_t* out) {
  if (!g || local < 0 || local >= g->nlocal) return 0;
  const std::vector<TraceRec>& t = g->trace[local];
  const uint32_t n = (uint32_t)std::min<size_t>(t.size(), m);
  for (uint32_t i = 0; i < n; ++i) {
    const TraceRec& r = t[t.size() - n + i];
    out[3 * i] = r.id;
    out[3 * i + 1] = r.t_ready;
    out[3 * i + 2] = r.t_agreed;
  }
  return n;
}
}  // namespace hvd_neg

extern "C" {

int hvd_negotiator_create(const char* shm_name, int rank, int size, int nlocal, uint32_t max_tensors,
                          uint64_t timeout_ms, hvd_negotiator** out) {
  if (!out || size < 1 || rank < 0 || nlocal < 1 || rank + nlocal > size || max_tensors == 0 ||
      max_tensors > (1u << 24))
    return HVD_ERR_INVALID;
  if (shm_name && (shm_name[0] != '/' || nlocal != 1)) return HVD_ERR_INVALID;
  *out = nullptr;
  hvd_negotiator* g = new hvd_negotiator();
  g->rank = rank;
  g->size = size;
  g->nlocal = nlocal;
  g->max = max_tensors;
  g->timeout_ms = timeout_ms ? timeout_ms : 60000;
  g->bytes = sizeof(Header) + (size_t)size * 2 * g->slot_bytes();
  g->pending.assign(nlocal, {});
  g->is_pending.assign(nlocal, std::vector<uint8_t>(max_tensors, 0));
  g->stamp.assign(max_tensors, 0);
  g->nranks.assign(max_tensors, 0);
  g->meta.assign(max_tensors, Entry{0, 0, 0});
  g->t_ready.assign(nlocal, std::vector<uint64_t>(max_tensors, 0));
  g->trace.assign(nlocal, {});
  Header* h = nullptr;
  if (!shm_name) {  // process-private: every rank lives in this process
    g->priv = true;
    g->base = static_cast<char*>(std::calloc(1, g->bytes));
    if (!g->base) {
      delete g;
      return HVD_ERR_INVALID;
    }
    h = reinterpret_cast<Header*>(g->base);
    h->size = (uint32_t)size;
    h->max_tensors = max_tensors;
    h->magic = kMagic;
  } else {
    g->name = shm_name;
    const auto t0 = std::chrono::steady_clock::now();
    if (rank == 0) {
      int fd = shm_open(shm_name, O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) {  // a stale segment of a crashed run: replace it
        shm_unlink(shm_name);
        fd = shm_open(shm_name, O_CREAT | O_EXCL | O_RDWR, 0600);
      }
      if (fd < 0 || ftruncate(fd, (off_t)g->bytes) != 0) {
        if (fd >= 0) close(fd);
        delete g;
        return HVD_ERR_UNSUPPORTED;
      }
      void* p = mmap(nullptr, g->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      close(fd);
      if (p == MAP_FAILED) {
        shm_unlink(shm_name);
        delete g;
        return HVD_ERR_UNSUPPORTED;
      }
      g->base = static_cast<char*>(p);
      g->owner = true;
      std::memset(g->base, 0, g->bytes);
      h = reinterpret_cast<Header*>(g->base);
      h->size = (uint32_t)size;
      h->max_tensors = max_tensors;
      h->creator_pid = (uint32_t)getpid();
      h->creator_start = proc_start((int)getpid());
      __atomic_store_n(&h->magic, kMagic, __ATOMIC_RELEASE);
    } else {
      for (;;) {  // wait for rank 0 to create and initialise the segment
        int fd = shm_open(shm_name, O_RDWR, 0600);
        if (fd >= 0) {
          struct stat st;
          if (fstat(fd, &st) == 0 && (size_t)st.st_size >= g->bytes) {
            void* p = mmap(nullptr, g->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (p != MAP_FAILED) {
              h = reinterpret_cast<Header*>(p);
              if (__atomic_load_n(&h->magic, __ATOMIC_ACQUIRE) == kMagic && creator_alive(h)) {
                g->base = static_cast<char*>(p);
                break;
              }
              munmap(p, g->bytes);
            }
          } else {
            close(fd);
          }
        }
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(g->timeout_ms)) {
          delete g;
          return HVD_ERR_TIMEOUT;
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (h->size != (uint32_t)size || h->max_tensors != max_tensors) {
        munmap(g->base, g->bytes);
        delete g;
        return HVD_ERR_INVALID;
      }
    }
  }
  *out = g;
  return HVD_OK;
}

int hvd_negotiator_ready(hvd_negotiator* g, int local, uint32_t id, uint64_t count, int dtype) {
  if (!g || local < 0 || local >= g->nlocal || id >= g->max || !valid_dtype(dtype)) return HVD_ERR_INVALID;
  if (g->is_pending[local][id]) return HVD_ERR_INVALID;
  g->is_pending[local][id] = 1;
  g->t_ready[local][id] = now_ns();
  g->pending[local].push_back(Entry{id, dtype, count});
  return HVD_OK;
}

int hvd_negotiator_cycle(hvd_negotiator* g, uint32_t* ids_out, uint32_t* n_out) {
  if (!g || !ids_out || !n_out) return HVD_ERR_INVALID;
  const uint64_t k = ++g->cycle;
  const int par = (int)(k & 1);
  // publish this process's ranks
  for (int l = 0; l < g->nlocal; ++l) {
    char* s = g->slot(g->rank + l, par);
    SlotHead* sh = reinterpret_cast<SlotHead*>(s);
    Entry* e = reinterpret_cast<Entry*>(s + sizeof(SlotHead));
    const std::vector<Entry>& p = g->pending[l];
    if (!p.empty()) std::memcpy(e, p.data(), p.size() * sizeof(Entry));
    sh->n = p.size();
    __atomic_store_n(&sh->seq, k, __ATOMIC_RELEASE);
  }
  // wait for every rank's cycle-k list
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < g->size; ++r) {
    SlotHead* sh = reinterpret_cast<SlotHead*>(g->slot(r, par));
    unsigned spins = 0;
    while (__atomic_load_n(&sh->seq, __ATOMIC_ACQUIRE) < k) {
      if (++spins > 64) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(g->timeout_ms)) {
          --g->cycle;  // this cycle did not happen (the lists stay pending)
          return HVD_ERR_TIMEOUT;
        }
        sched_yield();
      }
    }
  }
  // intersect: an id is agreed when all ranks list it; order = rank 0's list
  for (int r = 0; r < g->size; ++r) {
    const char* s = g->slot(r, par);
    const uint64_t n = reinterpret_cast<const SlotHead*>(s)->n;
    const Entry* e = reinterpret_cast<const Entry*>(s + sizeof(SlotHead));
    for (uint64_t i = 0; i < n; ++i) {
      const Entry x = e[i];
      if (x.id >= g->max) return HVD_ERR_INVALID;
      if (g->stamp[x.id] != k) {
        g->stamp[x.id] = k;
        g->nranks[x.id] = 1;
        g->meta[x.id] = x;
      } else {
        if (g->meta[x.id].dtype != x.dtype || g->meta[x.id].count != x.count) {
          *n_out = x.id;  // protocol error: the same tensor reported differently
          return HVD_ERR_INVALID;
        }
        g->nranks[x.id] += 1;
      }
    }
  }
  g->agreed.clear();
  {
    const char* s = g->slot(0, par);
    const uint64_t n = reinterpret_cast<const SlotHead*>(s)->n;
    const Entry* e = reinterpret_cast<const Entry*>(s + sizeof(SlotHead));
    for (uint64_t i = 0; i < n; ++i)
      if (g->nranks[e[i].id] == (uint32_t)g->size) g->agreed.push_back(e[i]);
  }
  for (size_t i = 0; i < g->agreed.size(); ++i) ids_out[i] = g->agreed[i].id;
  *n_out = (uint32_t)g->agreed.size();
  // drop the agreed ids from the local pending lists (order of the rest kept)
  const uint64_t t_agreed = now_ns();
  for (int l = 0; l < g->nlocal; ++l) {
    for (const Entry& a : g->agreed)
      if (g->trace[l].size() < kTraceCap) g->trace[l].push_back(TraceRec{a.id, g->t_ready[l][a.id], t_agreed});
    for (const Entry& a : g->agreed) g->is_pending[l][a.id] = 2;  // mark for removal
    std::vector<Entry>& p = g->pending[l];
    size_t w = 0;
    for (size_t i = 0; i < p.size(); ++i) {
      if (g->is_pending[l][p[i].id] == 2) {
        g->is_pending[l][p[i].id] = 0;
      } else {
        p[w++] = p[i];
      }
    }
    p.resize(w);
  }
  return HVD_OK;
}

int hvd_negotiator_pending(const hvd_negotiator* g, int local, uint32_t* ids_out, uint32_t* n_out) {
  if (!g || !n_out || local < 0 || local >= g->nlocal) return HVD_ERR_INVALID;
  const std::vector<Entry>& p = g->pending[local];
  if (ids_out)
    for (size_t i = 0; i < p.size(); ++i) ids_out[i] = p[i].id;
  *n_out = (uint32_t)p.size();
  return HVD_OK;
}

int hvd_negotiator_trace(hvd_negotiator* g, int local, uint64_t* out, uint32_t cap, uint32_t* n_out) {
  if (!g || !n_out || local < 0 || local >= g->nlocal) return HVD_ERR_INVALID;
  std::vector<TraceRec>& t = g->trace[local];
  if (!out) {
    *n_out = (uint32_t)t.size();
    return HVD_OK;
  }
  const uint32_t n = (uint32_t)std::min<size_t>(t.size(), cap);
  for (uint32_t i = 0; i < n; ++i) {
    out[3 * i] = t[i].id;
    out[3 * i + 1] = t[i].t_ready;
    out[3 * i + 2] = t[i].t_agreed;
  }
  *n_out = n;
  t.erase(t.begin(), t.begin() + n);
  return HVD_OK;
}

int hvd_negotiator_destroy(hvd_negotiator* g) {
  if (!g) return HVD_OK;
  if (g->priv) {
    std::free(g->base);
  } else if (g->base) {
    munmap(g->base, g->bytes);
    if (g->owner) shm_unlink(g->name.c_str());
  }
  delete g;
  return HVD_OK;
}

}  // extern "C"
