// Job-wide Horovod Timeline (§6): a Chrome about:tracing trace of
// what every rank was doing throughout the job — one span per API call on a "host calls"
// lane and one span per kernel launch on a "device kernels" lane, per rank.  Enabled by
// one environment variable (HVD_TIMELINE=<path>) or hvd_timeline_start.
#pragma once

#include <cstdint>
#include <deque>
#include <vector>
#include <string>

#include <cuda_runtime.h>

#include "hvd_internal.h"

namespace hvd {

class JobTrace {
 public:
  // ranks[l]: ring rank of local rank l.  truncate: start a new file (writes "[").
  // Returns an hvd_status; *out stays null on failure.
  static int create(const char* path, bool truncate, int device, int nlocal, const int* ranks, int size,
                    JobTrace** out);
  ~JobTrace();

  // Timeline record for the launch about to be issued (seq not consumed until launched()).
  JtRef reserve();
  // The reserved launch was issued: kind = HVD_KERNEL_*, bytes = payload it reduces/copies.
  void launched(int kind, uint64_t bytes);

  // Host span of one public API call (nested calls fold into the outermost).
  void call_begin(const char* name, uint64_t tensors, uint64_t bytes);
  void call_end(int status);
  // Negotiation phase of one tensor on local rank `local`: reported ready at
  // t_ready, agreed by every rank at t_agreed (CLOCK_REALTIME ns); a span on the
  // "negotiation" lane.
  void negotiate(int local, uint64_t id, int64_t t_ready, int64_t t_agreed);

  // Write the records of finished launches; all = the device is synchronised, so a
  // launch still unfinished never will be (dropped and counted).
  void drain(bool all);
  void flush();

  uint64_t launches() const { return seq_; }
  uint64_t dropped() const { return dropped_; }
  double clock_uncertainty_us() const { return clk_err_ns_ * 1e-3; }

 private:
  struct Meta {
    uint64_t seq, call, bytes;
    int kind;
    int64_t t_launch;  // host ns
  };
  JobTrace() = default;
  int calibrate();
  double dev_us(uint64_t g) const;  // device %globaltimer -> host CLOCK_REALTIME, microseconds
  void append(const char* line, int len);

  int fd_ = -1;
  int device_ = 0, nlocal_ = 1, size_ = 1;
  int ranks_[kMaxLocal] = {};
  unsigned long long* dev_ = nullptr;    // [kJtSlots][kMaxLocal][kJtWords]
  unsigned long long* host_ = nullptr;   // host-mapped, same shape
  unsigned long long* hostd_ = nullptr;  // device alias of host_
  unsigned long long* clk_ = nullptr;    // host-mapped word for the clock calibration
  unsigned long long* clkd_ = nullptr;
  cudaStream_t stream_ = nullptr;
  int64_t offset_ns_ = 0;                // globaltimer - CLOCK_REALTIME
  int64_t clk_err_ns_ = 0;
  uint64_t seq_ = 0, dropped_ = 0, call_id_ = 0;
  int depth_ = 0;
  int64_t call_t0_ = 0;
  uint64_t call_launches_ = 0;
  std::string call_name_;
  uint64_t call_tensors_ = 0, call_bytes_ = 0;
  std::deque<Meta> pending_;
  std::string out_;
};

int64_t realtime_ns();

}  // namespace hvd
