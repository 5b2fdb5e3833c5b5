// bs_internal.h — host-side runtime shared by the C-ABI translation units:
// the context (stream, growable device/pinned scratch, last error), the
// uploaded model set, and error helpers.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <condition_variable>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "biscale_gpu.h"
#include "bs_device.cuh"

namespace bs {
struct HostPool;
#ifndef BS_HOST_WORKERS
#define BS_HOST_WORKERS 3
#endif
constexpr int kHostWorkers = BS_HOST_WORKERS;  // host pool workers (plus the calling thread)
}  // namespace bs

struct bs_ctx_s {
  int device = 0;
  uint64_t last_h2d = 0;  // bytes moved by the last entry point
  uint64_t last_d2h = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  double stats[16] = {};  // phase timings / counters of the last entry point
  int n_stats = 0;
  int grid_cache[8] = {};  // occupancy-sized persistent grids, computed once per context (bs_mpc.cu)
  // exhaustive-MPC limits (bs_ctx_set_exhaustive_limits): the sweep-depth
  // threshold and the frontier capacities (12 B per final entry: 24 GB; 40 B
  // per level entry, two ping-pong lists: 20 GB)
  double ex_sweep3_min = 16777216.0;
  unsigned long long ex_level_cap = 250000000ull;
  unsigned long long ex_final_cap = 2000000000ull;
  std::unique_ptr<bs::HostPool> host_pool;  // started on first use (parallel_chunks)
  cudaEvent_t slice_ev[4] = {};  // per-slice D2H events of the MPC result copy (created once, bs_mpc.cu)
  size_t greedy_smem[6] = {};     // dynamic shared memory the greedy kernels were opened to (bs_mpc.cu)
  int greedy_no_cluster = -1;     // BS_GREEDY_NO_CLUSTER set: no cluster launch for single decisions (A/B)
  std::string fg_key;             // (models, pairs) of the reduced grids in the one-shot slot (bs_mpc.cu)
  bs::HostPool& pool();

  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  static constexpr int kSlots = 16;
  Buf dev[kSlots];
  Buf host[kSlots];

  void* dev_buf(int slot, size_t bytes);   // grow-only device scratch
  void* host_buf(int slot, size_t bytes);  // grow-only pinned host scratch
  ~bs_ctx_s();
};

struct bs_models_s {
  unsigned long long serial = 0;  // unique per upload (caches keyed on a model set)
  bs::DModels dm{};
  void* dmem = nullptr;  // one allocation: knots, values, idle arrays
  size_t bytes = 0;
  bool grid_positive[4] = {false, false, false, false};  // every value > 0 and finite
  std::vector<double> hbuf;  // host mirror of dmem's doubles
  bs::DGrid hgrid[4]{};      // dm.grid with pointers into hbuf (host-side FastGrid construction)
};

namespace bs {

// Scratch slot ids (each kernel family owns a few).
enum Slot : int {
  kSlotCfg = 0,
  kSlotProblems = 1,
  kSlotWaiting = 2,
  kSlotRunning = 3,
  kSlotTables = 4,
  kSlotOut = 5,
  kSlotLevels = 6,
  kSlotBest = 7,
  kSlotWork = 8,
  kSlotCounts = 9,
  kSlotMisc = 10,
  kSlotMisc2 = 11,
  kSlotReplay = 12,
  kSlotFastGrids = 13,
  kSlotIlp = 14,
};

int set_error(bs_ctx_t ctx, int code, const char* fmt, ...);

// The calling thread's default context on device 0 (created on first use;
// nullptr when no device is usable): what the entry points that accept a
// NULL context run on.
bs_ctx_t default_ctx();

#define BS_CUDA_TRY(ctx, expr)                                                                     \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return ::bs::set_error((ctx), BS_CUDA_ERROR, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                             __FILE__, __LINE__);                                                  \
  } while (0)

#define BS_LAUNCH_CHECK(ctx)                                                                         \
  do {                                                                                               \
    (ctx)->launches += 1;                                                                            \
    cudaError_t e_ = cudaGetLastError();                                                             \
    if (e_ != cudaSuccess)                                                                           \
      return ::bs::set_error((ctx), BS_CUDA_ERROR, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), \
                             __FILE__, __LINE__);                                                    \
  } while (0)

// FrequencyLadder::validate + select (perfmodel.hpp:56-91) on the host;
// returns the candidate count or a negative status.
int ladder_select(bs_ctx_t ctx, const double* ladder, int n_ladder, int n, double* out, int cap);

// MpcConfig::validate (dvfs.hpp:25-31) and SchedulerPolicy::validate
// (scheduler.hpp:17-21), then pack into the device layout.
int pack_mpc_cfg(bs_ctx_t ctx, const bs_mpc_config& c, const bs_scheduler_policy& p, DMpcCfg* out);

// Packs problems + configs into one pinned staging buffer and copies it to
// HBM with a single cudaMemcpyAsync.  Device pointers returned in `dev`.
struct PackedProblems {
  DMpcCfg* cfgs = nullptr;
  DProblem* problems = nullptr;
  DWaiting* waiting = nullptr;
  DRunning* running = nullptr;
  char* base = nullptr;  // device blob holding all four arrays
  size_t off_cfg = 0, off_prob = 0, off_wait = 0, off_run = 0;
  int n = 0;
  int n_cfgs = 0;
  size_t h2d_bytes = 0;
  int max_horizon = 0;
  int max_nc = 0;
  std::vector<std::pair<int, int>> fg_pairs;  // distinct (configuration, tp); DProblem::fgi indexes them
  void rebase(char* b) {
    base = b;
    cfgs = reinterpret_cast<DMpcCfg*>(b + off_cfg);
    problems = reinterpret_cast<DProblem*>(b + off_prob);
    waiting = reinterpret_cast<DWaiting*>(b + off_wait);
    running = reinterpret_cast<DRunning*>(b + off_run);
  }
};
int pack_problems(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies, int n_cfgs,
                  const bs_mpc_problem* problems, int n, PackedProblems* out);

// A small pool of host worker threads owned by a context, started on first
// use and blocked on a condition variable between jobs (they never spin, so
// they take no cores from anything else the process runs).  run(tasks, fn)
// calls fn(i) for i in [0, tasks) on the workers and the calling thread and
// returns when all are done.
struct HostPool {
  std::vector<std::thread> th;
  std::mutex m;
  std::condition_variable cv, done_cv;
  std::function<void(int)> job;
  int tasks = 0, next = 0, finished = 0;
  unsigned long long gen = 0;
  bool stop = false;

  void start(int workers) {
    for (int w = 0; w < workers; ++w)
      th.emplace_back([this] {
        unsigned long long seen = 0;
        for (;;) {
          std::unique_lock<std::mutex> lk(m);
          cv.wait(lk, [&] { return stop || gen != seen; });
          if (stop) return;
          seen = gen;
          while (next < tasks) {
            const int i = next++;
            lk.unlock();
            job(i);
            lk.lock();
            if (++finished == tasks) done_cv.notify_all();
          }
        }
      });
  }
  void run(int n_tasks, const std::function<void(int)>& fn) {
    std::unique_lock<std::mutex> lk(m);
    job = fn;
    tasks = n_tasks;
    next = 0;
    finished = 0;
    ++gen;
    cv.notify_all();
    while (next < tasks) {  // the caller takes tasks too
      const int i = next++;
      lk.unlock();
      job(i);
      lk.lock();
      ++finished;
    }
    done_cv.wait(lk, [&] { return finished == tasks; });
    job = nullptr;
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : th) t.join();
  }
};

// fn(begin, end) over [0, n) in contiguous chunks of at least `grain` items
// on the context's host pool (serial for small n).  Used for the per-problem
// host work of large batches (packing, result expansion), independent per item.
template <class Fn>
void parallel_chunks(bs_ctx_t ctx, int n, int grain, Fn&& fn) {
  const int chunks = std::min(kHostWorkers + 1, n / std::max(1, grain));
  if (chunks <= 1 || !ctx) {
    fn(0, n);
    return;
  }
  HostPool& pool = ctx->pool();
  pool.run(chunks, [&](int c) {
    fn(static_cast<int>(static_cast<long long>(n) * c / chunks),
       static_cast<int>(static_cast<long long>(n) * (c + 1) / chunks));
  });
}

}  // namespace bs
