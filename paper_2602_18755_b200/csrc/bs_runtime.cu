// bs_runtime.cu — context, model upload, packing and the model-query entry
// points of the C ABI (include/biscale_gpu.h).
#include <cstddef>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>

#include <atomic>

#include "bs_internal.h"

using namespace bs;

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------

void* bs_ctx_s::dev_buf(int slot, size_t bytes) {
  Buf& b = dev[slot];
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return b.p;
  if (b.p) cudaFree(b.p);
  size_t cap = std::max(bytes, b.cap * 2);
  b.p = nullptr;
  b.cap = 0;
  if (cudaMalloc(&b.p, cap) != cudaSuccess) {
    b.p = nullptr;
    return nullptr;
  }
  b.cap = cap;
  return b.p;
}

void* bs_ctx_s::host_buf(int slot, size_t bytes) {
  Buf& b = host[slot];
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return b.p;
  if (b.p) cudaFreeHost(b.p);
  size_t cap = std::max(bytes, b.cap * 2);
  b.p = nullptr;
  b.cap = 0;
  if (cudaMallocHost(&b.p, cap) != cudaSuccess) {
    b.p = nullptr;
    return nullptr;
  }
  b.cap = cap;
  return b.p;
}

bs::HostPool& bs_ctx_s::pool() {
  if (!host_pool) {
    host_pool = std::make_unique<bs::HostPool>();
    host_pool->start(bs::kHostWorkers);
  }
  return *host_pool;
}

bs_ctx_s::~bs_ctx_s() {
  for (cudaEvent_t e : slice_ev)
    if (e) cudaEventDestroy(e);
  for (auto& b : dev)
    if (b.p) cudaFree(b.p);
  for (auto& b : host)
    if (b.p) cudaFreeHost(b.p);
  if (stream) cudaStreamDestroy(stream);
}

namespace bs {

thread_local std::string g_host_err;

bs_ctx_t default_ctx() {
  struct Holder {
    bs_ctx_t c = nullptr;
    bool tried = false;
    ~Holder() {
      if (c) bs_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.tried) {
    h.tried = true;
    if (bs_ctx_create(0, &h.c) != BS_OK) h.c = nullptr;
  }
  return h.c;
}

int set_error(bs_ctx_t ctx, int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx)
    ctx->err = buf;
  else
    g_host_err = buf;  // host-only entry points called without a context
  return code;
}

int ladder_select(bs_ctx_t ctx, const double* l, int size, int n, double* out, int cap) {
  if (size < 1 || l == nullptr) return -set_error(ctx, BS_PARAMETER_ERROR, "frequency ladder: empty");
  double prev = 0.0;
  for (int i = 0; i < size; ++i) {
    if (l[i] <= prev)
      return -set_error(ctx, BS_PARAMETER_ERROR, "frequency ladder: must be strictly increasing and > 0");
    prev = l[i];
  }
  if (n == 0 || n < 0) return -set_error(ctx, BS_PARAMETER_ERROR, "frequency ladder: select(0)");
  int m = 0;
  auto push = [&](double v) {
    if (m == 0 || out[m - 1] != v) {
      if (m < cap) out[m] = v;
      ++m;
    }
  };
  if (n >= size) {
    for (int i = 0; i < size; ++i) push(l[i]);
  } else if (n == 1) {
    push(l[size - 1]);
  } else {
    for (int i = 0; i < n; ++i) {
      size_t idx = (static_cast<size_t>(i) * static_cast<size_t>(size - 1)) / static_cast<size_t>(n - 1);
      push(l[idx]);
    }
  }
  if (m > cap) return -set_error(ctx, BS_PARAMETER_ERROR, "mpc: %d candidate rungs exceed the device limit %d", m, cap);
  return m;
}

int pack_mpc_cfg(bs_ctx_t ctx, const bs_mpc_config& c, const bs_scheduler_policy& p, DMpcCfg* out) {
  std::memset(out, 0, sizeof *out);
  if (c.horizon_K < 1) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: horizon_K must be >= 1");
  if (c.ladder_N < 1) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: ladder_N must be >= 1");
  int nc = ladder_select(ctx, c.ladder_mhz, c.n_ladder, c.ladder_N, out->cand, kMaxCand);
  if (nc < 0) return -nc;
  if (c.ttft_ms <= 0.0 || c.tpot_ms <= 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "slo: bounds must be > 0");
  if (c.percentile <= 0.0 || c.percentile > 1.0)
    return set_error(ctx, BS_PARAMETER_ERROR, "slo: percentile must be in (0,1]");
  if (c.margin < 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: margin must be >= 0");
  if (c.horizon_K > kMaxK)
    return set_error(ctx, BS_PARAMETER_ERROR, "mpc: horizon_K %d exceeds the device limit %d", c.horizon_K, kMaxK);
  if (p.max_batch_tokens < 1) return set_error(ctx, BS_PARAMETER_ERROR, "scheduler: max_batch_tokens must be >= 1");
  if (p.max_batch_requests < 1)
    return set_error(ctx, BS_PARAMETER_ERROR, "scheduler: max_batch_requests must be >= 1");
  if (p.kv_capacity_tokens < 1)
    return set_error(ctx, BS_PARAMETER_ERROR, "scheduler: kv_capacity_tokens must be >= 1");
  out->horizon = c.horizon_K;
  out->nc = nc;
  out->ttft = c.ttft_ms;
  out->switch_ms = c.switch_latency_ms;
  out->one_plus_margin = 1.0 + c.margin;
  out->max_mhz = out->cand[nc - 1];
  out->max_batch_tokens = p.max_batch_tokens;
  out->max_batch_requests = p.max_batch_requests;
  out->chunking = p.chunking ? 1 : 0;
  return BS_OK;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static_assert(sizeof(DWaiting) == sizeof(bs_waiting) && offsetof(DWaiting, id) == offsetof(bs_waiting, id) &&
                  offsetof(DWaiting, arrival) == offsetof(bs_waiting, arrival_ms) &&
                  offsetof(DWaiting, total) == offsetof(bs_waiting, total_len) &&
                  offsetof(DWaiting, remaining) == offsetof(bs_waiting, remaining_len),
              "DWaiting mirrors bs_waiting");

// Problems per host-pool chunk of the pack copies.
#ifndef BS_PACK_GRAIN
#define BS_PACK_GRAIN 256
#endif
// Minimum problems per pipelined pack slice (H2D of a slice overlaps the next slice's packing).
#ifndef BS_PACK_SLICE
#define BS_PACK_SLICE 256
#endif
#ifndef BS_PACK_SLICES_MAX
#define BS_PACK_SLICES_MAX 4
#endif

int pack_problems(bs_ctx_t ctx, const bs_mpc_config* cfgs, const bs_scheduler_policy* policies, int n_cfgs,
                  const bs_mpc_problem* problems, int n, PackedProblems* out) {
  out->fg_pairs.clear();
  if (n_cfgs < 1 || cfgs == nullptr || policies == nullptr)
    return set_error(ctx, BS_PARAMETER_ERROR, "mpc: no controller configuration");
  if (n < 0) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: negative problem count");
  size_t n_wait = 0, n_run = 0;
  for (int i = 0; i < n; ++i) {
    const bs_snapshot& s = problems[i].snap;
    if (problems[i].cfg_index < 0 || problems[i].cfg_index >= n_cfgs)
      return set_error(ctx, BS_PARAMETER_ERROR, "mpc: problem %d has cfg_index %d out of range", i,
                       problems[i].cfg_index);
    if (s.n_waiting < 0 || s.n_running < 0) return set_error(ctx, BS_PARAMETER_ERROR, "mpc: negative queue size");
    n_wait += static_cast<size_t>(s.n_waiting);
    if (s.running_active) n_run += static_cast<size_t>(s.n_running);
  }
  const size_t o_cfg = 0;
  const size_t o_prob = align_up(o_cfg + sizeof(DMpcCfg) * n_cfgs, 256);
  const size_t o_wait = align_up(o_prob + sizeof(DProblem) * std::max(n, 1), 256);
  const size_t o_run = align_up(o_wait + sizeof(DWaiting) * std::max<size_t>(n_wait, 1), 256);
  const size_t total = align_up(o_run + sizeof(DRunning) * std::max<size_t>(n_run, 1), 256);
  char* h = static_cast<char*>(ctx->host_buf(kSlotProblems, total));
  char* d = static_cast<char*>(ctx->dev_buf(kSlotProblems, total));
  if (!h || !d) return set_error(ctx, BS_CUDA_ERROR, "mpc: cannot allocate %zu bytes of staging", total);

  DMpcCfg* hc = reinterpret_cast<DMpcCfg*>(h + o_cfg);
  int max_h = 0, max_nc = 0;
  for (int c = 0; c < n_cfgs; ++c) {
    int rc = pack_mpc_cfg(ctx, cfgs[c], policies[c], &hc[c]);
    if (rc) return rc;
    max_h = std::max(max_h, hc[c].horizon);
    max_nc = std::max(max_nc, hc[c].nc);
  }
  DProblem* hp = reinterpret_cast<DProblem*>(h + o_prob);
  DWaiting* hw = reinterpret_cast<DWaiting*>(h + o_wait);
  DRunning* hr = reinterpret_cast<DRunning*>(h + o_run);
  // serial: offsets and the distinct (configuration, tp) pairs; then the
  // independent per-problem copies, in parallel for large batches
  std::vector<size_t> woff(static_cast<size_t>(n) + 1), roff(static_cast<size_t>(n) + 1);
  std::vector<int> fgi(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const bs_snapshot& s = problems[i].snap;
    woff[i + 1] = woff[i] + static_cast<size_t>(s.n_waiting);
    roff[i + 1] = roff[i] + (s.running_active ? static_cast<size_t>(s.n_running) : 0);
    const std::pair<int, int> key(problems[i].cfg_index, s.tp);
    auto it = std::find(out->fg_pairs.begin(), out->fg_pairs.end(), key);
    fgi[i] = static_cast<int>(it - out->fg_pairs.begin());
    if (it == out->fg_pairs.end()) out->fg_pairs.push_back(key);
  }
  // Large batches are packed in slices of problems; each slice's ranges of
  // the problem / waiting / running regions are copied as soon as the slice
  // is packed, so the H2D transfer overlaps the packing of the next slice.
  const int n_slices = std::max(1, std::min(BS_PACK_SLICES_MAX, n / BS_PACK_SLICE));
  for (int sl = 0; sl < n_slices; ++sl) {
    const int s_lo = static_cast<int>(static_cast<long long>(n) * sl / n_slices);
    const int s_hi = static_cast<int>(static_cast<long long>(n) * (sl + 1) / n_slices);
    parallel_chunks(ctx, s_hi - s_lo, BS_PACK_GRAIN, [&](int lo, int hi) {
      for (int i = s_lo + lo; i < s_lo + hi; ++i) {
        const bs_snapshot& s = problems[i].snap;
        DProblem& p = hp[i];
        p.now = s.now_ms;
        p.cur_freq = s.current_freq_mhz;
        p.target_freq = s.target_freq_mhz;
        p.run_wr = s.running_work_remaining;
        p.run_n = s.running_features.n_requests;
        p.run_sum = s.running_features.sum_len;
        p.tp = s.tp;
        p.run_active = s.running_active ? 1 : 0;
        p.n_wait = s.n_waiting;
        p.n_run = s.running_active ? s.n_running : 0;
        p.cfg = problems[i].cfg_index;
        p.fgi = fgi[i];
        p.wait_off = static_cast<long long>(woff[i]);
        p.run_off = static_cast<long long>(roff[i]);
        // bs_waiting and DWaiting share one layout (static_asserts above): one copy per snapshot
        if (s.n_waiting > 0) std::memcpy(hw + woff[i], s.waiting, sizeof(DWaiting) * static_cast<size_t>(s.n_waiting));
        if (s.running_active) {
          for (int j = 0; j < s.n_running; ++j) {
            hr[roff[i] + j].arrival = s.running_arrivals_ms[j];
            hr[roff[i] + j].completes = s.running_completes[j] ? 1 : 0;
          }
        }
      }
    });
    if (n_slices == 1) {
      BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, ctx->stream));
      break;
    }
    auto h2d = [&](size_t off, size_t bytes) -> int {
      if (bytes) BS_CUDA_TRY(ctx, cudaMemcpyAsync(d + off, h + off, bytes, cudaMemcpyHostToDevice, ctx->stream));
      return BS_OK;
    };
    if (sl == 0 && h2d(o_cfg, o_prob - o_cfg)) return BS_CUDA_ERROR;
    if (h2d(o_prob + sizeof(DProblem) * s_lo, sizeof(DProblem) * (s_hi - s_lo)) ||
        h2d(o_wait + sizeof(DWaiting) * woff[s_lo], sizeof(DWaiting) * (woff[s_hi] - woff[s_lo])) ||
        h2d(o_run + sizeof(DRunning) * roff[s_lo], sizeof(DRunning) * (roff[s_hi] - roff[s_lo])))
      return BS_CUDA_ERROR;
  }
  out->off_cfg = o_cfg;
  out->off_prob = o_prob;
  out->off_wait = o_wait;
  out->off_run = o_run;
  out->rebase(d);
  out->n = n;
  out->n_cfgs = n_cfgs;
  out->h2d_bytes = total;
  out->max_horizon = max_h;
  out->max_nc = max_nc;
  return BS_OK;
}

}  // namespace bs

// ---------------------------------------------------------------------------
// model kernels
// ---------------------------------------------------------------------------

namespace {

__global__ void predict_kernel(DModels m, int which, const bs_features* feats, const int32_t* tp, const double* freq,
                               int n, double* out, int32_t* status, uint32_t* clamps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned c = 0;
  double v = 0.0;
  int st = BS_OK;
  if (which < 4) {
    const DGrid& g = m.grid[which];
    if (g.bad_axis) {
      st = BS_MODEL_ERROR;
    } else {
      v = interp(g, make_query(feats[i].n_requests, feats[i].sum_len, tp[i], freq[i]), &c);
      if (!model_value_ok(v)) st = BS_MODEL_ERROR;
    }
  } else {
    if (!idle_power(m.idle, tp[i], freq[i], &v)) st = BS_MODEL_ERROR;
  }
  out[i] = st == BS_OK ? v : 0.0;
  status[i] = st;
  if (clamps) clamps[i] = c;
}

__global__ void interp_kernel(DGrid g, const double* coords, int n, double* out, uint32_t* clamps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned c = 0;
  out[i] = interp_coords(g, coords + static_cast<size_t>(i) * g.rank, &c);
  if (clamps) clamps[i] = c;
}

// FP64 issue microbenchmark: 8 independent DADD chains per thread.
__global__ void __launch_bounds__(256) fp64_issue_kernel(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1.0, x2 = x0 + 2.0, x3 = x0 + 3.0;
  double x4 = x0 + 4.0, x5 = x0 + 5.0, x6 = x0 + 6.0, x7 = x0 + 7.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = __dadd_rn(x0, a);
      x1 = __dadd_rn(x1, a);
      x2 = __dadd_rn(x2, a);
      x3 = __dadd_rn(x3, a);
      x4 = __dadd_rn(x4, a);
      x5 = __dadd_rn(x5, a);
      x6 = __dadd_rn(x6, a);
      x7 = __dadd_rn(x7, a);
    }
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678) out[blockIdx.x] = s;  // keeps the chains live
}

int validate_grid(bs_ctx_t ctx, const bs_grid& g, const char* name) {
  if (g.rank < 1) return set_error(ctx, BS_MODEL_ERROR, "grid: no axes (%s)", name);
  if (g.rank > kMaxRank) return set_error(ctx, BS_PARAMETER_ERROR, "grid %s: rank %d > %d", name, g.rank, kMaxRank);
  for (int d = 0; d < g.rank; ++d) {
    if (g.n_knots[d] < 1 || g.knots[d] == nullptr) return set_error(ctx, BS_MODEL_ERROR, "grid: axis has no knots (%s)", name);
    for (int i = 1; i < g.n_knots[d]; ++i)
      if (g.knots[d][i] <= g.knots[d][i - 1])
        return set_error(ctx, BS_MODEL_ERROR, "grid: axis knots not strictly increasing (%s)", name);
  }
  if (g.values == nullptr) return set_error(ctx, BS_MODEL_ERROR, "grid: value count does not match axes (%s)", name);
  return BS_OK;
}

size_t grid_values(const bs_grid& g) {
  size_t n = 1;
  for (int d = 0; d < g.rank; ++d) n *= static_cast<size_t>(g.n_knots[d]);
  return n;
}

}  // namespace

extern "C" {

int bs_abi_version(void) { return BS_ABI_VERSION; }

int bs_ctx_create(int device, bs_ctx_t* out) {
  if (!out) return BS_PARAMETER_ERROR;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return BS_CUDA_ERROR;
  if (device < 0 || device >= count) return BS_PARAMETER_ERROR;
  if (cudaSetDevice(device) != cudaSuccess) return BS_CUDA_ERROR;
  bs_ctx_t ctx = new (std::nothrow) bs_ctx_s();
  if (!ctx) return BS_CUDA_ERROR;
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return BS_CUDA_ERROR;
  }
  *out = ctx;
  return BS_OK;
}

void bs_ctx_destroy(bs_ctx_t ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

const char* bs_last_error(bs_ctx_t ctx) { return ctx ? ctx->err.c_str() : bs::g_host_err.c_str(); }

int bs_ctx_info(bs_ctx_t ctx, int* device, int* sm_count) {
  if (!ctx) return BS_PARAMETER_ERROR;
  if (device) *device = ctx->device;
  if (sm_count) *sm_count = ctx->sm_count;
  return BS_OK;
}

int bs_ctx_set_exhaustive_limits(bs_ctx_t ctx, double sweep3_min_prefixes, uint64_t level_cap, uint64_t final_cap) {
  if (!ctx) return BS_PARAMETER_ERROR;
  if (!(sweep3_min_prefixes >= 0.0))
    return bs::set_error(ctx, BS_PARAMETER_ERROR, "exhaustive limits: sweep threshold must be >= 0");
  ctx->ex_sweep3_min = sweep3_min_prefixes > 0.0 ? sweep3_min_prefixes : 16777216.0;
  ctx->ex_level_cap = level_cap ? level_cap : 250000000ull;
  ctx->ex_final_cap = final_cap ? final_cap : 2000000000ull;
  return BS_OK;
}

int bs_ctx_sync(bs_ctx_t ctx) {
  if (!ctx) return BS_PARAMETER_ERROR;
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return BS_OK;
}

int64_t bs_ctx_kernel_launches(bs_ctx_t ctx) { return ctx ? ctx->launches : -1; }

int bs_ctx_stats(bs_ctx_t ctx, double* out, int n) {
  if (!ctx || !out) return 0;
  const int m = std::min(n, ctx->n_stats);
  for (int i = 0; i < m; ++i) out[i] = ctx->stats[i];
  return ctx->n_stats;
}

void* bs_ctx_stream(bs_ctx_t ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int bs_ctx_last_transfer(bs_ctx_t ctx, uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  if (!ctx) return BS_PARAMETER_ERROR;
  if (h2d_bytes) *h2d_bytes = ctx->last_h2d;
  if (d2h_bytes) *d2h_bytes = ctx->last_d2h;
  return BS_OK;
}

int bs_fp64_peak(bs_ctx_t ctx, double* ops_per_s, double* ms_out) {
  if (!ctx) return BS_PARAMETER_ERROR;
  double* d = static_cast<double*>(ctx->dev_buf(kSlotMisc2, 8 * 4096));
  if (!d) return set_error(ctx, BS_CUDA_ERROR, "fp64 peak: allocation failed");
  const int blocks = ctx->sm_count * 8, threads = 256, iters = 2048;
  cudaEvent_t e0, e1;
  BS_CUDA_TRY(ctx, cudaEventCreate(&e0));
  BS_CUDA_TRY(ctx, cudaEventCreate(&e1));
  float best = 1e30f;
  for (int rep = 0; rep < 6; ++rep) {
    BS_CUDA_TRY(ctx, cudaEventRecord(e0, ctx->stream));
    fp64_issue_kernel<<<blocks, threads, 0, ctx->stream>>>(d, iters, 1e-9);
    BS_LAUNCH_CHECK(ctx);
    BS_CUDA_TRY(ctx, cudaEventRecord(e1, ctx->stream));
    BS_CUDA_TRY(ctx, cudaEventSynchronize(e1));
    float ms = 0.f;
    BS_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0 && ms < best) best = ms;  // first launch is warm-up
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double ops = static_cast<double>(blocks) * threads * iters * 32.0;
  if (ops_per_s) *ops_per_s = ops / (best * 1e-3);
  if (ms_out) *ms_out = best;
  return BS_OK;
}

int bs_models_upload(bs_ctx_t ctx, const bs_model_set* m, bs_models_t* out) {
  if (!ctx || !m || !out) return set_error(ctx, BS_PARAMETER_ERROR, "bs_models_upload: null argument");
  *out = nullptr;
  const bs_grid* grids[4] = {&m->latency_prefill, &m->latency_decode, &m->power_prefill, &m->power_decode};
  const char* names[4] = {"latency_prefill", "latency_decode", "power_prefill", "power_decode"};
  size_t doubles = 0;
  for (int i = 0; i < 4; ++i) {
    int rc = validate_grid(ctx, *grids[i], names[i]);
    if (rc) return rc;
    for (int d = 0; d < grids[i]->rank; ++d) doubles += grids[i]->n_knots[d];
    doubles += grid_values(*grids[i]);
  }
  if (m->n_idle < 0 || (m->n_idle > 0 && !m->idle)) return set_error(ctx, BS_PARAMETER_ERROR, "idle model: bad entries");
  size_t idle_pts = 0;
  for (int i = 0; i < m->n_idle; ++i) {
    if (m->idle[i].n < 0) return set_error(ctx, BS_PARAMETER_ERROR, "idle model: negative size");
    idle_pts += static_cast<size_t>(m->idle[i].n);
  }
  doubles += 2 * idle_pts;
  const size_t ints = 3 * static_cast<size_t>(m->n_idle);
  const size_t bytes = doubles * sizeof(double) + ints * sizeof(int) + 64;

  std::vector<char> host(bytes, 0);
  bs_models_t mm = new (std::nothrow) bs_models_s();
  static std::atomic<unsigned long long> serials{0};
  if (mm) mm->serial = ++serials;
  if (!mm) return set_error(ctx, BS_CUDA_ERROR, "out of host memory");
  if (cudaMalloc(&mm->dmem, bytes) != cudaSuccess) {
    delete mm;
    return set_error(ctx, BS_CUDA_ERROR, "cudaMalloc(%zu) for models failed", bytes);
  }
  mm->bytes = bytes;
  char* dbase = static_cast<char*>(mm->dmem);
  double* hd = reinterpret_cast<double*>(host.data());
  size_t o = 0;
  for (int i = 0; i < 4; ++i) {
    const bs_grid& g = *grids[i];
    DGrid& dg = mm->dm.grid[i];
    dg.rank = g.rank;
    dg.bad_axis = 0;
    for (int d = 0; d < kMaxRank; ++d) {
      dg.role[d] = d < g.rank ? g.role[d] : 0;
      dg.n[d] = d < g.rank ? g.n_knots[d] : 1;
      dg.knots[d] = nullptr;
    }
    for (int d = 0; d < g.rank; ++d) {
      if (g.role[d] < BS_AXIS_SUM_LEN || g.role[d] > BS_AXIS_FREQ) dg.bad_axis = 1;
      std::memcpy(hd + o, g.knots[d], sizeof(double) * g.n_knots[d]);
      dg.knots[d] = reinterpret_cast<const double*>(dbase + o * sizeof(double));
      o += g.n_knots[d];
    }
    const size_t nv = grid_values(g);
    std::memcpy(hd + o, g.values, sizeof(double) * nv);
    dg.values = reinterpret_cast<const double*>(dbase + o * sizeof(double));
    bool pos = true;
    for (size_t v = 0; v < nv; ++v)
      if (!(g.values[v] > 0.0) || !std::isfinite(g.values[v]) || g.values[v] > 1e300) pos = false;
    mm->grid_positive[i] = pos;
    o += nv;
  }
  DIdle& di = mm->dm.idle;
  di.n_entries = m->n_idle;
  double* hf = hd + o;
  di.freqs = reinterpret_cast<const double*>(dbase + o * sizeof(double));
  size_t io = 0;
  for (int i = 0; i < m->n_idle; ++i) {
    std::memcpy(hf + io, m->idle[i].freqs_mhz, sizeof(double) * m->idle[i].n);
    io += m->idle[i].n;
  }
  o += idle_pts;
  double* hw = hd + o;
  di.watts = reinterpret_cast<const double*>(dbase + o * sizeof(double));
  io = 0;
  for (int i = 0; i < m->n_idle; ++i) {
    std::memcpy(hw + io, m->idle[i].idle_w, sizeof(double) * m->idle[i].n);
    io += m->idle[i].n;
  }
  o += idle_pts;
  int* hi = reinterpret_cast<int*>(hd + o);
  const size_t int_base = o * sizeof(double);
  di.tp = reinterpret_cast<const int*>(dbase + int_base);
  di.n = reinterpret_cast<const int*>(dbase + int_base + sizeof(int) * m->n_idle);
  di.off = reinterpret_cast<const int*>(dbase + int_base + 2 * sizeof(int) * m->n_idle);
  int off = 0;
  for (int i = 0; i < m->n_idle; ++i) {
    hi[i] = m->idle[i].tp;
    hi[m->n_idle + i] = m->idle[i].n;
    hi[2 * m->n_idle + i] = off;
    off += m->idle[i].n;
  }
  if (cudaMemcpy(mm->dmem, host.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(mm->dmem);
    delete mm;
    return set_error(ctx, BS_CUDA_ERROR, "model upload copy failed");
  }
  // host mirror for host-built FastGrids (bs_sim.cuh fast_grid2)
  mm->hbuf.assign(reinterpret_cast<const double*>(host.data()),
                  reinterpret_cast<const double*>(host.data()) + bytes / sizeof(double));
  for (int i = 0; i < 4; ++i) {
    mm->hgrid[i] = mm->dm.grid[i];
    auto rebase = [&](const double* p) {
      return mm->hbuf.data() + (reinterpret_cast<const char*>(p) - dbase) / sizeof(double);
    };
    for (int d = 0; d < mm->dm.grid[i].rank; ++d) mm->hgrid[i].knots[d] = rebase(mm->dm.grid[i].knots[d]);
    mm->hgrid[i].values = rebase(mm->dm.grid[i].values);
  }
  *out = mm;
  return BS_OK;
}

void bs_models_free(bs_ctx_t ctx, bs_models_t m) {
  (void)ctx;
  if (!m) return;
  if (m->dmem) cudaFree(m->dmem);
  delete m;
}

int bs_predict(bs_ctx_t ctx, bs_models_t models, int which, const bs_features* feats, const int32_t* tp,
               const double* freq, int n, double* out, int32_t* status, uint32_t* clamp_events) {
  if (!ctx || !models) return set_error(ctx, BS_PARAMETER_ERROR, "bs_predict: null context or models");
  if (which < 0 || which > 4) return set_error(ctx, BS_PARAMETER_ERROR, "bs_predict: which must be 0..4");
  if (n <= 0) return BS_OK;
  // layout (every section 256-byte aligned): feats | freq | tp || out | status | clamps
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t o_f = 0, o_fr = up(sizeof(bs_features) * n), o_tp = o_fr + up(sizeof(double) * n);
  const size_t in_bytes = o_tp + up(sizeof(int32_t) * n);
  const size_t o_out = in_bytes, o_st = o_out + up(sizeof(double) * n), o_cl = o_st + up(sizeof(int32_t) * n);
  const size_t total = o_cl + up(sizeof(uint32_t) * n);
  char* h = static_cast<char*>(ctx->host_buf(kSlotMisc, total));
  char* d = static_cast<char*>(ctx->dev_buf(kSlotMisc, total));
  if (!h || !d) return set_error(ctx, BS_CUDA_ERROR, "bs_predict: allocation failed");
  std::memcpy(h + o_f, feats, sizeof(bs_features) * n);
  std::memcpy(h + o_fr, freq, sizeof(double) * n);
  std::memcpy(h + o_tp, tp, sizeof(int32_t) * n);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  predict_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(
      models->dm, which, reinterpret_cast<const bs_features*>(d + o_f), reinterpret_cast<const int32_t*>(d + o_tp),
      reinterpret_cast<const double*>(d + o_fr), n, reinterpret_cast<double*>(d + o_out),
      reinterpret_cast<int32_t*>(d + o_st), reinterpret_cast<uint32_t*>(d + o_cl));
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(h + o_out, d + o_out, total - o_out, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  std::memcpy(out, h + o_out, sizeof(double) * n);
  std::memcpy(status, h + o_st, sizeof(int32_t) * n);
  if (clamp_events) std::memcpy(clamp_events, h + o_cl, sizeof(uint32_t) * n);
  for (int i = 0; i < n; ++i)
    if (status[i] != BS_OK) {
      set_error(ctx, status[i], "%s model returned non-positive value or has an unknown axis",
                which == 0 || which == 1 ? "latency" : (which < 4 ? "power" : "idle"));
      break;
    }
  return BS_OK;
}

int bs_grid_interpolate(bs_ctx_t ctx, const bs_grid* grid, const double* coords, int n, double* out,
                        uint32_t* clamp_events) {
  if (!ctx || !grid) return set_error(ctx, BS_PARAMETER_ERROR, "bs_grid_interpolate: null argument");
  int rc = validate_grid(ctx, *grid, "query");
  if (rc) return rc;
  if (n <= 0) return BS_OK;
  // Temporary upload of one grid: knots + values + coords.
  size_t nk = 0;
  for (int d = 0; d < grid->rank; ++d) nk += grid->n_knots[d];
  const size_t nv = grid_values(*grid);
  const size_t in_doubles = nk + nv + static_cast<size_t>(n) * grid->rank;
  const size_t bytes = in_doubles * sizeof(double) + n * (sizeof(double) + sizeof(uint32_t));
  char* h = static_cast<char*>(ctx->host_buf(kSlotMisc2, bytes));
  char* d = static_cast<char*>(ctx->dev_buf(kSlotMisc2, bytes));
  if (!h || !d) return set_error(ctx, BS_CUDA_ERROR, "bs_grid_interpolate: allocation failed");
  double* hd = reinterpret_cast<double*>(h);
  DGrid g{};
  g.rank = grid->rank;
  size_t o = 0;
  for (int k = 0; k < kMaxRank; ++k) {
    g.n[k] = 1;
    g.role[k] = 0;
  }
  for (int k = 0; k < grid->rank; ++k) {
    g.n[k] = grid->n_knots[k];
    std::memcpy(hd + o, grid->knots[k], sizeof(double) * grid->n_knots[k]);
    g.knots[k] = reinterpret_cast<const double*>(d) + o;
    o += grid->n_knots[k];
  }
  std::memcpy(hd + o, grid->values, sizeof(double) * nv);
  g.values = reinterpret_cast<const double*>(d) + o;
  o += nv;
  std::memcpy(hd + o, coords, sizeof(double) * n * grid->rank);
  const double* dcoords = reinterpret_cast<const double*>(d) + o;
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, in_doubles * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  double* dout = reinterpret_cast<double*>(d + in_doubles * sizeof(double));
  uint32_t* dcl = reinterpret_cast<uint32_t*>(d + in_doubles * sizeof(double) + n * sizeof(double));
  interp_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(g, dcoords, n, dout, dcl);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(out, dout, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  if (clamp_events)
    BS_CUDA_TRY(ctx, cudaMemcpyAsync(clamp_events, dcl, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return BS_OK;
}

}  // extern "C"
