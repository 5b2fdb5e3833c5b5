// bs_decode.cu — decode slack-aware frequency pick on sm_100a:
// select_decode_freq_ex (dvfs.hpp:274-293), one warp per query.  Lane j
// evaluates rung j (in 32-rung chunks, ascending) and a ballot finds the
// first rung with L_dec * (1 + margin) <= tbt -- the rung the reference's
// ascending walk stops at; eval_count is that rung's 1-based position.
#include <cstring>

#include "bs_internal.h"

using namespace bs;

namespace {

struct DDecodeCfg {
  double tbt;
  double kv_threshold;
  double one_plus_margin;
  int n_ladder;
  int ladder_off;
};

struct DDecodeQuery {
  long long n_requests;
  long long sum_len;
  long long cap;
  long long used;
  int tp;
  int cfg;
};

struct DDecodeOut {
  double freq;
  long long eval_count;
  int kv_override;
  int status;
};

__global__ void decode_kernel(DGrid lat, const DDecodeCfg* cfgs, const double* ladders, const DDecodeQuery* qs,
                              DDecodeOut* out, int n) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n) return;
  const DDecodeQuery q = qs[warp];
  const DDecodeCfg c = cfgs[q.cfg];
  const double* L = ladders + c.ladder_off;
  DDecodeOut o;
  o.freq = L[c.n_ladder - 1];
  o.eval_count = 0;
  o.kv_override = 0;
  o.status = BS_OK;
  // KVCacheState::utilization (controller.hpp:21-23)
  const double util = q.cap > 0 ? __ddiv_rn(static_cast<double>(q.used), static_cast<double>(q.cap)) : 0.0;
  if (util > c.kv_threshold) {
    o.kv_override = 1;
  } else if (lat.bad_axis) {
    o.eval_count = 1;
    o.status = BS_MODEL_ERROR;
  } else {
    const Query base = make_query(q.n_requests, q.sum_len, q.tp, 0.0);
    bool done = false;
    for (int j0 = 0; j0 < c.n_ladder && !done; j0 += 32) {
      const int j = j0 + lane;
      bool fits = false, bad = false;
      if (j < c.n_ladder) {
        Query qq = base;
        qq.c[BS_AXIS_FREQ] = L[j];
        const double v = interp(lat, qq, nullptr);
        bad = !model_value_ok(v);
        fits = !bad && __dmul_rn(v, c.one_plus_margin) <= c.tbt;  // dvfs.hpp:285-286
      }
      // the reference stops at the first rung that fits or throws
      const unsigned stop = __ballot_sync(0xffffffffu, fits || bad);
      if (stop) {
        const int first = __ffs(stop) - 1;
        const int rung = j0 + first;
        o.eval_count = rung + 1;
        const unsigned badm = __ballot_sync(0xffffffffu, bad);
        if ((badm >> first) & 1u) {
          o.status = BS_MODEL_ERROR;
        } else {
          o.freq = L[rung];
        }
        done = true;
      }
    }
    if (!done) o.eval_count = c.n_ladder;  // dvfs.hpp:291
  }
  if (lane == 0) out[warp] = o;
}

}  // namespace

extern "C" int bs_decode_pick(bs_ctx_t ctx, bs_models_t models, const bs_decode_config* cfgs, int n_cfgs,
                              const bs_decode_query* queries, int n, bs_decode_result* out) {
  if (!ctx || !models) return set_error(ctx, BS_PARAMETER_ERROR, "bs_decode_pick: null context or models");
  if (n_cfgs < 1 || !cfgs) return set_error(ctx, BS_PARAMETER_ERROR, "decode: no policy configuration");
  if (n <= 0) return BS_OK;
  // DecodePolicyConfig::validate (dvfs.hpp:42-47), once per configuration.
  size_t n_rungs = 0;
  for (int c = 0; c < n_cfgs; ++c) {
    const bs_decode_config& dc = cfgs[c];
    if (dc.tbt_slo_ms <= 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "decode policy: tbt_slo_ms must be > 0");
    if (dc.kv_threshold <= 0.0 || dc.kv_threshold >= 1.0)
      return set_error(ctx, BS_PARAMETER_ERROR, "decode policy: kv_threshold in (0,1)");
    if (dc.n_ladder < 1 || !dc.ladder_mhz) return set_error(ctx, BS_PARAMETER_ERROR, "frequency ladder: empty");
    double prev = 0.0;
    for (int j = 0; j < dc.n_ladder; ++j) {
      if (dc.ladder_mhz[j] <= prev)
        return set_error(ctx, BS_PARAMETER_ERROR, "frequency ladder: must be strictly increasing and > 0");
      prev = dc.ladder_mhz[j];
    }
    if (dc.margin < 0.0) return set_error(ctx, BS_PARAMETER_ERROR, "decode policy: margin must be >= 0");
    n_rungs += static_cast<size_t>(dc.n_ladder);
  }
  const size_t o_cfg = 0;
  const size_t o_lad = (sizeof(DDecodeCfg) * n_cfgs + 255) / 256 * 256;
  const size_t o_q = o_lad + (8 * n_rungs + 255) / 256 * 256;
  const size_t o_out = o_q + (sizeof(DDecodeQuery) * n + 255) / 256 * 256;
  const size_t total = o_out + sizeof(DDecodeOut) * n;
  char* h = static_cast<char*>(ctx->host_buf(kSlotMisc, total));
  char* d = static_cast<char*>(ctx->dev_buf(kSlotMisc, total));
  if (!h || !d) return set_error(ctx, BS_CUDA_ERROR, "decode: allocation failed");
  DDecodeCfg* hc = reinterpret_cast<DDecodeCfg*>(h + o_cfg);
  double* hl = reinterpret_cast<double*>(h + o_lad);
  int lo = 0;
  for (int c = 0; c < n_cfgs; ++c) {
    hc[c].tbt = cfgs[c].tbt_slo_ms;
    hc[c].kv_threshold = cfgs[c].kv_threshold;
    hc[c].one_plus_margin = 1.0 + cfgs[c].margin;
    hc[c].n_ladder = cfgs[c].n_ladder;
    hc[c].ladder_off = lo;
    std::memcpy(hl + lo, cfgs[c].ladder_mhz, sizeof(double) * cfgs[c].n_ladder);
    lo += cfgs[c].n_ladder;
  }
  DDecodeQuery* hq = reinterpret_cast<DDecodeQuery*>(h + o_q);
  for (int i = 0; i < n; ++i) {
    if (queries[i].cfg_index < 0 || queries[i].cfg_index >= n_cfgs)
      return set_error(ctx, BS_PARAMETER_ERROR, "decode: query %d cfg_index out of range", i);
    hq[i].n_requests = queries[i].batch.n_requests;
    hq[i].sum_len = queries[i].batch.sum_len;
    hq[i].cap = queries[i].kv_capacity_tokens;
    hq[i].used = queries[i].kv_used_tokens;
    hq[i].tp = queries[i].tp;
    hq[i].cfg = queries[i].cfg_index;
  }
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(d, h, o_out, cudaMemcpyHostToDevice, ctx->stream));
  const int threads = 256;
  const long long blocks = (static_cast<long long>(n) * 32 + threads - 1) / threads;
  decode_kernel<<<static_cast<unsigned>(blocks), threads, 0, ctx->stream>>>(
      models->dm.grid[1], reinterpret_cast<const DDecodeCfg*>(d + o_cfg), reinterpret_cast<const double*>(d + o_lad),
      reinterpret_cast<const DDecodeQuery*>(d + o_q), reinterpret_cast<DDecodeOut*>(d + o_out), n);
  BS_LAUNCH_CHECK(ctx);
  BS_CUDA_TRY(ctx, cudaMemcpyAsync(h + o_out, d + o_out, sizeof(DDecodeOut) * n, cudaMemcpyDeviceToHost, ctx->stream));
  BS_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  const DDecodeOut* ho = reinterpret_cast<const DDecodeOut*>(h + o_out);
  int first_err = -1;
  for (int i = 0; i < n; ++i) {
    out[i].freq_mhz = ho[i].freq;
    out[i].eval_count = ho[i].eval_count;
    out[i].kv_override = ho[i].kv_override;
    out[i].status = ho[i].status;
    if (ho[i].status != BS_OK && first_err < 0) first_err = i;
  }
  if (first_err >= 0) return set_error(ctx, BS_MODEL_ERROR, "latency model returned non-positive value");
  return BS_OK;
}
