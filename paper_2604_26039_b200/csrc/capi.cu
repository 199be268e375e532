// extern "C" boundary of libramp_b200.so (declared in include/ramp_b200.h).
// Argument validation mirrors the reference's ValueError checks; every entry
// point is stream-ordered and returns a status code instead of throwing.
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/ramp_b200.h"
#include "launch.h"
#include "route.cuh"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t err, const char* where) {
  return fail(RAMP_ECUDA, std::string(where) + ": " + cudaGetErrorString(err));
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct WorkspaceLayout {
  size_t ctrl, hist, sorted, tiles, done, acc, xs, act, acc_a, split_cnt, xq, xsf, actq, actsf, xqt, xsft, total;
  int64_t capacity, rows;
};

// Device workspace of one fused_moe call (all regions 256-byte aligned):
// route control words, histogram, aligned ids, M-tile experts, split-mode
// counters, the fp32 output accumulator, expert-sorted tokens and the
// split-mode intermediate activations.
WorkspaceLayout layout_for(int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k) {
  WorkspaceLayout w{};
  const int64_t n_assign = (int64_t)S * top_k;
  w.capacity = ramp_align_capacity(n_assign, E, ramp::kMaxBm);
  w.rows = w.capacity + 128;  // an M-tile box may read up to 128 rows past the end
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + bytes, 256);
    return at;
  };
  w.ctrl = take(64);
  w.hist = take(sizeof(int32_t) * E);
  w.sorted = take(sizeof(int32_t) * w.capacity);
  w.tiles = take(sizeof(int32_t) * w.capacity);
  w.done = take(sizeof(int32_t) * w.capacity);
  w.acc = take(sizeof(float) * (size_t)S * H);
  w.xs = take(2 * (size_t)w.rows * H);
  w.act = take(2 * (size_t)w.rows * I);
  w.acc_a = take(4 * (size_t)w.rows * 2 * I);
  // M-tiles: n_post_pad / bm <= n_assign / bm + E, bm >= 4
  const int64_t mt_max = n_assign / 4 + E + 1;
  // split-K arrival counters, one per (M-tile, stripe): stripes = I / (ttn/2) <= I / 64
  w.split_cnt = take(sizeof(int32_t) * (size_t)mt_max * (I / 64 + 1));
  w.xq = take((size_t)w.rows * H);
  w.xsf = take((size_t)mt_max * (H / 128 + 1) * 512);
  w.actq = take((size_t)w.rows * I);
  w.actsf = take((size_t)mt_max * (I / 128 + 1) * 512);
  w.xqt = take((size_t)S * H);        // FP8: tokens quantised once, [S, H] e4m3
  w.xsft = take((size_t)S * (H / 32)); //      and their scales [S, H/32]
  w.total = off;
  return w;
}

// The layout a workspace of `bytes` bytes gets for a call of S tokens: the
// regions are sized for the LARGEST token count the buffer holds, not for S,
// so one workspace reused across batch sizes keeps every region at the same
// offset and the zero-at-entry invariants of the read-and-clear regions
// (fp32 output accumulator, split-K partials and counters) carry over from
// call to call.  Returns total > bytes when even S does not fit.
WorkspaceLayout layout_in(size_t bytes, int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k) {
  WorkspaceLayout w = layout_for(S, H, I, E, top_k);
  if (w.total > bytes) return w;
  int64_t lo = S, hi = S > 0 ? S : 1;  // lo fits; grow hi until it does not
  while (hi < (int64_t(1) << 28) && layout_for((int32_t)(2 * hi), H, I, E, top_k).total <= bytes) hi *= 2;
  if (lo < hi) lo = hi;
  hi = 2 * hi;  // does not fit (or is past the cap)
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (layout_for((int32_t)mid, H, I, E, top_k).total <= bytes) lo = mid; else hi = mid;
  }
  return layout_for((int32_t)lo, H, I, E, top_k);
}

// A workspace whose layout key (geometry, size) changes between calls is
// re-zeroed first: its regions move, and the new read-and-clear regions
// would otherwise start on the old layout's data.  Tracked per buffer
// address on the host (no device round trip; stream-ordered memset, which
// is capturable).
struct WsKey {
  int32_t H, I, E, top_k;
  size_t bytes;
  bool operator==(const WsKey& o) const {
    return H == o.H && I == o.I && E == o.E && top_k == o.top_k && bytes == o.bytes;
  }
};
std::mutex g_ws_mu;
std::unordered_map<const void*, WsKey> g_ws_keys;

cudaError_t ensure_layout(void* ws, const WsKey& key, cudaStream_t st) {
  bool reset = false;
  {
    std::lock_guard<std::mutex> g(g_ws_mu);
    auto it = g_ws_keys.find(ws);
    if (it == g_ws_keys.end()) {
      if (g_ws_keys.size() > 4096) g_ws_keys.clear();
      g_ws_keys.emplace(ws, key);  // first use: the caller zero-filled it (ABI contract)
    } else if (!(it->second == key)) {
      it->second = key;
      reset = true;
    }
  }
  return reset ? cudaMemsetAsync(ws, 0, key.bytes, st) : cudaSuccess;
}

int check_table(const ramp_table_t* t) {
  if (!t) return fail(RAMP_EINVAL, "table is null");
  if (t->n_cfg < 1) return fail(RAMP_EINVAL, "dispatch table over an empty pool");
  if (t->n_ubm < 1 || t->n_ubm > ramp::kMaxUbm) return fail(RAMP_EINVAL, "n_ubm out of range [1, 128]");
  if (t->sm_count < 1) return fail(RAMP_EINVAL, "sm_count must be >= 1");
  if (t->N < 1) return fail(RAMP_EINVAL, "N must be >= 1");
  if (!t->bm || !t->ttn || !t->split_k || !t->ubm || !t->ubm_index || !t->a || !t->b || !t->c || !t->d)
    return fail(RAMP_EINVAL, "table arrays must be non-null");
  return RAMP_OK;
}

}  // namespace

extern "C" {

int ramp_version(void) { return 100; }

void ramp_set_profile_buffer(unsigned long long* dev_buf) { ramp::g_prof_buffer = dev_buf; }

const char* ramp_last_error(void) { return g_last_error.c_str(); }

int ramp_device_ok(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? 1 : 0;
}

int64_t ramp_align_capacity(int64_t n_assign, int32_t E, int32_t bm) {
  if (n_assign < 0 || E < 1 || bm < 1) return 0;
  const int64_t cap = n_assign + (int64_t)E * (bm - 1);
  return (cap + bm - 1) / bm * bm;
}

int64_t ramp_config_smem_bytes(int32_t bm, int32_t ttn, int32_t stg, int32_t mode) {
  return ramp::config_smem_bytes(bm, ttn, stg, mode, false);
}

int64_t ramp_config_smem_bytes_kps(int32_t bm, int32_t ttn, int32_t stg, int32_t mode, int32_t kps) {
  return ramp::config_smem_bytes(bm, ttn, stg, mode, false, kps);
}

int64_t ramp_config_smem_bytes_fp8(int32_t bm, int32_t ttn, int32_t stg) {
  return ramp_config_smem_bytes_fp8_kps(bm, ttn, stg, 1);
}

int64_t ramp_config_smem_bytes_fp8_kps(int32_t bm, int32_t ttn, int32_t stg, int32_t kps) {
  // accumulators below the TMEM scale-factor columns; kps 1 or 2 with at most
  // 16 scale atoms per stage
  if (bm < 4 || ttn < 256 || (ttn / 128) * ramp::bm_mma_host(bm) > ramp::kSfCol) return 0;
  if (kps != 1 && (kps != 2 || kps * (ttn / 128 + 1) > 16)) return 0;
  return ramp::config_smem_bytes(bm, ttn, stg, 1, true, kps);
}

int ramp_moe_align(const int32_t* topk_ids, int64_t n_assign, int32_t E, int32_t bm, int32_t* hist,
                   int32_t* sorted_ids, int32_t* tile_expert, int32_t* n_post_pad, void* stream) {
  if (E < 1 || E > ramp::kMaxExperts) return fail(RAMP_EINVAL, "E must be in [1, 512]");
  if (bm < 1) return fail(RAMP_EINVAL, "bm must be >= 1");
  if (n_assign < 0 || n_assign >= (int64_t(1) << 31) - (int64_t)E * bm)
    return fail(RAMP_EINVAL, "n_assign out of range");
  if (!hist || !sorted_ids || !tile_expert || !n_post_pad || (n_assign > 0 && !topk_ids))
    return fail(RAMP_EINVAL, "null buffer");
  cudaError_t err = ramp::launch_align(topk_ids, n_assign, E, bm, hist, sorted_ids, tile_expert, n_post_pad,
                                       static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "ramp_moe_align");
  return RAMP_OK;
}

int ramp_dispatch_select(const int32_t* hist, int32_t E, const ramp_table_t* table, int32_t* cfg_out,
                         int32_t* n_eval_out, int64_t* grid_out, double* pred_out, void* stream) {
  if (int rc = check_table(table)) return rc;
  if (E < 1 || E > ramp::kMaxExperts) return fail(RAMP_EINVAL, "E must be in [1, 512]");
  if (!hist || !cfg_out) return fail(RAMP_EINVAL, "null buffer");
  cudaError_t err = ramp::launch_select(hist, E, *table, cfg_out, n_eval_out, grid_out, pred_out,
                                        static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "ramp_dispatch_select");
  return RAMP_OK;
}

size_t ramp_fused_moe_workspace_size(int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k) {
  if (S < 0 || H < 1 || I < 1 || E < 1 || top_k < 1) return 0;
  return layout_for(S, H, I, E, top_k).total;
}

static int fused_impl(const void* x, const void* w1, const uint8_t* w1_sf, const void* w2, const uint8_t* w2_sf,
                      const float* topk_w, const int32_t* topk_ids, int32_t S, int32_t H, int32_t I, int32_t E,
                      int32_t top_k, const ramp_table_t* table, int32_t forced_cfg, void* out, int32_t* sel_out,
                      void* workspace, size_t workspace_bytes, int32_t phases, void* stream, bool fp8,
                      const void* logits = nullptr, int32_t logits_bf16 = 0, int32_t renorm = 0,
                      float* w_out = nullptr, const uint8_t* xsf_in = nullptr,
                      const ramp_row_strides_t* rs = nullptr) {
  if (phases < 1 || phases > 3) return fail(RAMP_EINVAL, "phases must be 1 (route), 2 (megakernel) or 3");
  if (int rc = check_table(table)) return rc;
  if (S < 0) return fail(RAMP_EINVAL, "S must be >= 0");
  if (E < 1 || E > ramp::kMaxExperts) return fail(RAMP_EINVAL, "E must be in [1, 512]");
  if (top_k < 1 || top_k > E) return fail(RAMP_EINVAL, "top_k must be in [1, E]");
  if (H < 128 || H % 128 != 0) return fail(RAMP_EINVAL, "H (d_model) must be a positive multiple of 128");
  if (I < 128 || I % 128 != 0) return fail(RAMP_EINVAL, "I (d_ff) must be a positive multiple of 128");
  if (table->N != 2 * I) return fail(RAMP_EINVAL, "table geometry N must equal 2*I");
  if (forced_cfg >= table->n_cfg) return fail(RAMP_EINVAL, "forced_cfg out of range");
  if (S > 0 && (!x || !w1 || !w2 || !topk_w || !topk_ids || !out))
    return fail(RAMP_EINVAL, "null tensor");
  for (const void* p : {x, w1, w2, (const void*)out})
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0) return fail(RAMP_EINVAL, "tensors must be 16-byte aligned");
  const WorkspaceLayout L = layout_in(workspace_bytes, S, H, I, E, top_k);
  if (!workspace || workspace_bytes < L.total) return fail(RAMP_EINVAL, "workspace too small");
  if (reinterpret_cast<uintptr_t>(workspace) % 256 != 0)
    return fail(RAMP_EINVAL, "workspace must be 256-byte aligned");
  auto* ws = static_cast<unsigned char*>(workspace);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaError_t err = ensure_layout(workspace, WsKey{H, I, E, top_k, workspace_bytes}, st); err != cudaSuccess)
    return cuda_fail(err, "workspace reset");
  if (S == 0) {
    if (sel_out) {
      cudaError_t err = cudaMemsetAsync(sel_out, 0, 4 * sizeof(int32_t), st);
      if (err != cudaSuccess) return cuda_fail(err, "ramp_fused_moe_bf16");
    }
    return RAMP_OK;
  }

  ramp::RouteArgs ra{};
  ra.topk_ids = topk_ids;
  ra.ids_stride = rs ? rs->ids_stride : 0;
  ra.n_assign = (int64_t)S * top_k;
  ra.E = E;
  ra.forced_cfg = forced_cfg;
  ra.table = *table;
  ra.ctrl = reinterpret_cast<int32_t*>(ws + L.ctrl);
  ra.hist_out = reinterpret_cast<int32_t*>(ws + L.hist);
  ra.sorted_ids = reinterpret_cast<int32_t*>(ws + L.sorted);
  ra.tile_expert = reinterpret_cast<int32_t*>(ws + L.tiles);
  ra.sel_out = sel_out;
  ra.done = reinterpret_cast<int*>(ws + L.done);
  ra.prof = ramp::g_prof_buffer ? ramp::g_prof_buffer + 148 * 32 : nullptr;
  ra.S = S;
  ra.H = H;
  ra.top_k = top_k;
  ra.pdl_early = ramp::pdl_mode() == 1;
  ra.pdl_prev = ramp::pdl_prev_enabled() ? 1 : 0;
  // FP8 from bf16 tokens, large batches: quantise each token once (all SMs
  // but a few) ahead of the route kernel (its programmatic dependent) instead
  // of re-quantising every gathered row in the megakernel's phase 0 (top_k x
  // the work).  Small batches keep the single in-megakernel pass: the extra
  // launch costs more than it saves (measured on Qwen3-30B-A3B, H = 2048:
  // +3-5 % at S*k <= 1024, -3 / -7 % at S*k = 4096 / 16384).  The in-kernel
  // pass quantises S*k rows of H elements, so the switch is on that volume:
  // DeepSeek-V3 (H = 7168) at S*k = 2048 spent 24 us in it.
  constexpr int64_t kQuantTokensMinElems = int64_t(4096) * 2048;
  // (dense tokens only: the quantisation kernel reads x as [S, H])
  const bool quant_tokens = fp8 && !xsf_in && !(rs && rs->x_stride) && (int64_t)S * top_k * H >= kQuantTokensMinElems;
  if (quant_tokens && (phases & 2)) ra.pdl_prev = 2;
  ra.logits = logits;
  ra.logits_bf16 = logits_bf16;
  ra.renorm = renorm;
  ra.w_out = w_out;
  cudaError_t err = cudaSuccess;
  if (quant_tokens && (phases & 2)) {
    err = ramp::launch_mx_quant_tokens(x, S, H, ws + L.xqt, ws + L.xsft, st);
    if (err != cudaSuccess) return cuda_fail(err, "token quantisation kernel");
  }
  if (phases & 1) {
    err = ramp::launch_route(ra, st);
    if (err != cudaSuccess) return cuda_fail(err, "route kernel");
  }
  if (!(phases & 2)) return RAMP_OK;

  ramp::MoeLaunch ml{};
  ml.x = x;
  ml.w1 = w1;
  ml.w2 = w2;
  ml.topk_w = topk_w;
  ml.ctrl = ra.ctrl;
  ml.sorted_ids = ra.sorted_ids;
  ml.tile_expert = ra.tile_expert;
  ml.out_acc = reinterpret_cast<float*>(ws + L.acc);
  ml.out = out;
  ml.x_sorted = ws + L.xs;
  ml.act_g = ws + L.act;
  ml.done = ra.done;
  ml.job_counter = ra.ctrl + 7;
  ml.rows = L.rows;
  ml.acc_a = reinterpret_cast<float*>(ws + L.acc_a);
  ml.split_cnt = reinterpret_cast<int*>(ws + L.split_cnt);
  ml.fp8 = fp8;
  ml.w1_sf = w1_sf;
  ml.w2_sf = w2_sf;
  ml.x_q = ws + L.xq;
  ml.x_sf = ws + L.xsf;
  ml.act_q = ws + L.actq;
  ml.act_sf = ws + L.actsf;
  ml.xq_in = xsf_in ? static_cast<const uint8_t*>(x) : (quant_tokens ? ws + L.xqt : nullptr);  // e4m3 rows
  ml.xsf_in = xsf_in ? xsf_in : (quant_tokens ? ws + L.xsft : nullptr);
  ml.x_stride = rs && !quant_tokens ? rs->x_stride : 0;
  ml.sf_stride = rs && xsf_in ? rs->sf_stride : 0;
  ml.w_stride = rs ? rs->w_stride : 0;
  ml.table = *table;
  ml.S = S;
  ml.H = H;
  ml.I = I;
  ml.E = E;
  ml.top_k = top_k;
  const char* why = nullptr;
  err = ramp::launch_fused_moe(ml, st, &why);
  if (err != cudaSuccess) return why ? fail(RAMP_ECUDA, why) : cuda_fail(err, "fused_moe kernel");
  return RAMP_OK;
}

int ramp_fused_moe_bf16_ex(const void* x, const void* w1, const void* w2, const float* topk_w,
                           const int32_t* topk_ids, int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k,
                           const ramp_table_t* table, int32_t forced_cfg, void* out, int32_t* sel_out,
                           void* workspace, size_t workspace_bytes, int32_t phases, void* stream) {
  return fused_impl(x, w1, nullptr, w2, nullptr, topk_w, topk_ids, S, H, I, E, top_k, table, forced_cfg, out,
                    sel_out, workspace, workspace_bytes, phases, stream, false);
}

int ramp_fused_moe_bf16(const void* x, const void* w1, const void* w2, const float* topk_w,
                        const int32_t* topk_ids, int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k,
                        const ramp_table_t* table, int32_t forced_cfg, void* out, int32_t* sel_out,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return ramp_fused_moe_bf16_ex(x, w1, w2, topk_w, topk_ids, S, H, I, E, top_k, table, forced_cfg, out, sel_out,
                                workspace, workspace_bytes, 3, stream);
}

int ramp_fused_moe_gating_bf16(const void* x, const void* w1, const void* w2, const void* router_logits,
                               int32_t logits_bf16, int32_t renormalize, float* topk_w_out, int32_t* topk_ids_out,
                               int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k, const ramp_table_t* table,
                               int32_t forced_cfg, void* out, int32_t* sel_out, void* workspace,
                               size_t workspace_bytes, void* stream) {
  if (top_k < 1 || top_k > ramp::kMaxTopK) return fail(RAMP_EINVAL, "router fusion needs 1 <= top_k <= 32");
  if ((int64_t)S * top_k > ramp::kIdCache)
    return fail(RAMP_EINVAL, "router fusion needs S * top_k <= 16384 (the ids stay in shared memory)");
  if (S > 0 && (!router_logits || !topk_w_out || !topk_ids_out)) return fail(RAMP_EINVAL, "null router buffer");
  return fused_impl(x, w1, nullptr, w2, nullptr, topk_w_out, topk_ids_out, S, H, I, E, top_k, table, forced_cfg, out,
                    sel_out, workspace, workspace_bytes, 3, stream, false, router_logits, logits_bf16, renormalize,
                    topk_w_out);
}

int ramp_fused_moe_fp8(const void* x, const void* w1_q, const uint8_t* w1_sf, const void* w2_q,
                       const uint8_t* w2_sf, const float* topk_w, const int32_t* topk_ids, int32_t S, int32_t H,
                       int32_t I, int32_t E, int32_t top_k, const ramp_table_t* table, int32_t forced_cfg, void* out,
                       int32_t* sel_out, void* workspace, size_t workspace_bytes, int32_t phases, void* stream) {
  if (S > 0 && (!w1_sf || !w2_sf)) return fail(RAMP_EINVAL, "null scale-factor tensor");
  if (I % 256 != 0) return fail(RAMP_EINVAL, "FP8 path needs d_ff a multiple of 256");
  return fused_impl(x, w1_q, w1_sf, w2_q, w2_sf, topk_w, topk_ids, S, H, I, E, top_k, table, forced_cfg, out,
                    sel_out, workspace, workspace_bytes, phases, stream, true);
}

int ramp_fused_moe_fp8_prequant(const uint8_t* x_q, const uint8_t* x_sf, const void* w1_q, const uint8_t* w1_sf,
                                const void* w2_q, const uint8_t* w2_sf, const float* topk_w, const int32_t* topk_ids,
                                int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k, const ramp_table_t* table,
                                int32_t forced_cfg, void* out, int32_t* sel_out, void* workspace,
                                size_t workspace_bytes, int32_t phases, void* stream) {
  if (S > 0 && (!w1_sf || !w2_sf || !x_sf)) return fail(RAMP_EINVAL, "null scale-factor tensor");
  if (reinterpret_cast<uintptr_t>(x_sf) % 4 != 0) return fail(RAMP_EINVAL, "x_sf must be 4-byte aligned");
  if (I % 256 != 0) return fail(RAMP_EINVAL, "FP8 path needs d_ff a multiple of 256");
  return fused_impl(x_q, w1_q, w1_sf, w2_q, w2_sf, topk_w, topk_ids, S, H, I, E, top_k, table, forced_cfg, out,
                    sel_out, workspace, workspace_bytes, phases, stream, true, nullptr, 0, 0, nullptr, x_sf);
}

int ramp_fused_moe_strided(const void* x, const uint8_t* x_sf, const void* w1, const uint8_t* w1_sf, const void* w2,
                           const uint8_t* w2_sf, const float* topk_w, const int32_t* topk_ids,
                           const ramp_row_strides_t* strides, int32_t S, int32_t H, int32_t I, int32_t E,
                           int32_t top_k, const ramp_table_t* table, int32_t forced_cfg, void* out, int32_t* sel_out,
                           void* workspace, size_t workspace_bytes, int32_t phases, void* stream) {
  const bool fp8 = w1_sf != nullptr;
  ramp_row_strides_t rs{};
  if (strides) rs = *strides;
  const int64_t x_bytes = (fp8 && x_sf) ? H : 2 * (int64_t)H;
  if (rs.x_stride < 0 || rs.sf_stride < 0 || rs.ids_stride < 0 || rs.w_stride < 0)
    return fail(RAMP_EINVAL, "strides must be >= 0");
  if (rs.x_stride && (rs.x_stride < x_bytes || rs.x_stride % 16 != 0))
    return fail(RAMP_EINVAL, "x_stride must be >= the row's bytes and a multiple of 16");
  if (rs.sf_stride && (!x_sf || rs.sf_stride < H / 32 || rs.sf_stride % 4 != 0))
    return fail(RAMP_EINVAL, "sf_stride needs x_sf, >= H/32 and a multiple of 4");
  if ((rs.ids_stride && rs.ids_stride < top_k) || (rs.w_stride && rs.w_stride < top_k))
    return fail(RAMP_EINVAL, "ids_stride / w_stride must be >= top_k");
  if (rs.ids_stride == top_k) rs.ids_stride = 0;
  if (rs.w_stride == top_k) rs.w_stride = 0;
  if (rs.x_stride == x_bytes) rs.x_stride = 0;
  if (rs.sf_stride == H / 32) rs.sf_stride = 0;
  if (fp8) {
    if (S > 0 && !w2_sf) return fail(RAMP_EINVAL, "null scale-factor tensor");
    if (x_sf && reinterpret_cast<uintptr_t>(x_sf) % 4 != 0) return fail(RAMP_EINVAL, "x_sf must be 4-byte aligned");
    if (I % 256 != 0) return fail(RAMP_EINVAL, "FP8 path needs d_ff a multiple of 256");
  } else if (x_sf || w2_sf) {
    return fail(RAMP_EINVAL, "x_sf / w2_sf given without w1_sf (BF16 layer)");
  }
  return fused_impl(x, w1, w1_sf, w2, w2_sf, topk_w, topk_ids, S, H, I, E, top_k, table, forced_cfg, out, sel_out,
                    workspace, workspace_bytes, phases, stream, fp8, nullptr, 0, 0, nullptr, x_sf, &rs);
}

// ------------------------------------------------------------ expert parallelism
struct ramp_ep_comm {
  void* nccl;
  int32_t world, rank;
};

static int ep_check(const void* x, const int32_t* topk_ids, const float* topk_w, int32_t S, int32_t H, int32_t E,
                    int32_t top_k, int32_t world, int32_t cap, int32_t wire) {
  if (world < 1 || world > 32) return fail(RAMP_EINVAL, "world must be in [1, 32]");
  if (E < 1 || E % world != 0) return fail(RAMP_EINVAL, "E must be a positive multiple of world");
  if (S < 0 || cap < 0) return fail(RAMP_EINVAL, "S and cap must be >= 0");
  if (top_k < 1 || top_k > E) return fail(RAMP_EINVAL, "top_k must be in [1, E]");
  if (H < 128 || H % 128 != 0) return fail(RAMP_EINVAL, "H (d_model) must be a positive multiple of 128");
  if (wire != RAMP_EP_WIRE_BF16 && wire != RAMP_EP_WIRE_MXFP8) return fail(RAMP_EINVAL, "unknown wire format");
  if (S > 0 && (!x || !topk_ids || !topk_w)) return fail(RAMP_EINVAL, "null tensor");
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return fail(RAMP_EINVAL, "x must be 16-byte aligned");
  return RAMP_OK;
}

int ramp_ep_row_layout(int32_t H, int32_t top_k, int32_t wire, int32_t* out4) {
  if (!out4) return fail(RAMP_EINVAL, "null output");
  if (H < 128 || H % 128 != 0) return fail(RAMP_EINVAL, "H (d_model) must be a positive multiple of 128");
  if (top_k < 1) return fail(RAMP_EINVAL, "top_k must be >= 1");
  if (wire != RAMP_EP_WIRE_BF16 && wire != RAMP_EP_WIRE_MXFP8) return fail(RAMP_EINVAL, "unknown wire format");
  ramp::ep_row_layout(H, top_k, wire == RAMP_EP_WIRE_MXFP8, out4);
  return RAMP_OK;
}

int ramp_ep_pack(const void* x, const int32_t* topk_ids, const float* topk_w, int32_t S, int32_t H, int32_t E,
                 int32_t top_k, int32_t world, int32_t cap, int32_t wire, void* send, int32_t* pos, int32_t* counts,
                 int32_t* overflow, void* stream) {
  if (int rc = ep_check(x, topk_ids, topk_w, S, H, E, top_k, world, cap, wire)) return rc;
  if ((!send && (int64_t)world * cap > 0) || (!pos && S > 0) || !counts || !overflow)
    return fail(RAMP_EINVAL, "null send buffer");
  if (reinterpret_cast<uintptr_t>(send) % 16 != 0) return fail(RAMP_EINVAL, "send must be 16-byte aligned");
  int32_t lay[4];
  ramp::ep_row_layout(H, top_k, wire == RAMP_EP_WIRE_MXFP8, lay);
  ramp::EpPackArgs a{topk_ids, topk_w, x, S, H, top_k, E, world, cap, static_cast<uint8_t*>(send),
                     lay[0], lay[1], lay[2], lay[3], pos, counts, overflow};
  cudaError_t err = ramp::launch_ep_pack(a, wire == RAMP_EP_WIRE_MXFP8, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "ramp_ep_pack");
  return RAMP_OK;
}

int ramp_ep_reduce(const void* back, const int32_t* pos, int32_t S, int32_t H, int32_t world, int32_t cap,
                   void* out, void* stream) {
  if (world < 1 || world > 32 || S < 0 || cap < 0 || H < 128 || H % 128 != 0)
    return fail(RAMP_EINVAL, "bad geometry");
  if (S > 0 && (!back || !pos || !out)) return fail(RAMP_EINVAL, "null tensor");
  if (reinterpret_cast<uintptr_t>(back) % 16 != 0 || reinterpret_cast<uintptr_t>(out) % 16 != 0)
    return fail(RAMP_EINVAL, "tensors must be 16-byte aligned");
  cudaError_t err = ramp::launch_ep_combine(back, pos, S, H, world, cap, out, static_cast<cudaStream_t>(stream));
  if (err != cudaSuccess) return cuda_fail(err, "ramp_ep_reduce");
  return RAMP_OK;
}

int ramp_ep_get_unique_id(unsigned char* out128) {
  if (!out128) return fail(RAMP_EINVAL, "null id buffer");
  const char* why = nullptr;
  if (ramp::nccl_unique_id(out128, &why) != 0) return fail(RAMP_ECUDA, std::string("NCCL: ") + (why ? why : "?"));
  return RAMP_OK;
}

int ramp_ep_comm_init(ramp_ep_comm** comm, const unsigned char* id128, int32_t world, int32_t rank) {
  if (!comm || !id128) return fail(RAMP_EINVAL, "null argument");
  if (world < 1 || world > 32 || rank < 0 || rank >= world) return fail(RAMP_EINVAL, "bad world / rank");
  const char* why = nullptr;
  void* c = ramp::nccl_comm_init(id128, world, rank, &why);
  if (!c) return fail(RAMP_ECUDA, std::string("ncclCommInitRank: ") + (why ? why : "?"));
  *comm = new ramp_ep_comm{c, world, rank};
  return RAMP_OK;
}

int ramp_ep_comm_destroy(ramp_ep_comm* comm) {
  if (!comm) return RAMP_OK;
  ramp::nccl_comm_destroy(comm->nccl);
  delete comm;
  return RAMP_OK;
}

int ramp_ep_dispatch(ramp_ep_comm* comm, const void* x, const int32_t* topk_ids, const float* topk_w, int32_t S,
                     int32_t H, int32_t E, int32_t top_k, int32_t cap, int32_t wire, void* send, int32_t* pos,
                     int32_t* counts, int32_t* overflow, void* recv, void* stream) {
  if (!comm) return fail(RAMP_EINVAL, "null communicator");
  if (!recv) return fail(RAMP_EINVAL, "null receive buffer");
  const int32_t P = comm->world;
  if (int rc = ramp_ep_pack(x, topk_ids, topk_w, S, H, E, top_k, P, cap, wire, send, pos, counts, overflow, stream))
    return rc;
  int32_t lay[4];
  ramp::ep_row_layout(H, top_k, wire == RAMP_EP_WIRE_MXFP8, lay);
  const void* snd[1] = {send};
  void* rcv[1] = {recv};
  const size_t bytes[1] = {(size_t)cap * lay[3]};
  const char* why = nullptr;
  if (ramp::nccl_all_to_all(comm->nccl, P, snd, rcv, bytes, 1, static_cast<cudaStream_t>(stream), &why))
    return fail(RAMP_ECUDA, std::string("NCCL dispatch: ") + (why ? why : "?"));
  return RAMP_OK;
}

int ramp_ep_combine(ramp_ep_comm* comm, const void* partial, void* back, const int32_t* pos, int32_t S, int32_t H,
                    int32_t cap, void* out, void* stream) {
  if (!comm) return fail(RAMP_EINVAL, "null communicator");
  if (!partial || !back) return fail(RAMP_EINVAL, "null buffer");
  const void* snd[1] = {partial};
  void* rcv[1] = {back};
  const size_t bytes[1] = {(size_t)cap * H * 2};
  const char* why = nullptr;
  if (ramp::nccl_all_to_all(comm->nccl, comm->world, snd, rcv, bytes, 1, static_cast<cudaStream_t>(stream), &why))
    return fail(RAMP_ECUDA, std::string("NCCL combine: ") + (why ? why : "?"));
  return ramp_ep_reduce(back, pos, S, H, comm->world, cap, out, stream);
}

}  // extern "C"
