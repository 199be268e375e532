// Route stage of the hot path: expert histogram -> routing-aware dispatcher ->
// moe_align_block_size, all inside ONE thread block so the whole control plane
// is a single launch with no host round trip (the paper's "single fused
// dispatch kernel", here also emitting the
// alignment the megakernel consumes).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <math_constants.h>

#include "../../include/ramp_b200.h"

namespace ramp {

// Development probe (-DRAMP_ROUTE_CLOCKS): thread 0 records clock64() at the
// numbered points of the route block into prof[16 + k].
#ifdef RAMP_ROUTE_CLOCKS
__shared__ unsigned long long* g_rclk;  // shared: a global pointer load would stall each probe
#define RCLK(k)                                                          \
  do {                                                                   \
    if (threadIdx.x == 0 && g_rclk) g_rclk[k] = clock64();               \
  } while (0)
#else
#define RCLK(k) \
  do {          \
  } while (0)
#endif

constexpr int kRouteThreads = 1024;
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kMaxExperts = 512;
constexpr int kMaxUbm = 128;
constexpr int kIdCache = 16384;  // topk ids kept in shared memory between the two passes
constexpr int kStageMax = 20480; // sorted ids staged in shared memory, then copied out coalesced
constexpr int kAlignMaxBm = 128;
constexpr int kCfgStageMax = 1024;      // configs whose static fields are staged in shared memory
constexpr size_t kRouteSmemLimit = 220 * 1024;

// Dynamic shared memory layout of the route block (sized by E and n).
//   hist[E]       bincount
//   off[E+1]      exclusive scan of the padded counts
//   cnt[E][32]    per-(expert, warp) counts, then exclusive prefixes over warps
//   ids[min(n, kIdCache)]
//   stage[stage_cap]  sorted ids built here (scattered shared stores), then
//                     written to global memory with coalesced 16-byte stores
struct RouteSmem {
  int32_t* hist;
  int32_t* off;
  int32_t* cnt;
  int32_t* ids;
  int32_t* stage;
  int stage_cap;
  bool cached;
  // dispatch table staged by cp.async at kernel entry (null: read from global)
  double *ca, *cb, *cc, *cd, *clam;
  int32_t *csk, *cubm_idx, *ctiles, *cubm;
  int ubm_stride;  // cubm[u] was staged by lane 0 of warp u % ubm_stride (0: not staged)
};

__host__ __device__ inline int route_stage_cap(int E, int64_t n) {
  const int64_t want = n + (int64_t)E * (kAlignMaxBm - 1);
  return static_cast<int>(want < kStageMax ? want : kStageMax);
}

__host__ __device__ inline size_t route_smem_base(int E, int64_t n) {
  const int64_t cache = n <= kIdCache ? n : 0;
  return sizeof(int32_t) * ((size_t)E * 34 + 1 + (size_t)cache + 4 + (size_t)route_stage_cap(E, n)) + 64;
}
__host__ __device__ inline size_t cfg_stage_bytes(int n_cfg) {
  return (size_t)n_cfg * (5 * 8 + 3 * 4) + kMaxUbm * 4 + 16;
}
// Stage the table in shared memory when it is small enough and fits.
__host__ __device__ inline bool route_cfg_staged(int E, int64_t n, int n_cfg) {
  return n_cfg > 0 && n_cfg <= kCfgStageMax && route_smem_base(E, n) + cfg_stage_bytes(n_cfg) <= kRouteSmemLimit;
}
__host__ __device__ inline size_t route_smem_bytes(int E, int64_t n, int n_cfg = 0) {
  return route_smem_base(E, n) + (route_cfg_staged(E, n, n_cfg) ? cfg_stage_bytes(n_cfg) : 0);
}

__device__ inline RouteSmem carve_route_smem(unsigned char* base, int E, int64_t n, int n_cfg = 0) {
  RouteSmem s;
  s.hist = reinterpret_cast<int32_t*>(base);
  s.off = s.hist + E;
  s.cnt = s.off + E + 1;
  // 16-byte aligned: filled with cp.async 16-byte copies (the byte budget's
  // 64-byte tail covers this and the stage's alignment)
  s.ids = reinterpret_cast<int32_t*>((reinterpret_cast<uintptr_t>(s.cnt + 32 * E) + 15) & ~static_cast<uintptr_t>(15));
  s.cached = n <= kIdCache;
  const uintptr_t st = reinterpret_cast<uintptr_t>(s.ids + (s.cached ? n : 0));
  s.stage = reinterpret_cast<int32_t*>((st + 15) & ~static_cast<uintptr_t>(15));
  s.stage_cap = route_stage_cap(E, n);
  s.ca = s.cb = s.cc = s.cd = s.clam = nullptr;
  s.csk = s.cubm_idx = s.ctiles = s.cubm = nullptr;
  s.ubm_stride = 0;
  if (route_cfg_staged(E, n, n_cfg)) {
    const uintptr_t c0 = (reinterpret_cast<uintptr_t>(s.stage + s.stage_cap) + 15) & ~static_cast<uintptr_t>(15);
    s.ca = reinterpret_cast<double*>(c0);
    s.cb = s.ca + n_cfg;
    s.cc = s.cb + n_cfg;
    s.cd = s.cc + n_cfg;
    s.clam = s.cd + n_cfg;
    s.csk = reinterpret_cast<int32_t*>(s.clam + n_cfg);
    s.cubm_idx = s.csk + n_cfg;
    s.ctiles = s.cubm_idx + n_cfg;
    s.cubm = s.ctiles + n_cfg;
  }
  return s;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
// x / d for x >= 0, d > 0: a shift when d is a power of two (every bm of the
// B200 pools), else the integer division (the reference pools' even bm).
// The route block runs one cold pass: a 30-instruction division chain per
// expert and bm is latency on the critical path.
__device__ __forceinline__ int div_pos(int x, int d) {
  return (d & (d - 1)) == 0 ? (x >> (__ffs(d) - 1)) : x / d;
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// with an L2 eviction-priority hint (the dispatch table is re-read every
// layer call while the megakernel streams gigabytes of evict-first weights)
__device__ __forceinline__ void cp_async4_hint(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8_hint(void* dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "l"(pol)
               : "memory");
}

// Kernel entry: thread i copies config i's static fields (and lane 0 of warp
// u % ubm_stride the distinct bm value u -- the warp that reads it in
// block_dispatch's M-tile loop, so no block barrier is needed before that
// read) into shared memory asynchronously -- no registers stay live, and the
// global latency overlaps the histogram pass.  The lines are marked
// evict-last in L2 so the next layer call finds them there.
__device__ inline void stage_table(const ramp_table_t& t, RouteSmem& s, int ubm_stride) {
  if (!s.ca) return;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const int i = threadIdx.x;
  if (i < t.n_cfg) {
    cp_async8_hint(s.ca + i, t.a + i, pol);
    cp_async8_hint(s.cb + i, t.b + i, pol);
    cp_async8_hint(s.cc + i, t.c + i, pol);
    cp_async8_hint(s.cd + i, t.d + i, pol);
    if (t.lam) cp_async8_hint(s.clam + i, t.lam + i, pol);
    cp_async4_hint(s.csk + i, t.split_k + i, pol);
    cp_async4_hint(s.cubm_idx + i, t.ubm_index + i, pol);
    cp_async4_hint(s.ctiles + i, t.ntile ? t.ntile + i : t.ttn + i, pol);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
#pragma unroll 1
    for (int u = w; w < ubm_stride && u < t.n_ubm; u += ubm_stride) cp_async4_hint(s.cubm + u, t.ubm + u, pol);
  s.ubm_stride = ubm_stride;
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Lanes of the warp holding the same value e (e < 0 marks an empty lane):
// __match_any_sync rebuilt from one ballot per bit of e, which is much
// cheaper than MATCH.ANY when the warp holds many distinct experts.
// Lanes of the warp holding the same expert id (all -1 lanes together):
// one match.any instead of a ballot per id bit (the rank walk: 8.4K -> 6.6K
// cycles at n = 4096, 30K -> 17K at n = 16384, scripts/route_clocks.py).
__device__ __forceinline__ unsigned match_peers(int e, int /*nbits*/) {
  return __match_any_sync(0xffffffffu, e);
}

__host__ __device__ inline int bits_for(int E) {
  int b = 0;
  while ((1 << b) < E) ++b;
  return b;
}

// --------------------------------------------------------------- router
// Router fusion: softmax top-k of the router logits, one
// warp per token.  Lane l holds experts l, l+32, ...; the k picks are k
// rounds of a warp arg-max (higher probability first, ties to the lower
// expert id); weights are the softmax probabilities (fp32, expf), divided by
// their sum over the picks when `renorm` (vLLM's fused_topk semantics).  The
// ids land in shared memory (the histogram pass reads them there) and, with
// the weights, in global memory for the megakernel and the caller.
constexpr int kMaxTopK = 32;
__device__ inline void block_topk(const void* __restrict__ logits, bool bf16, int S, int E, int k, bool renorm,
                                  int32_t* ids_smem, int32_t* __restrict__ ids_out, float* __restrict__ w_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int per = (E + 31) >> 5;  // <= 16 for E <= 512
  for (int t = warp; t < S; t += nwarps) {
    float v[kMaxExperts / 32];
    float mx = -CUDART_INF_F;
#pragma unroll
    for (int j = 0; j < kMaxExperts / 32; ++j) {
      v[j] = -CUDART_INF_F;
      const int e = lane + 32 * j;
      if (j < per && e < E) {
        const size_t at = static_cast<size_t>(t) * E + e;
        v[j] = bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(logits)[at])
                    : reinterpret_cast<const float*>(logits)[at];
        mx = fmaxf(mx, v[j]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxExperts / 32; ++j)
      if (j < per && lane + 32 * j < E) sum += expf(v[j] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    unsigned taken = 0;
    float mine = 0.f, picked = 0.f;
    for (int r = 0; r < k; ++r) {
      float bv = -CUDART_INF_F;
      int be = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < kMaxExperts / 32; ++j) {
        const int e = lane + 32 * j;
        if (j < per && e < E && !((taken >> j) & 1) && (v[j] > bv || (v[j] == bv && e < be))) {
          bv = v[j];
          be = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (ov > bv || (ov == bv && oe < be)) {
          bv = ov;
          be = oe;
        }
      }
      if ((be & 31) == lane) taken |= 1u << (be >> 5);
      const float pr = expf(bv - mx) / sum;
      picked += pr;
      if (lane == r) mine = pr;
      if (lane == 0) {
        ids_smem[t * k + r] = be;
        ids_out[t * k + r] = be;
      }
    }
    if (lane < k) w_out[t * k + lane] = renorm ? mine / picked : mine;
  }
}

// --------------------------------------------------------------- histogram
// Pass 1 of the stable counting sort.  The n flat assignments are cut into 32
// contiguous segments, one per warp; each warp counts its segment per expert
// (warp-aggregated with match.any, no atomics: the warp owns column w of
// cnt), then one warp scan per expert turns the 32 counts into exclusive
// prefixes and the total, i.e. bincount(topk_ids, minlength=E).
// Ids outside [0, E) set *bad (ExpertHistogram rejects them, ramp/routing.py:45-50),
// except -1: a slot whose expert lives on another rank (vLLM's expert-parallel
// convention) -- skipped, it is neither counted nor aligned.
// Assignment i of a row-strided id source (ids_stride > 0: token t's top_k ids
// start at ids + t * ids_stride, e.g. the rows of an expert-parallel message;
// 0: dense [S, top_k]).
__device__ __forceinline__ int32_t ld_id(const int32_t* __restrict__ ids, int64_t i, int k, int64_t stride) {
  return stride == 0 ? __ldg(ids + i) : __ldg(ids + (i / k) * stride + i % k);
}

__device__ inline void block_count(const int32_t* __restrict__ ids, int64_t n, int E, RouteSmem& s,
                                   int* bad, bool ids_in_smem = false, int ids_k = 1, int64_t ids_stride = 0) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (s.cached && !ids_in_smem) {
    // asynchronous 16-byte copies: every thread's loads are in flight at
    // once (the synchronous loop exposed one L2 round trip per 1024 ids)
    const bool al = (reinterpret_cast<uintptr_t>(ids) & 15) == 0 && (reinterpret_cast<uintptr_t>(s.ids) & 15) == 0;
    if (ids_stride == 0 && al && (n & 3) == 0) {
      for (int64_t q = tid; q < n / 4; q += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(
                         __cvta_generic_to_shared(s.ids + 4 * q))),
                     "l"(ids + 4 * q)
                     : "memory");
    } else if (ids_stride != 0 && al && (ids_k & 3) == 0 && (ids_stride & 3) == 0) {
      // row-strided: each token's k ids are k/4 aligned 16-byte chunks
      const int per = ids_k >> 2;
      for (int q = tid; q < static_cast<int>(n / 4); q += blockDim.x) {  // n <= kIdCache here
        const int t = q / per, c = q - t * per;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(
                         __cvta_generic_to_shared(s.ids + 4 * q))),
                     "l"(ids + static_cast<int64_t>(t) * ids_stride + 4 * c)
                     : "memory");
      }
    } else {
      for (int64_t i = tid; i < n; i += blockDim.x) s.ids[i] = ld_id(ids, i, ids_k, ids_stride);
    }
  }
  for (int x = tid; x < 32 * E; x += blockDim.x) s.cnt[x] = 0;
  asm volatile("cp.async.wait_all;" ::: "memory");
  RCLK(1);
  __syncthreads();
  RCLK(2);
  const int64_t seg = (n + kRouteWarps - 1) / kRouteWarps;
  const int64_t lo = warp * seg, hi = lo + seg < n ? lo + seg : n;
  for (int64_t c0 = lo; c0 < hi; c0 += 32) {
    const int64_t i = c0 + lane;
    int e = -1;
    if (i < hi) {
      e = s.cached ? s.ids[i] : ld_id(ids, i, ids_k, ids_stride);
      if (e != -1 && (e < 0 || e >= E)) {
        *bad = 1;
        e = -1;
      }
    }
    // (shared atomics: measured faster here than a match.any-aggregated add)
    if (e >= 0) atomicAdd(s.cnt + e * 32 + warp, 1);  // counts commute: no ordering needed here
  }
  RCLK(3);
  __syncthreads();
  RCLK(4);
  for (int x = warp; x < E; x += kRouteWarps) {
    const int v = s.cnt[x * 32 + lane];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    s.cnt[x * 32 + lane] = incl - v;
    if (lane == 31) s.hist[x] = incl;
  }
  RCLK(5);
  __syncthreads();
  RCLK(6);
}

// --------------------------------------------------------------- dispatcher
struct ArgMin {
  double v;
  int i;
};

// np.argmin order: NaN is the minimum, then ties break to the lowest index.
__device__ inline bool argmin_better(const ArgMin& x, const ArgMin& y) {
  const bool xn = isnan(x.v), yn = isnan(y.v);
  if (xn != yn) return xn;
  if (!xn && x.v != y.v) return x.v < y.v;
  return x.i < y.i;
}

// Warp-wide argmin_better over (v, i) with three redux.sync.min on 32-bit
// words instead of five shuffle rounds: v maps to an order-preserving u64 key
// (NaN -> 0, the minimum, as in np.argmin; -0.0 == +0.0 as in the compare
// above), then the lowest index among the lanes holding the minimum key wins.
__device__ __forceinline__ unsigned long long argmin_key(double v) {
  if (isnan(v)) return 0ull;
  if (v == 0.0) v = 0.0;
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ ArgMin warp_argmin(const ArgMin& x) {
  const unsigned long long k = argmin_key(x.v);
  const unsigned hi = static_cast<unsigned>(k >> 32), lo = static_cast<unsigned>(k);
  const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
  const bool at_min = hi == mhi && lo == mlo;
  const unsigned mi = __reduce_min_sync(0xffffffffu, at_min ? static_cast<unsigned>(x.i) : 0xffffffffu);
  // the value is the one held by the winning lane (bit-identical to its v)
  const int src = __ffs(__ballot_sync(0xffffffffu, at_min && static_cast<unsigned>(x.i) == mi)) - 1;
  return ArgMin{__shfl_sync(0xffffffffu, x.v, src), static_cast<int>(mi)};
}

// Static fields of one config (the table is constant; only g depends on the
// routing): from the shared-memory stage when the kernel staged the table,
// else straight from global memory.
struct CfgRegs {
  long long stripes;  // work tiles per M-tile (ntile, or ceil(N/ttn))
  int sk, ubm_idx;
  double a, b, c, d, lam;
};

__device__ __forceinline__ CfgRegs load_cfg(const ramp_table_t& t, int i, const RouteSmem* s) {
  CfgRegs r;
  const bool st = s && s->ca && i < kCfgStageMax;
  r.sk = st ? s->csk[i] : __ldg(t.split_k + i);
  r.ubm_idx = st ? s->cubm_idx[i] : __ldg(t.ubm_index + i);
  const int tl = st ? s->ctiles[i] : (t.ntile ? __ldg(t.ntile + i) : __ldg(t.ttn + i));
  r.stripes = t.ntile ? tl : (static_cast<long long>(t.N) + tl - 1) / tl;
  r.a = st ? s->ca[i] : __ldg(t.a + i);
  r.b = st ? s->cb[i] : __ldg(t.b + i);
  r.c = st ? s->cc[i] : __ldg(t.c + i);
  r.d = st ? s->cd[i] : __ldg(t.d + i);
  r.lam = t.lam ? (st ? s->clam[i] : __ldg(t.lam + i)) : 0.0;
  return r;
}

// Evaluates every config of the table on the histogram in shared memory and
// returns (in every thread) the selected id.  fp64 arithmetic follows
// predict_batch exactly: ((a + b*ceil(g/sm)) + c*g) + d*log(g+1)
// (ramp/cost_model.py:104-114), gate (g/split_k)/sm < 0.2 (ramp/dispatch.py:107-114),
// first argmin over +inf-masked predictions (:118-119).  With `rs` the
// static config fields come from the kernel-entry shared-memory stage.
//
// Runs on warps [0, nwarps) of the block; with nwarps < blockDim/32 the group
// synchronises on named barrier 3 only, so the other warps can walk the
// alignment ranks meanwhile (route_kernel).  Threads outside the group must
// not call it.
__device__ __forceinline__ void group_sync(int nwarps) {
  if (nwarps * 32 == static_cast<int>(blockDim.x)) {
    __syncthreads();
  } else {
    asm volatile("bar.sync 3, %0;" ::"r"(nwarps * 32) : "memory");
  }
}

__device__ inline int block_dispatch(const int32_t* hist, int E, const ramp_table_t& t, const RouteSmem* rs,
                                     int64_t* grid_out, double* pred_out, int* n_eval_out,
                                     int64_t* mt_smem /*[kMaxUbm]*/, ArgMin* red_smem /*[32]*/,
                                     int* cnt_smem /*[32]*/, unsigned long long* stamps = nullptr,
                                     int nwarps = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (nwarps <= 0) nwarps = blockDim.x >> 5;
  auto stamp = [&](int slot) {
    if (stamps && threadIdx.x == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      stamps[slot] = tt;
    }
  };
  // M-tiles per distinct bm: sum over active experts of ceil(c_e / bm)
  // (m_tile_counts, ramp/routing.py:197-203).
  if (rs && rs->ca) cp_async_wait_all();  // this thread's staged fields have landed
  __syncwarp();
  RCLK(7);
#pragma unroll 1
  for (int u = warp; u < t.n_ubm; u += nwarps) {
    const int bm = (rs && rs->ca && rs->ubm_stride == nwarps) ? rs->cubm[u] : t.ubm[u];
    unsigned acc = 0;  // <= n + E M-tiles
#pragma unroll 4
    for (int e = lane; e < E; e += 32) {
      const int c = hist[e];
      if (c > 0) acc += div_pos(c + bm - 1, bm);
    }
    acc = __reduce_add_sync(0xffffffffu, acc);  // one redux instead of five shuffle rounds
    if (lane == 0) mt_smem[u] = acc;
    if (u == warp) RCLK(24);
  }
  RCLK(23);
  // Active experts (only the B4 traffic grid needs them): every warp of the
  // group counts them itself (one redux), so no second barrier is needed.
  unsigned na = 0;
  if (t.lam) {
#pragma unroll 4
    for (int e = lane; e < E; e += 32) na += hist[e] > 0 ? 1u : 0u;
    na = __reduce_add_sync(0xffffffffu, na);
  }
  const double nact = static_cast<double>(na);
  RCLK(8);
  group_sync(nwarps);
  RCLK(9);
  stamp(12);

  const double sm = static_cast<double>(t.sm_count);
  const double omega_max = t.omega_max > 0.0 ? t.omega_max : 0.2;
  ArgMin best{CUDART_INF, 0x7fffffff};
  int kept = 0;
  const long long smi = t.sm_count;
#pragma unroll 1
  for (int i = threadIdx.x; i < t.n_cfg; i += nwarps * 32) {
    const CfgRegs r = load_cfg(t, i, rs);
    const int sk = r.sk;
    const long long stripes = r.stripes;
    const long long g = mt_smem[r.ubm_idx] * stripes * sk;
    const double gd = static_cast<double>(g);
    bool keep = true;
    // (an infinite threshold keeps every finite ratio: skip the divisions)
    if (sk > 1) {
      if (omega_max == 0.2 && (sk & (sk - 1)) == 0 && g < (1ll << 40) && smi < (1ll << 20)) {
        // Exact integer form of the fp64 gate: for a power-of-two split g/sk
        // is exact, so the test is RN(q) < RN(0.2) with q = g/(sk*sm); a
        // rational with a denominator < 2^30 is either exactly 1/5 or at
        // least 1/(5*sk*sm) away from it, far beyond half an ulp, so this
        // equals q < 1/5, i.e. 5g < sk*sm.
        keep = t.kappa_ok && 5 * g < static_cast<long long>(sk) * smi;
      } else {
        keep = t.kappa_ok &&
               (isinf(omega_max) || __ddiv_rn(__ddiv_rn(gd, static_cast<double>(sk)), sm) < omega_max);
      }
    }
    // B4: HBM-equivalent traffic grid (first M-tile of an expert streams its
    // weights from HBM, later ones re-read them at lam x the cost from L2)
    double gl = gd;
    if (t.lam) {
      const double mt = static_cast<double>(mt_smem[r.ubm_idx]);
      const double u = __dadd_rn(nact, __dmul_rn(r.lam, __dadd_rn(mt, -nact)));
      gl = __dmul_rn(static_cast<double>(stripes * sk), u);
    }
    // ceil(g / sm) as an integer division: the fp64 quotient of two integers
    // below 2^40 rounds to within far less than 1/sm of the true value, so
    // numpy's np.ceil(g / sm) is exactly this integer.
    const double waves = static_cast<double>(
        g < (1ll << 31) ? static_cast<long long>((static_cast<unsigned>(g) + static_cast<unsigned>(smi) - 1u) /
                                                 static_cast<unsigned>(smi))
                        : (g + smi - 1) / smi);
    double p = __dadd_rn(r.a, __dmul_rn(r.b, waves));
    p = __dadd_rn(p, __dmul_rn(r.c, gl));
    p = __dadd_rn(p, __dmul_rn(r.d, log(__dadd_rn(gl, 1.0))));
    if (grid_out) grid_out[i] = g;
    if (!keep) p = CUDART_INF;
    if (pred_out) pred_out[i] = p;
    kept += keep ? 1 : 0;
    const ArgMin cand{p, i};
    if (argmin_better(cand, best)) best = cand;
  }
  RCLK(10);
  stamp(13);
  // only warps that evaluated a config take part in the reduction
  const int cfg_warps = min(nwarps, (t.n_cfg + 31) >> 5);
  if (warp < cfg_warps) {
    best = warp_argmin(best);
    kept = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(kept));
    if (lane == 0) {
      red_smem[warp] = best;
      cnt_smem[warp] = kept;
    }
  }
  RCLK(11);
  group_sync(nwarps);
  RCLK(12);
  if (warp == 0) {
    ArgMin b = lane < cfg_warps ? red_smem[lane] : ArgMin{CUDART_INF, 0x7fffffff};
    int k = lane < cfg_warps ? cnt_smem[lane] : 0;
    b = warp_argmin(b);
    k = static_cast<int>(__reduce_add_sync(0xffffffffu, static_cast<unsigned>(k)));
    if (lane == 0) {
      red_smem[0] = b;
      cnt_smem[0] = k;
      if (n_eval_out) *n_eval_out = k;
    }
  }
  group_sync(nwarps);
  RCLK(13);
  stamp(14);
  const int sel = red_smem[0].i;
  group_sync(nwarps);
  return sel;
}

// --------------------------------------------------------------- alignment
// Block-wide exclusive scan of v (one value per thread, blockDim == 1024).
__device__ inline int block_exclusive_scan(int v, int* warp_tot /*[32]*/, int* total) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  const int before = (warp > 0 ? warp_tot[warp - 1] : 0) + x - v;
  if (total) *total = warp_tot[31];
  __syncthreads();
  return before;
}

// moe_align_block_size, pass 2 of the stable counting sort: flat assignment
// indices grouped by expert, ascending within an expert, each expert's run
// padded to a multiple of bm with the sentinel n (== S*top_k).  (The
// reference has no alignment code; this order is our contract.)
//
// Split in two so the bm-independent half can overlap the dispatcher:
//   block_walk_ranks  each of the 32 segments of pass 1 is walked in order;
//                     an assignment's rank within its expert = earlier
//                     segments' count of that expert + its running count in
//                     the segment + its rank within the 32-chunk (ballot-per-
//                     bit match).  The rank is packed into the cached id
//                     (id | rank << 10), so ids must be cached (n <= kIdCache).
//   block_place       with the selected bm: padded exclusive scan, padding /
//                     tile experts, then every assignment lands at
//                     off[e] + rank (shared-memory staged, coalesced copy-out).
// Requires blockDim.x == 1024, E <= kMaxExperts and block_count() first.
constexpr int kRankShift = 10;  // E <= 512 fits below it; rank < 16384 above

__device__ inline void block_walk_ranks(int64_t n, int E, RouteSmem& s, int first_warp, int n_walkers) {
  const int warp = (threadIdx.x >> 5) - first_warp, lane = threadIdx.x & 31;
  const int nbits = bits_for(E);
  const int64_t seg = (n + kRouteWarps - 1) / kRouteWarps;
  for (int sg = warp; sg < kRouteWarps; sg += n_walkers) {
    const int64_t lo = sg * seg, hi = lo + seg < n ? lo + seg : n;
    for (int64_t c0 = lo; c0 < hi; c0 += 32) {
      const int64_t i = c0 + lane;
      int e = -1;
      if (i < hi) {
        e = s.ids[i];
        if (e < 0 || e >= E) {
          e = -1;
          s.ids[i] = -1;  // skipped (or rejected) slots never reach block_place
        }
      }
      const unsigned peers = match_peers(e, nbits);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      int base = 0;
      if (e >= 0) {
        base = s.cnt[e * 32 + sg];
        s.ids[i] = e | ((base + rank) << kRankShift);
      }
      __syncwarp();
      if (e >= 0 && rank == 0) s.cnt[e * 32 + sg] = base + __popc(peers);
      __syncwarp();
    }
  }
}

// After the padded scan (s.off final, block barrier passed): the padding
// slots of every expert's run get the sentinel n and every M-tile its expert,
// written by the lanes of one warp per expert (an expert's padding is up to
// bm - 1 slots: one thread per expert would serialise them).
__device__ __forceinline__ void pad_and_tiles(int64_t n, int E, int bm, const RouteSmem& s, int32_t* dst,
                                              int32_t* __restrict__ tile_expert) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 1
  for (int e = warp; e < E; e += kRouteWarps) {
    const int o = s.off[e], end = s.off[e + 1];
    if (o == end) continue;
    for (int q = o + s.hist[e] + lane; q < end; q += 32) dst[q] = static_cast<int32_t>(n);
    for (int tt = div_pos(o, bm) + lane; tt < div_pos(end, bm); tt += 32) tile_expert[tt] = e;
  }
}

struct NoPublish {
  __device__ void operator()(int) const {}
};

// `on_offsets(n_post_pad)` runs (in every thread, after a block barrier) as
// soon as the padded offsets and tile_expert[] are final -- before the
// bm-dependent placement of the assignments.
template <class Publish = NoPublish>
__device__ inline void block_place(int64_t n, int E, int bm, RouteSmem& s, int* warp_tot,
                                   int32_t* __restrict__ sorted_ids, int32_t* __restrict__ tile_expert,
                                   int32_t* n_post_pad_out, unsigned long long* stamps = nullptr,
                                   Publish on_offsets = Publish{}) {
  auto stamp = [&](int slot) {
    if (stamps && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      stamps[slot] = t;
    }
  };
  const int tid = threadIdx.x;
  int padded = 0, c = 0;
  if (tid < E) {
    c = s.hist[tid];
    padded = div_pos(c + bm - 1, bm) * bm;
  }
  int total = 0;
  RCLK(14);
  const int off = block_exclusive_scan(padded, warp_tot, &total);
  RCLK(15);
  // stage in shared memory when the list is long enough for scattered global
  // stores to cost more than the copy-out, and fits (total is block-uniform)
  const bool staged = n >= 2048 && total <= s.stage_cap;
  int32_t* const dst = staged ? s.stage : sorted_ids;
  if (tid < E) s.off[tid] = off;
  if (tid == 0) {
    s.off[E] = total;
    if (n_post_pad_out) *n_post_pad_out = total;
  }
  RCLK(16);
  __syncthreads();
  RCLK(17);
  pad_and_tiles(n, E, bm, s, dst, tile_expert);
  stamp(5);
  on_offsets(total);
  RCLK(18);
    for (int64_t i = tid; i < n; i += blockDim.x) {
    const int v = s.ids[i];
    if (v >= 0) dst[s.off[v & ((1 << kRankShift) - 1)] + (v >> kRankShift)] = static_cast<int32_t>(i);
  }
  RCLK(19);
  __syncthreads();
  RCLK(20);
  if (staged) {
    // coalesced copy-out (sorted_ids is 16-byte aligned in the workspace)
    const bool vec = (reinterpret_cast<uintptr_t>(sorted_ids) & 15) == 0;
    const int n4 = vec ? total / 4 : 0;
    const int4* src4 = reinterpret_cast<const int4*>(s.stage);
    int4* dst4 = reinterpret_cast<int4*>(sorted_ids);
        for (int q = tid; q < n4; q += blockDim.x) dst4[q] = src4[q];
        for (int q = n4 * 4 + tid; q < total; q += blockDim.x) sorted_ids[q] = s.stage[q];
    __syncthreads();
  }
}

// Single pass (no dispatch to overlap with): padded scan first, then one walk
// that writes every position straight to global memory.  Ids come from the
// shared-memory cache when n <= kIdCache, else from global memory.
template <class Publish = NoPublish>
__device__ inline void block_align(const int32_t* __restrict__ ids, int64_t n, int E, int bm,
                                   RouteSmem& s, int* warp_tot, int32_t* __restrict__ sorted_ids,
                                   int32_t* __restrict__ tile_expert, int32_t* n_post_pad_out,
                                   unsigned long long* stamps = nullptr, Publish on_offsets = Publish{},
                                   int ids_k = 1, int64_t ids_stride = 0) {
  auto stamp = [&](int slot) {
    if (stamps && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      stamps[slot] = t;
    }
  };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int padded = 0, c = 0;
  if (tid < E) {
    c = s.hist[tid];
    padded = div_pos(c + bm - 1, bm) * bm;
  }
  int total = 0;
  const int off = block_exclusive_scan(padded, warp_tot, &total);
  if (tid < E) s.off[tid] = off;
  if (tid == 0) {
    s.off[E] = total;
    if (n_post_pad_out) *n_post_pad_out = total;
  }
  __syncthreads();
  pad_and_tiles(n, E, bm, s, sorted_ids, tile_expert);
  stamp(5);
  on_offsets(total);
  const int nbits = bits_for(E);
  const int64_t seg = (n + kRouteWarps - 1) / kRouteWarps;
  const int64_t lo = warp * seg, hi = lo + seg < n ? lo + seg : n;
  for (int64_t c0 = lo; c0 < hi; c0 += 32) {
    const int64_t i = c0 + lane;
    int e = -1;
    if (i < hi) {
      e = s.cached ? s.ids[i] : ld_id(ids, i, ids_k, ids_stride);
      if (e < 0 || e >= E) e = -1;
    }
    const unsigned peers = match_peers(e, nbits);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    int base = 0;
    if (e >= 0) {
      base = s.cnt[e * 32 + warp];
      sorted_ids[s.off[e] + base + rank] = static_cast<int32_t>(i);
    }
    __syncwarp();
    if (e >= 0 && rank == 0) s.cnt[e * 32 + warp] = base + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
}

}  // namespace ramp
