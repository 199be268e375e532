// Route stage of the hot path: expert histogram -> routing-aware dispatcher ->
// moe_align_block_size, all inside ONE thread block so the whole control plane
// is a single launch with no host round trip (the paper's "single fused
// dispatch kernel", here also emitting the
// alignment the megakernel consumes).
#pragma once
#include <cstdint>
#include <math_constants.h>

#include "../../include/ramp_b200.h"

namespace ramp {

constexpr int kRouteThreads = 1024;
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kMaxExperts = 512;
constexpr int kMaxUbm = 128;
constexpr int kIdCache = 16384;  // topk ids kept in shared memory between the two passes

// Dynamic shared memory layout of the route block (sized by E and n).
//   hist[E]       bincount
//   off[E+1]      exclusive scan of the padded counts
//   cnt[E][32]    per-(expert, warp) counts, then exclusive prefixes over warps
//   ids[min(n, kIdCache)]
struct RouteSmem {
  int32_t* hist;
  int32_t* off;
  int32_t* cnt;
  int32_t* ids;
  bool cached;
};

__host__ __device__ inline size_t route_smem_bytes(int E, int64_t n) {
  const int64_t cache = n <= kIdCache ? n : 0;
  return sizeof(int32_t) * ((size_t)E * 34 + 1 + (size_t)cache) + 64;
}

__device__ inline RouteSmem carve_route_smem(unsigned char* base, int E, int64_t n) {
  RouteSmem s;
  s.hist = reinterpret_cast<int32_t*>(base);
  s.off = s.hist + E;
  s.cnt = s.off + E + 1;
  s.ids = s.cnt + 32 * E;
  s.cached = n <= kIdCache;
  return s;
}

// Lanes of the warp holding the same value e (e < 0 marks an empty lane):
// __match_any_sync rebuilt from one ballot per bit of e, which is much
// cheaper than MATCH.ANY when the warp holds many distinct experts.
__device__ __forceinline__ unsigned match_peers(int e, int nbits) {
  unsigned peers = 0xffffffffu;
  for (int b = 0; b < nbits; ++b) {
    const bool bit = (e >> b) & 1;
    const unsigned m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  const unsigned empty = __ballot_sync(0xffffffffu, e < 0);
  return peers & (e < 0 ? empty : ~empty);
}

__host__ __device__ inline int bits_for(int E) {
  int b = 0;
  while ((1 << b) < E) ++b;
  return b;
}

// --------------------------------------------------------------- histogram
// Pass 1 of the stable counting sort.  The n flat assignments are cut into 32
// contiguous segments, one per warp; each warp counts its segment per expert
// (warp-aggregated with match.any, no atomics: the warp owns column w of
// cnt), then one warp scan per expert turns the 32 counts into exclusive
// prefixes and the total, i.e. bincount(topk_ids, minlength=E).
// Ids outside [0, E) set *bad (ExpertHistogram rejects them, ramp/routing.py:45-50).
__device__ inline void block_count(const int32_t* __restrict__ ids, int64_t n, int E, RouteSmem& s,
                                   int* bad) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (s.cached)
    for (int64_t i = tid; i < n; i += blockDim.x) s.ids[i] = __ldg(ids + i);
  for (int x = tid; x < 32 * E; x += blockDim.x) s.cnt[x] = 0;
  __syncthreads();
  const int64_t seg = (n + kRouteWarps - 1) / kRouteWarps;
  const int64_t lo = warp * seg, hi = lo + seg < n ? lo + seg : n;
  for (int64_t c0 = lo; c0 < hi; c0 += 32) {
    const int64_t i = c0 + lane;
    int e = -1;
    if (i < hi) {
      e = s.cached ? s.ids[i] : __ldg(ids + i);
      if (e < 0 || e >= E) {
        *bad = 1;
        e = -1;
      }
    }
    if (e >= 0) atomicAdd(s.cnt + e * 32 + warp, 1);  // counts commute: no ordering needed here
  }
  __syncthreads();
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
  __syncthreads();
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

// Evaluates every config of the table on the histogram in shared memory and
// returns (in every thread) the selected id.  fp64 arithmetic follows
// predict_batch exactly: ((a + b*ceil(g/sm)) + c*g) + d*log(g+1)
// (ramp/cost_model.py:104-114), gate (g/split_k)/sm < 0.2 (ramp/dispatch.py:107-114),
// first argmin over +inf-masked predictions (:118-119).
__device__ inline int block_dispatch(const int32_t* hist, int E, const ramp_table_t& t,
                                     int64_t* grid_out, double* pred_out, int* n_eval_out,
                                     int64_t* mt_smem /*[kMaxUbm]*/, ArgMin* red_smem /*[32]*/,
                                     int* cnt_smem /*[32]*/) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  // M-tiles per distinct bm: sum over active experts of ceil(c_e / bm)
  // (m_tile_counts, ramp/routing.py:197-203).
  for (int u = warp; u < t.n_ubm; u += nwarps) {
    const int bm = t.ubm[u];
    long long acc = 0;
    for (int e = lane; e < E; e += 32) {
      const int c = hist[e];
      if (c > 0) acc += (c + bm - 1) / bm;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) mt_smem[u] = acc;
  }
  // Active experts (only the B4 traffic grid needs them).
  __shared__ int s_nact;
  if (t.lam && warp == nwarps - 1) {
    int na = 0;
    for (int e = lane; e < E; e += 32) na += hist[e] > 0 ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) na += __shfl_xor_sync(0xffffffffu, na, o);
    if (lane == 0) s_nact = na;
  }
  __syncthreads();
  const double nact = t.lam ? static_cast<double>(s_nact) : 0.0;

  const double sm = static_cast<double>(t.sm_count);
  const double omega_max = t.omega_max > 0.0 ? t.omega_max : 0.2;
  ArgMin best{CUDART_INF, 0x7fffffff};
  int kept = 0;
  for (int i = threadIdx.x; i < t.n_cfg; i += blockDim.x) {
    const int ttn = t.ttn[i], sk = t.split_k[i];
    const long long stripes = t.ntile ? t.ntile[i] : (static_cast<long long>(t.N) + ttn - 1) / ttn;
    const long long g = mt_smem[t.ubm_index[i]] * stripes * sk;
    const double gd = static_cast<double>(g);
    bool keep = true;
    if (sk > 1) keep = t.kappa_ok && (__ddiv_rn(__ddiv_rn(gd, static_cast<double>(sk)), sm) < omega_max);
    // B4: HBM-equivalent traffic grid (first M-tile of an expert streams its
    // weights from HBM, later ones re-read them at lam x the cost from L2)
    double gl = gd;
    if (t.lam) {
      const double mt = static_cast<double>(mt_smem[t.ubm_index[i]]);
      const double u = __dadd_rn(nact, __dmul_rn(t.lam[i], __dadd_rn(mt, -nact)));
      gl = __dmul_rn(static_cast<double>(stripes * sk), u);
    }
    double p = __dadd_rn(t.a[i], __dmul_rn(t.b[i], ceil(__ddiv_rn(gd, sm))));
    p = __dadd_rn(p, __dmul_rn(t.c[i], gl));
    p = __dadd_rn(p, __dmul_rn(t.d[i], log(__dadd_rn(gl, 1.0))));
    if (grid_out) grid_out[i] = g;
    if (!keep) p = CUDART_INF;
    if (pred_out) pred_out[i] = p;
    kept += keep ? 1 : 0;
    const ArgMin cand{p, i};
    if (argmin_better(cand, best)) best = cand;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMin other{__shfl_xor_sync(0xffffffffu, best.v, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
    if (argmin_better(other, best)) best = other;
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
  }
  if (lane == 0) {
    red_smem[warp] = best;
    cnt_smem[warp] = kept;
  }
  __syncthreads();
  if (warp == 0) {
    ArgMin b = lane < nwarps ? red_smem[lane] : ArgMin{CUDART_INF, 0x7fffffff};
    int k = lane < nwarps ? cnt_smem[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMin other{__shfl_xor_sync(0xffffffffu, b.v, o), __shfl_xor_sync(0xffffffffu, b.i, o)};
      if (argmin_better(other, b)) b = other;
      k += __shfl_xor_sync(0xffffffffu, k, o);
    }
    if (lane == 0) {
      red_smem[0] = b;
      cnt_smem[0] = k;
      if (n_eval_out) *n_eval_out = k;
    }
  }
  __syncthreads();
  const int sel = red_smem[0].i;
  __syncthreads();
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
// Requires blockDim.x == 1024, E <= kMaxExperts and block_count() first.
__device__ inline void block_align(const int32_t* __restrict__ ids, int64_t n, int E, int bm,
                                   RouteSmem& s, int* warp_tot, int32_t* __restrict__ sorted_ids,
                                   int32_t* __restrict__ tile_expert, int32_t* n_post_pad_out,
                                   unsigned long long* stamps = nullptr) {
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
    padded = (c + bm - 1) / bm * bm;
  }
  int total = 0;
  const int off = block_exclusive_scan(padded, warp_tot, &total);
  if (tid < E) {
    s.off[tid] = off;
    for (int q = off + c; q < off + padded; ++q) sorted_ids[q] = static_cast<int32_t>(n);
    for (int tt = off / bm; tt < (off + padded) / bm; ++tt) tile_expert[tt] = tid;
  }
  if (tid == 0) {
    s.off[E] = total;
    if (n_post_pad_out) *n_post_pad_out = total;
  }
  __syncthreads();
  stamp(5);
  // each warp walks its segment again in order; position = expert base +
  // earlier warps' count + this warp's running count + rank within the chunk
  const int nbits = bits_for(E);
  const int64_t seg = (n + kRouteWarps - 1) / kRouteWarps;
  const int64_t lo = warp * seg, hi = lo + seg < n ? lo + seg : n;
  for (int64_t c0 = lo; c0 < hi; c0 += 32) {
    const int64_t i = c0 + lane;
    int e = -1;
    if (i < hi) {
      e = s.cached ? s.ids[i] : __ldg(ids + i);
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
