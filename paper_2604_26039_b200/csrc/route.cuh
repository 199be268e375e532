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
constexpr int kMaxExperts = 1024;
constexpr int kMaxUbm = 128;

// Dynamic shared memory layout of the route block (sized by E).
struct RouteSmem {
  int32_t* hist;      // [E]      bincount
  int32_t* off;       // [E+1]    exclusive scan of padded counts
  int32_t* cursor;    // [E]      running within-expert rank across rounds
  int32_t* rtot;      // [E]      per-round totals
  uint16_t* cnt;      // [32][E]  per-warp counts -> per-warp prefixes
};

__host__ __device__ inline size_t route_smem_bytes(int E) {
  return sizeof(int32_t) * (4 * (size_t)E + 1) + sizeof(uint16_t) * 32 * (size_t)E + 64;
}

__device__ inline RouteSmem carve_route_smem(unsigned char* base, int E) {
  RouteSmem s;
  s.hist = reinterpret_cast<int32_t*>(base);
  s.off = s.hist + E;
  s.cursor = s.off + E + 1;
  s.rtot = s.cursor + E;
  s.cnt = reinterpret_cast<uint16_t*>(s.rtot + E);
  return s;
}

// --------------------------------------------------------------- histogram
// bincount(topk_ids, minlength=E) into shared memory.  Ids outside [0, E)
// set *bad (the reference's ExpertHistogram rejects them, ramp/routing.py:45-50).
__device__ inline void block_histogram(const int32_t* __restrict__ ids, int64_t n, int E,
                                       int32_t* hist, int* bad) {
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    int e = __ldg(ids + i);
    if (e < 0 || e >= E) {
      *bad = 1;
      continue;
    }
    atomicAdd(hist + e, 1);
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
  __syncthreads();

  const double sm = static_cast<double>(t.sm_count);
  ArgMin best{CUDART_INF, 0x7fffffff};
  int kept = 0;
  for (int i = threadIdx.x; i < t.n_cfg; i += blockDim.x) {
    const int ttn = t.ttn[i], sk = t.split_k[i];
    const long long stripes = (static_cast<long long>(t.N) + ttn - 1) / ttn;
    const long long g = mt_smem[t.ubm_index[i]] * stripes * sk;
    const double gd = static_cast<double>(g);
    bool keep = true;
    if (sk > 1) keep = t.kappa_ok && (__ddiv_rn(__ddiv_rn(gd, static_cast<double>(sk)), sm) < 0.2);
    double p = __dadd_rn(t.a[i], __dmul_rn(t.b[i], ceil(__ddiv_rn(gd, sm))));
    p = __dadd_rn(p, __dmul_rn(t.c[i], gd));
    p = __dadd_rn(p, __dmul_rn(t.d[i], log(__dadd_rn(gd, 1.0))));
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

// moe_align_block_size: stable counting sort of the flat assignment indices
// by expert; each expert's run padded to a multiple of bm with the sentinel
// n (== S*top_k).  Within an expert, indices ascend (a deterministic order we
// define; the reference has no alignment code).
// Requires blockDim.x == 1024 and E <= 1024.
__device__ inline void block_align(const int32_t* __restrict__ ids, int64_t n, int E, int bm,
                                   RouteSmem& s, int* warp_tot, int32_t* __restrict__ sorted_ids,
                                   int32_t* __restrict__ tile_expert, int32_t* n_post_pad_out) {
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
    s.cursor[tid] = 0;
    // padding slots and per-tile expert ids
    for (int p = off + c; p < off + padded; ++p) sorted_ids[p] = static_cast<int32_t>(n);
    for (int tt = off / bm; tt < (off + padded) / bm; ++tt) tile_expert[tt] = tid;
  }
  if (tid == 0) {
    s.off[E] = total;
    if (n_post_pad_out) *n_post_pad_out = total;
  }
  __syncthreads();

  const unsigned lt_mask = (1u << lane) - 1u;
  uint16_t* my_cnt = s.cnt + warp * E;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + tid;
    int e = i < n ? __ldg(ids + i) : -1;
    if (e >= E) e = -1;  // invalid ids were flagged by block_histogram
    for (int x = lane; x < E; x += 32) my_cnt[x] = 0;
    __syncwarp();
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & lt_mask);
    if (e >= 0 && rank == 0) my_cnt[e] = static_cast<uint16_t>(__popc(peers));
    __syncthreads();
    // per-expert exclusive prefix over the 32 warps: one warp scan per expert
    for (int x = warp; x < E; x += kRouteWarps) {
      const int v = s.cnt[lane * E + x];
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      s.cnt[lane * E + x] = static_cast<uint16_t>(incl - v);
      if (lane == 31) s.rtot[x] = incl;
    }
    __syncthreads();
    if (e >= 0) sorted_ids[s.off[e] + s.cursor[e] + my_cnt[e] + rank] = static_cast<int32_t>(i);
    __syncthreads();
    if (tid < E) s.cursor[tid] += s.rtot[tid];
  }
  __syncthreads();
}

}  // namespace ramp
