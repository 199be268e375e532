// The route stage inside the megakernel (BF16 path): no separate route
// launch, no PDL hand-off, and the token gather fused with the placement.
//
//   step 1  CTA b counts its contiguous slice of the flat top-k ids per
//           expert (shared atomics) and adds the non-zero counts into the
//           global histogram (`tot`) -> grid barrier A
//   step 2  every CTA reads the histogram and evaluates the dispatcher
//           redundantly (the same fp64 block_dispatch as the route kernel, so
//           every CTA selects the same config, bit-exact with the reference's
//           select_config); then the bm-padded exclusive scan `off`
//   step 3  CTA b reserves a contiguous run inside each expert's segment for
//           its slice (one global atomicAdd per (CTA, expert) on `cursor`),
//           writes sorted_ids and copies the token rows into x_sorted; the
//           owner CTA of expert e (e % grid) writes e's padding and M-tile
//           experts -> arrive on grid barrier C (the producers wait on it
//           before their first job)
//
// Within an expert the order of assignments is by CTA arrival, not by flat
// index: the layer's result does not depend on it (each token is one MMA
// column; the k-way reduction is an fp32 atomic sum anyway).  The stable,
// bit-exact alignment contract belongs to ramp_moe_align (route kernel).
//
// Grid barriers use arrival counters that the last arriver resets, plus a
// monotonically increasing generation flag (read once at kernel entry), so
// nothing needs clearing between calls.
#pragma once
#include <cstdint>

#include "ptx.cuh"
#include "route.cuh"

namespace ramp {

struct InlineRouteScratch {  // lives in the (not yet used) pipeline ring
  int32_t lc[kMaxExperts];    // this CTA's count per expert, then its local rank cursor
  int32_t base[kMaxExperts];  // this CTA's reserved start inside each expert's run
  int32_t tot[kMaxExperts];   // histogram
  int64_t mt[kMaxUbm];
  ArgMin red[32];
  int32_t cnt[32];
  int32_t warp_tot[32];
  int32_t off[kMaxExperts + 1];  // bm-padded exclusive offsets
  int32_t bad;
};

// Arrive on a generation barrier (one thread per CTA); the last arriver
// resets the counter and publishes generation `target`.
__device__ __forceinline__ void gen_arrive(int* cnt, int* flag, int target) {
  __threadfence();
  if (atomicAdd(cnt, 1) == static_cast<int>(gridDim.x) - 1) {
    atomicExch(cnt, 0);
    __threadfence();
    st_release_gpu(flag, target);
  }
}
__device__ __forceinline__ void gen_wait(const int* flag, int target) {
  while (ld_acquire_gpu(flag) - target < 0) __nanosleep(32);
}

struct InlineRouteResult {
  int cfg, n_post_pad, n_eval;
};

// All threads of the CTA call it.  Returns the same result in every thread of
// every CTA; tile_expert[] is written by the owner CTAs (visible after barrier C).
template <int kThreads>
__device__ inline InlineRouteResult inline_route(const int32_t* __restrict__ ids, int n, int E, int top_k,
                                                 int forced_cfg, const ramp_table_t& table,
                                                 const __nv_bfloat16* __restrict__ x, __nv_bfloat16* x_sorted, int H,
                                                 int32_t* __restrict__ sorted_ids, int* tot_g, int* cursor_g,
                                                 int* cnt_a, int* cnt_c, int* gflag, int g0, int* bad_flag,
                                                 int32_t* __restrict__ tile_expert, InlineRouteScratch& sc) {
  int32_t* off = sc.off;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, b = blockIdx.x;
  const int lo = static_cast<int>(static_cast<int64_t>(b) * n / G);
  const int hi = static_cast<int>(static_cast<int64_t>(b + 1) * n / G);

  // ---- step 1: local counts of this CTA's slice -> global histogram
  for (int e = tid; e < E; e += kThreads) sc.lc[e] = 0;
  if (tid == 0) sc.bad = 0;
  __syncthreads();
  for (int i = lo + tid; i < hi; i += kThreads) {
    const int e = __ldg(ids + i);
    if (e >= 0 && e < E) {
      atomicAdd(&sc.lc[e], 1);
    } else if (e != -1) {
      sc.bad = 1;
    }
  }
  __syncthreads();
  for (int e = tid; e < E; e += kThreads)
    if (sc.lc[e]) atomicAdd(tot_g + e, sc.lc[e]);
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    if (sc.bad) atomicOr(bad_flag, 1);
    gen_arrive(cnt_a, gflag, g0 + 1);
    gen_wait(gflag, g0 + 1);
  }
  __syncthreads();

  // ---- step 2: histogram, dispatch (redundant per CTA), padded offsets
  for (int e = tid; e < E; e += kThreads) sc.tot[e] = __ldcg(tot_g + e);
  __syncthreads();
  int sel = forced_cfg, n_eval = 0;
  if (sel < 0) {
    sel = block_dispatch(sc.tot, E, table, nullptr, nullptr, nullptr, nullptr, sc.mt, sc.red, sc.cnt, nullptr,
                         kThreads / 32);
    n_eval = sc.cnt[0];
  }
  const int bm = __ldg(table.bm + sel);
  // exclusive scan of the padded counts (E <= 512: two per thread, block scan)
  int p0 = 0, p1 = 0;
  const int e0 = 2 * tid, e1 = 2 * tid + 1;
  if (e0 < E) p0 = (sc.tot[e0] + bm - 1) / bm * bm;
  if (e1 < E) p1 = (sc.tot[e1] + bm - 1) / bm * bm;
  int v = p0 + p1;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) sc.warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kThreads / 32 ? sc.warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    sc.warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  const int excl = (warp > 0 ? sc.warp_tot[warp - 1] : 0) + v - (p0 + p1);
  if (e0 < E) off[e0] = excl;
  if (e1 < E) off[e1] = excl + p0;
  const int n_post_pad = sc.warp_tot[kThreads / 32 - 1];
  if (tid == 0) off[E] = n_post_pad;

  // ---- step 3: reserve runs, place, gather
  for (int e = tid; e < E; e += kThreads) {
    const int c = sc.lc[e];
    sc.base[e] = c ? atomicAdd(cursor_g + e, c) : 0;
    sc.lc[e] = 0;  // becomes the local rank cursor
  }
  __syncthreads();
  const int row_vec = H / 8;  // 16-byte vectors per row
  const int4* xv = reinterpret_cast<const int4*>(x);
  int4* dv = reinterpret_cast<int4*>(x_sorted);
  // one warp per assignment row: position, then the 2 KB..16 KB row copy
  for (int i = lo + warp; i < hi; i += kThreads / 32) {
    const int e = __ldg(ids + i);
    if (e < 0 || e >= E) continue;
    int pos = 0;
    if (lane == 0) {
      pos = off[e] + sc.base[e] + atomicAdd(&sc.lc[e], 1);
      sorted_ids[pos] = i;
    }
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const int4* src = xv + static_cast<int64_t>(i / top_k) * row_vec;
    int4* dst = dv + static_cast<int64_t>(pos) * row_vec;
    for (int c = lane; c < row_vec; c += 32) dst[c] = __ldg(src + c);
  }
  // padding of the experts this CTA owns: sentinel ids and zero rows, and
  // their M-tiles' expert
  for (int e = b; e < E; e += G) {
    for (int t = off[e] / bm + tid; t < off[e + 1] / bm; t += kThreads) tile_expert[t] = e;
    const int start = off[e] + sc.tot[e], end = off[e + 1];
    for (int q = start + warp; q < end; q += kThreads / 32) {
      if (lane == 0) sorted_ids[q] = n;
      int4* dst = dv + static_cast<int64_t>(q) * row_vec;
      for (int c = lane; c < row_vec; c += 32) dst[c] = make_int4(0, 0, 0, 0);
    }
  }
  __threadfence();  // rows and ids are published by the caller's barrier-C arrival
  __syncthreads();
  return {sel, n_post_pad, n_eval};
}

}  // namespace ramp
