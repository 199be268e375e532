// Route kernels: histogram, dispatcher and alignment (compiled with
// -fmad=false so the fp64 cost model matches numpy's unfused arithmetic).
#include <cuda_runtime.h>

#include "launch.h"
#include "ptx.cuh"
#include "route.cuh"

namespace ramp {

struct RouteStatic {
  int64_t mt[kMaxUbm];
  ArgMin red[32];
  int cnt[32];
  int warp_tot[32];
  int bad;
};

// One route block.  Specialised at compile time on router fusion (kGating)
// and on device dispatch (kDispatch; false = forced config, the profiling
// sweep): the kernel runs once per layer on one cold SM, so every byte of
// code it does not need costs instruction-cache misses.
template <bool kGating, bool kDispatch>
__device__ __forceinline__ void route_body(const RouteArgs& a) {
  if (a.pdl_early) pdl_launch_dependents();  // let the megakernel's prologue start on idle SMs
  auto stamp = [&](int slot) {
    if (a.prof && threadIdx.x == 0) a.prof[slot] = globaltimer();
  };
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ RouteStatic st;
  RouteSmem s = carve_route_smem(dyn, a.E, a.n_assign, kDispatch ? a.table.n_cfg : 0);
  stamp(0);
  if (a.prof && threadIdx.x == 0) a.prof[6] = clock64();
#ifdef RAMP_ROUTE_CLOCKS
  if (threadIdx.x == 0) g_rclk = a.prof ? a.prof + 16 : nullptr;
  RCLK(0);
#endif
  // Warp specialisation (below): the dispatcher needs one thread per config;
  // the remaining warps walk the (bm-independent) alignment ranks meanwhile.
  // (at least one warp per distinct bm, up to 8: the M-tile counts per bm are
  // then one parallel step instead of a serial loop on one warp)
  const int cfg_warps = max((a.table.n_cfg + 31) >> 5, min(a.table.n_ubm, 8));
  const bool overlap = kDispatch && s.cached && cfg_warps <= kRouteWarps - 8;
  // the dispatch table is constant: start copying it to shared memory now
  if constexpr (kDispatch) stage_table(a.table, s, overlap ? cfg_warps : kRouteWarps);
  // Launched as a programmatic dependent of the previous kernel in the stream
  // (typically the previous layer's megakernel): everything above overlaps its
  // tail; nothing above touches the inputs or the workspace.
  if (a.pdl_prev == 1) pdl_wait();
  if (threadIdx.x == 0) st.bad = 0;
  if constexpr (kGating) {
    // router fusion: the top-k is computed here (host checked n <= kIdCache)
    block_topk(a.logits, a.logits_bf16 != 0, a.S, a.E, a.top_k, a.renorm != 0, s.ids,
               const_cast<int32_t*>(a.topk_ids), a.w_out);
  }
  __syncthreads();
  block_count(a.topk_ids, a.n_assign, a.E, s, &st.bad, kGating, a.top_k, a.ids_stride);
  stamp(1);
  int sel = a.forced_cfg;
  int n_eval = 0;
  // Device StepCache (ramp/dispatch.py:40-54): a selection cached for this
  // step's M skips the dispatcher; a new step clears the entries.
  int cached = -1;
  int step_m = 0;  // thread 0: this call's M (kept in a register: st.warp_tot is reused by the alignment scan)
  int32_t* const scache = a.table.step_cache;
  if (kDispatch && scache) {
    if (threadIdx.x < 32) {
      int m = 0;
#pragma unroll 1
      for (int e = threadIdx.x; e < a.E; e += 32) m += s.hist[e];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
      if (threadIdx.x == 0) {
        if (scache[1] != scache[0]) {
          scache[1] = scache[0];
          scache[2] = 0;
        }
        const int nc = scache[2];
        int hit = -1;
#pragma unroll 1
        for (int q = 0; q < nc; ++q)
          if (scache[3 + 2 * q] == m) hit = scache[4 + 2 * q];
        st.cnt[31] = hit;
        step_m = m;
      }
    }
    __syncthreads();
    cached = st.cnt[31];
  }
  if (kDispatch && cached >= 0) {
    sel = cached;  // hit: no evaluations (DispatchTable.evaluations unchanged)
    if (overlap) {
      // the walkers still need their ranks; every warp walks
      block_walk_ranks(a.n_assign, a.E, s, 0, kRouteWarps);
      __syncthreads();
    }
  } else if constexpr (kDispatch) {
    // one call site of each (the block runs cold: code size is latency)
    if (!overlap || static_cast<int>(threadIdx.x >> 5) < cfg_warps) {
      block_dispatch(s.hist, a.E, a.table, &s, a.grid_out, a.pred_out, a.n_eval_out, st.mt, st.red, st.cnt,
                     a.prof, overlap ? cfg_warps : 0);
    } else {
      block_walk_ranks(a.n_assign, a.E, s, cfg_warps, kRouteWarps - cfg_warps);
    }
    if (overlap) __syncthreads();
    sel = st.red[0].i;
    n_eval = st.cnt[0];
    if (scache && threadIdx.x == 0) {
      const int nc = scache[2];
      if (nc < a.table.step_cache_cap) {
        scache[3 + 2 * nc] = step_m;
        scache[4 + 2 * nc] = sel;
        scache[2] = nc + 1;
      }
    }
  }
  RCLK(22);
  stamp(2);
  if (a.prof && threadIdx.x == 0) a.prof[7] = clock64();
  // bm of the selection from the staged table (landed and visible: every
  // staging thread waited in block_dispatch, and a block barrier followed);
  // a step-cache hit skipped the dispatcher and reads it from global memory
  const bool table_landed = kDispatch && s.ca && cached < 0;
  const int bm = table_landed ? s.cubm[s.cubm_idx[sel]] : a.table.bm[sel];
  int32_t* n_post_pad = a.ctrl + 1;
  // Once the padded offsets and tile_expert[] are final: the selection
  // record and the megakernel's per-call counters.
  auto publish = [&](int npp) {
    const int ntiles = div_pos(npp, bm);
    if (a.done)
#pragma unroll 1
      for (int m = threadIdx.x; m < ntiles; m += blockDim.x) a.done[m] = 0;
    if (threadIdx.x == 0) {
      a.ctrl[0] = sel;
      a.ctrl[2] = ntiles;
      a.ctrl[3] = n_eval;
      a.ctrl[7] = 0;  // megakernel job counter
      a.ctrl[8] = 0;  // megakernel grid barrier 0 (rows gathered)
      a.ctrl[9] = 0;  // megakernel grid barrier 1 (all jobs reduced)
    }
  };
  if (kDispatch && overlap) {
    block_place(a.n_assign, a.E, bm, s, st.warp_tot, a.sorted_ids, a.tile_expert, n_post_pad, a.prof, publish);
  } else {
    block_align(a.topk_ids, a.n_assign, a.E, bm, s, st.warp_tot, a.sorted_ids, a.tile_expert, n_post_pad,
                a.prof, publish, a.top_k, a.ids_stride);
  }
  stamp(3);
  const int npp = s.off[a.E];
#pragma unroll 1
  for (int e = threadIdx.x; e < a.E; e += blockDim.x)
    if (a.hist_out) a.hist_out[e] = s.hist[e];
  if (threadIdx.x == 0) {
    a.ctrl[4] = st.bad;
    if (a.sel_out) {
      a.sel_out[0] = sel;
      a.sel_out[1] = npp;
      a.sel_out[2] = div_pos(npp, bm);
      a.sel_out[3] = n_eval;
    }
  }
  __syncthreads();
  RCLK(21);
  stamp(4);
  // the previous grid (the FP8 token quantisation) must be complete before
  // this one is, so the megakernel's wait on this grid covers it too
  if (a.pdl_prev == 2) pdl_wait();
  if (!a.pdl_early) pdl_launch_dependents();
}

template <bool kGating, bool kDispatch>
__global__ void __launch_bounds__(kRouteThreads, 1)
    route_kernel(const RouteArgs a) {
  route_body<kGating, kDispatch>(a);
}

__global__ void __launch_bounds__(kRouteThreads, 1)
    align_kernel(const int32_t* ids, int64_t n, int E, int bm, int32_t* hist_out, int32_t* sorted_ids,
                 int32_t* tile_expert, int32_t* n_post_pad) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ int warp_tot[32];
  __shared__ int bad;
  RouteSmem s = carve_route_smem(dyn, E, n);
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  block_count(ids, n, E, s, &bad);
  block_align(ids, n, E, bm, s, warp_tot, sorted_ids, tile_expert, n_post_pad);
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist_out[e] = s.hist[e];
}

__global__ void __launch_bounds__(kRouteThreads, 1)
    select_kernel(const int32_t* hist, int E, const ramp_table_t t, int32_t* cfg_out, int32_t* n_eval_out,
                  int64_t* grid_out, double* pred_out) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ RouteStatic st;
  int32_t* h = reinterpret_cast<int32_t*>(dyn);
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = hist[e];
  __syncthreads();
  const int sel = block_dispatch(h, E, t, nullptr, grid_out, pred_out, n_eval_out, st.mt, st.red, st.cnt);
  if (threadIdx.x == 0) *cfg_out = sel;
}

template <bool kGating, bool kDispatch>
static cudaError_t launch_route_t(const RouteArgs& a, cudaStream_t stream) {
  const size_t smem = route_smem_bytes(a.E, a.n_assign, kDispatch ? a.table.n_cfg : 0);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t err = cudaFuncSetAttribute(route_kernel<kGating, kDispatch>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRouteSmemLimit);
    if (err != cudaSuccess) return err;
    // same shared-memory carveout as the megakernel, so SMs need no
    // reconfiguration when the megakernel launches behind it (PDL overlap)
    err = cudaFuncSetAttribute(route_kernel<kGating, kDispatch>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               100);
    if (err != cudaSuccess) return err;
    attr_set = true;
  }
  // PDL on the route launch too: it may start (and stage its table) while the
  // previous kernel drains; it waits for it before reading anything it wrote
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kRouteThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = pdl;
  cfg.numAttrs = a.pdl_prev ? 1 : 0;
  cudaError_t err = cudaLaunchKernelEx(&cfg, route_kernel<kGating, kDispatch>, a);
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

cudaError_t launch_route(const RouteArgs& a, cudaStream_t stream) {
  const bool dispatch = a.forced_cfg < 0;
  if (a.logits) return dispatch ? launch_route_t<true, true>(a, stream) : launch_route_t<true, false>(a, stream);
  return dispatch ? launch_route_t<false, true>(a, stream) : launch_route_t<false, false>(a, stream);
}

cudaError_t launch_align(const int32_t* ids, int64_t n, int E, int bm, int32_t* hist, int32_t* sorted_ids,
                         int32_t* tile_expert, int32_t* n_post_pad, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t err = cudaFuncSetAttribute(align_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kRouteSmemLimit);
    if (err != cudaSuccess) return err;
    attr_set = true;
  }
  align_kernel<<<1, kRouteThreads, route_smem_bytes(E, n), stream>>>(ids, n, E, bm, hist, sorted_ids,
                                                                  tile_expert, n_post_pad);
  return cudaGetLastError();
}

cudaError_t launch_select(const int32_t* hist, int E, const ramp_table_t& t, int32_t* cfg_out,
                          int32_t* n_eval_out, int64_t* grid_out, double* pred_out,
                          cudaStream_t stream) {
  select_kernel<<<1, kRouteThreads, sizeof(int32_t) * E, stream>>>(hist, E, t, cfg_out, n_eval_out,
                                                                   grid_out, pred_out);
  return cudaGetLastError();
}

}  // namespace ramp
