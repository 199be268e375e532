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

__global__ void __launch_bounds__(kRouteThreads, 1)
    route_kernel(const RouteArgs a) {
  if (a.pdl_early) pdl_launch_dependents();  // let the megakernel's prologue start on idle SMs
  auto stamp = [&](int slot) {
    if (a.prof && threadIdx.x == 0) a.prof[slot] = globaltimer();
  };
  if (blockIdx.x > 0) {
    if (blockIdx.x == 1) stamp(8);
    // Helper blocks: clear the fp32 output accumulator, then (once block 0
    // has published the alignment) gather the token rows into expert-sorted
    // order so the megakernel can fetch a whole M-tile with one TMA box.
    const int nh = gridDim.x - 1, hb = blockIdx.x - 1;
    float4* acc4 = reinterpret_cast<float4*>(a.acc_clear);
    const int64_t n4 = a.acc_clear_n / 4;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = hb * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)nh * blockDim.x) acc4[i] = z;
    for (int64_t i = n4 * 4 + hb * (int64_t)blockDim.x + threadIdx.x; i < a.acc_clear_n;
         i += (int64_t)nh * blockDim.x)
      a.acc_clear[i] = 0.f;
    if (a.x_sorted == nullptr) return;
    if (blockIdx.x == 1) stamp(9);
    if (threadIdx.x == 0)
      while (ld_acquire_gpu(a.ctrl + 5) == 0) __nanosleep(64);
    __syncthreads();
    if (blockIdx.x == 1) stamp(10);
    const int npp = __ldcg(a.ctrl + 1);
    const int row_vec = a.H / 8;  // 16-byte vectors per row
    const int4* xv = reinterpret_cast<const int4*>(a.x);
    int4* dv = reinterpret_cast<int4*>(a.x_sorted);
    const int gw = hb * kRouteWarps + (threadIdx.x >> 5), nw = nh * kRouteWarps, lane = threadIdx.x & 31;
    for (int r = gw; r < npp; r += nw) {
      const int asg = __ldcg(a.sorted_ids + r);
      int4* d = dv + static_cast<int64_t>(r) * row_vec;
      if (asg < a.n_assign) {
        const int4* s = xv + static_cast<int64_t>(asg / a.top_k) * row_vec;
        for (int c = lane; c < row_vec; c += 32) d[c] = __ldg(s + c);
      } else {
        for (int c = lane; c < row_vec; c += 32) d[c] = make_int4(0, 0, 0, 0);
      }
    }
    __syncthreads();
    if (blockIdx.x == 1) stamp(11);
    if (threadIdx.x == 0) {
      // the last helper through resets the flag for the next call
      if (atomicAdd(a.ctrl + 6, 1) == nh - 1) {
        a.ctrl[6] = 0;
        a.ctrl[5] = 0;
      }
    }
    return;
  }
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ RouteStatic st;
  RouteSmem s = carve_route_smem(dyn, a.E, a.n_assign);
  stamp(0);
  if (a.prof && threadIdx.x == 0) a.prof[6] = clock64();
  // the dispatch table is constant: start loading this thread's config now
  const CfgRegs pre = a.forced_cfg < 0 ? dispatch_prefetch(a.table) : CfgRegs{};
  if (threadIdx.x == 0) st.bad = 0;
  if (a.logits) {
    // router fusion: the top-k is computed here (host checked n <= kIdCache)
    block_topk(a.logits, a.logits_bf16 != 0, a.S, a.E, a.top_k, a.renorm != 0, s.ids,
               const_cast<int32_t*>(a.topk_ids), a.w_out);
  }
  __syncthreads();
  block_count(a.topk_ids, a.n_assign, a.E, s, &st.bad, a.logits != nullptr);
  stamp(1);
  if (a.publish_hist && a.hist_out && (threadIdx.x >> 5) == kRouteWarps - 1) {
    // publish the histogram now: the megakernel CTAs (already resident under
    // PDL) start prefetching the active experts' weights while we dispatch
    for (int e = threadIdx.x & 31; e < a.E; e += 32) a.hist_out[e] = s.hist[e];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      __threadfence();
      st_release_gpu(a.ctrl + 11, 1);
    }
  }
  int sel = a.forced_cfg;
  int n_eval = 0;
  // Warp specialisation: the dispatcher needs one thread per config; the
  // remaining warps walk the (bm-independent) alignment ranks meanwhile.
  const int cfg_warps = (a.table.n_cfg + 31) >> 5;
  const bool overlap = s.cached && sel < 0 && cfg_warps <= kRouteWarps - 8;
  if (sel < 0) {
    if (!overlap) {
      sel = block_dispatch(s.hist, a.E, a.table, pre, a.grid_out, a.pred_out, a.n_eval_out, st.mt, st.red,
                           st.cnt, a.prof);
      n_eval = st.cnt[0];
    } else if (static_cast<int>(threadIdx.x >> 5) < cfg_warps) {
      block_dispatch(s.hist, a.E, a.table, pre, a.grid_out, a.pred_out, a.n_eval_out, st.mt, st.red, st.cnt,
                     a.prof, cfg_warps);
    } else {
      block_walk_ranks(a.n_assign, a.E, s, cfg_warps, kRouteWarps - cfg_warps);
    }
    if (overlap) {
      __syncthreads();
      sel = st.red[0].i;
      n_eval = st.cnt[0];
    }
  }
  stamp(2);
  if (a.prof && threadIdx.x == 0) a.prof[7] = clock64();
  const int bm = a.table.bm[sel];
  int32_t* n_post_pad = a.ctrl + 1;
  if (overlap) {
    block_place(a.n_assign, a.E, bm, s, st.warp_tot, a.sorted_ids, a.tile_expert, n_post_pad, a.prof);
  } else {
    block_align(a.topk_ids, a.n_assign, a.E, bm, s, st.warp_tot, a.sorted_ids, a.tile_expert, n_post_pad,
                a.prof);
  }
  stamp(3);
  const int npp = s.off[a.E];
  for (int e = threadIdx.x; e < a.E; e += blockDim.x)
    if (a.hist_out) a.hist_out[e] = s.hist[e];
  if (a.done)
    for (int m = threadIdx.x; m < npp / bm; m += blockDim.x) a.done[m] = 0;
  if (threadIdx.x == 0) {
    a.ctrl[0] = sel;
    a.ctrl[2] = npp / bm;
    a.ctrl[3] = n_eval;
    a.ctrl[4] = st.bad;
    a.ctrl[7] = 0;  // megakernel job counter
    a.ctrl[8] = 0;  // megakernel grid barrier 0 (rows gathered)
    a.ctrl[9] = 0;  // megakernel grid barrier 1 (all jobs reduced)
    if (a.sel_out) {
      a.sel_out[0] = sel;
      a.sel_out[1] = npp;
      a.sel_out[2] = npp / bm;
      a.sel_out[3] = n_eval;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.x_sorted != nullptr && gridDim.x > 1) {
    __threadfence();
    st_release_gpu(a.ctrl + 5, 1);
  }
  stamp(4);
  if (!a.pdl_early) pdl_launch_dependents();
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
  const CfgRegs pre = dispatch_prefetch(t);
  int32_t* h = reinterpret_cast<int32_t*>(dyn);
  for (int e = threadIdx.x; e < E; e += blockDim.x) h[e] = hist[e];
  __syncthreads();
  const int sel = block_dispatch(h, E, t, pre, grid_out, pred_out, n_eval_out, st.mt, st.red, st.cnt);
  if (threadIdx.x == 0) *cfg_out = sel;
}

cudaError_t launch_route(const RouteArgs& a, int zero_blocks, cudaStream_t stream) {
  const size_t smem = route_smem_bytes(a.E, a.n_assign);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t err = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)route_smem_bytes(kMaxExperts, kIdCache));
    if (err != cudaSuccess) return err;
    // same shared-memory carveout as the megakernel, so SMs need no
    // reconfiguration when the megakernel launches behind it (PDL overlap)
    err = cudaFuncSetAttribute(route_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (err != cudaSuccess) return err;
    attr_set = true;
  }
  route_kernel<<<1 + zero_blocks, kRouteThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_align(const int32_t* ids, int64_t n, int E, int bm, int32_t* hist, int32_t* sorted_ids,
                         int32_t* tile_expert, int32_t* n_post_pad, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t err = cudaFuncSetAttribute(align_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)route_smem_bytes(kMaxExperts, kIdCache));
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
