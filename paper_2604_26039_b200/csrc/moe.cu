// Host launcher of the persistent fused MoE megakernel: builds the three TMA
// tensor maps (tokens for gather4, W1, W2), then launches one CTA per SM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "fused_moe.cuh"
#include "launch.h"

namespace ramp {

unsigned long long* g_prof_buffer = nullptr;

bool pdl_prev_enabled() {
  static bool on = [] {
    const char* v = getenv("RAMP_PDL_PREV");
    return v ? atoi(v) != 0 : false;
  }();
  return on;
}

int pdl_mode() {
  static int mode = [] {
    const char* v = getenv("RAMP_PDL");
    return v ? atoi(v) : 1;
  }();
  return mode;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Tensor map with a 128-byte swizzle; dims/strides innermost first (strides
// in bytes for dims 1..rank-1); element type bf16 or raw bytes (e4m3).
static bool make_map(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, bool bytes = false) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t d[3], st[2];
  cuuint32_t b[3], e[3] = {1, 1, 1};
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
  }
  for (int i = 0; i < rank - 1; ++i) st[i] = strides[i];
  CUresult r = enc(map, bytes ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank,
                   const_cast<void*>(ptr), d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-major [rows, cols] matrix, (box_rows x 128-byte) boxes.
static bool make_map_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                        bool bytes = false) {
  const uint64_t esz = bytes ? 1 : 2;
  const uint64_t dims[2] = {cols, rows};
  const uint64_t strides[1] = {cols * esz};
  const uint32_t box[2] = {static_cast<uint32_t>(128 / esz), box_rows};
  return make_map(map, ptr, 2, dims, strides, box, bytes);
}

// MXFP8 quantisation of the token rows, once per token (the FP8 layer's
// phase 0 then only moves bytes into expert-sorted order): a lane turns 8
// bf16 into 8 e4m3 (one 16-byte load, one 8-byte store), 4 lanes share a
// 32-group's UE8M0 scale (the exact rule of mx_exponent, csrc/ptx.cuh).
// Launched ahead of the route kernel, which runs as its programmatic
// dependent: the two overlap (the route kernel does not read these rows and
// waits for this grid only before it completes).
__global__ void __launch_bounds__(256) mx_quant_tokens_kernel(const __nv_bfloat16* __restrict__ x, int64_t n8,
                                                              uint8_t* __restrict__ q, uint8_t* __restrict__ sf) {
  pdl_launch_dependents();
  const int4* xv = reinterpret_cast<const int4*>(x);
  for (int64_t c0 = blockIdx.x * (int64_t)blockDim.x; c0 < n8; c0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = c0 + threadIdx.x;  // 8-element chunk (groups never straddle rows: H % 32 == 0)
    int4 v = make_int4(0, 0, 0, 0);
    if (c < n8) v = __ldg(xv + c);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
    float f[8];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 t2 = __bfloat1622float2(h2[t]);
      f[2 * t] = t2.x;
      f[2 * t + 1] = t2.y;
    }
    uint32_t am = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) am = max(am, __float_as_uint(fabsf(f[t])));
    am = max(am, __shfl_xor_sync(0xffffffffu, am, 1));
    am = max(am, __shfl_xor_sync(0xffffffffu, am, 2));
    const int ex = mx_exponent(am);
    const float inv = mx_inv_scale(ex);
    uint2 qv;
    qv.x = static_cast<uint32_t>(e4m3x2_from_float(f[0] * inv, f[1] * inv)) |
           (static_cast<uint32_t>(e4m3x2_from_float(f[2] * inv, f[3] * inv)) << 16);
    qv.y = static_cast<uint32_t>(e4m3x2_from_float(f[4] * inv, f[5] * inv)) |
           (static_cast<uint32_t>(e4m3x2_from_float(f[6] * inv, f[7] * inv)) << 16);
    if (c < n8) {
      reinterpret_cast<uint2*>(q)[c] = qv;
      if ((threadIdx.x & 3) == 0) sf[c >> 2] = static_cast<uint8_t>(ex + 127);
    }
  }
}

cudaError_t launch_mx_quant_tokens(const void* x, int64_t S, int32_t H, uint8_t* q, uint8_t* sf,
                                   cudaStream_t stream) {
  const int64_t n8 = S * H / 8;
  if (n8 == 0) return cudaSuccess;
  // leave SMs free so the route block (its programmatic dependent) becomes resident at once
  const int64_t want = (n8 + 255) / 256;
  const int blocks = static_cast<int>(want < 96 ? want : 96);
  mx_quant_tokens_kernel<<<blocks, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(x), n8, q, sf);
  return cudaGetLastError();
}

int64_t config_smem_bytes(int bm, int ttn, int stg, int mode, bool fp8, int kps) {
  if (bm < 1 || bm > kMaxBm || (ttn != 128 && ttn != 256 && ttn != 512) || stg < 1 || stg > kMaxStages)
    return 0;
  if (mode != kModeFused && mode != kModeSplit) return 0;
  if (kps != 1 && (kps != 2 && kps != 4)) return 0;
  // TMEM: the phase-1 accumulator (ttn/128 tiles of bm_mma columns) within 512 columns
  if ((ttn >= 256 ? ttn / 128 : 1) * bm_mma_host(bm) > 512) return 0;
  if (fp8 && bm_mma_host(bm) > 128) return 0;
  const int b = moe_smem_bytes(bm, ttn, stg, mode, fp8, kps);
  return b <= kSmemLimit ? b : 0;
}

static int sm_count_cached() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static bool build_maps(const MoeLaunch& l, MoeMaps& maps) {
  bool ok = true;
  if (!l.fp8) {
    for (int i = 0; i < 5; ++i) {
      ok = ok && make_map_2d(&maps.xs[i], l.x_sorted, l.rows, l.H, 16u << i);
      ok = ok && make_map_2d(&maps.act[i], l.act_g, l.rows, l.I, 16u << i);
    }
    for (int i = 0; i < 3; ++i) {
      // W1 viewed as [2E][I][H]: plane 2e = gate rows, 2e+1 = up rows of expert e
      const uint64_t dims[3] = {(uint64_t)l.H, (uint64_t)l.I, 2ull * l.E};
      const uint64_t strides[2] = {(uint64_t)l.H * 2, (uint64_t)l.I * l.H * 2};
      const uint32_t box[3] = {64, 64u << i, 2};
      ok = ok && ((l.I % (64 << i)) != 0 || make_map(&maps.w1[i], l.w1, 3, dims, strides, box));
    }
    ok = ok && make_map_2d(&maps.w2, l.w2, (uint64_t)l.E * l.H, l.I, 128);
    {  // token rows straight from x (TMA gather4, decode-size blocks), row-strided
      const uint64_t dims[2] = {(uint64_t)l.H, (uint64_t)l.S};
      const uint64_t strides[1] = {l.x_stride ? (uint64_t)l.x_stride : (uint64_t)l.H * 2};
      const uint32_t box[2] = {64, 1};
      ok = ok && make_map(&maps.x, l.x, 2, dims, strides, box);
    }
  } else {
    for (int i = 0; i < 4; ++i) {
      ok = ok && make_map_2d(&maps.xq[i], l.x_q, l.rows, l.H, 16u << i, true);
      ok = ok && make_map_2d(&maps.actq[i], l.act_q, l.rows, l.I, 16u << i, true);
    }
    for (int i = 0; i < 2; ++i) {
      const uint64_t dims[3] = {(uint64_t)l.H, (uint64_t)l.I, 2ull * l.E};
      const uint64_t strides[2] = {(uint64_t)l.H, (uint64_t)l.I * l.H};
      const uint32_t box[3] = {128, 128u << i, 2};
      ok = ok && ((l.I % (128 << i)) != 0 || make_map(&maps.w1q[i], l.w1, 3, dims, strides, box, true));
    }
    ok = ok && make_map_2d(&maps.w2q, l.w2, (uint64_t)l.E * l.H, l.I, 128, true);
  }
  return ok;
}

template <bool kFp8>
static cudaError_t set_attrs() {
  static bool done = false;
  if (done) return cudaSuccess;
  cudaError_t err =
      cudaFuncSetAttribute(fused_moe_kernel<kFp8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
  if (err != cudaSuccess) return err;
  err = cudaFuncSetAttribute(fused_moe_kernel<kFp8>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (err == cudaSuccess) done = true;
  return err;
}

cudaError_t launch_fused_moe(const MoeLaunch& l, cudaStream_t stream, const char** why) {
  cudaError_t err = l.fp8 ? set_attrs<true>() : set_attrs<false>();
  if (err != cudaSuccess) return err;
  // Tensor maps depend only on pointers and shapes: encode once per
  // (workspace, weights, shape) and reuse (the encoder costs ~1 us per map).
  struct MapKey {
    const void *xs, *act, *w1, *w2, *x;
    int64_t rows, x_stride;
    int32_t S, H, I, E;
    bool fp8;
    bool operator==(const MapKey& o) const {
      return xs == o.xs && act == o.act && w1 == o.w1 && w2 == o.w2 && x == o.x && rows == o.rows &&
             x_stride == o.x_stride && S == o.S &&
             H == o.H && I == o.I && E == o.E && fp8 == o.fp8;
    }
  };
  struct MapEntry {
    MapKey key;
    alignas(64) MoeMaps maps;
    bool used;
  };
  static MapEntry cache[16];
  static int cache_next = 0;
  static std::mutex cache_mu;
  const MapKey key{l.fp8 ? l.x_q : l.x_sorted, l.fp8 ? l.act_q : l.act_g, l.w1, l.w2, l.x, l.rows, l.x_stride,
                   l.S, l.H, l.I, l.E, l.fp8};
  alignas(64) MoeMaps maps;  // copied into the launch's parameter buffer
  bool hit = false;
  {
    std::lock_guard<std::mutex> g(cache_mu);
    for (auto& c : cache)
      if (c.used && c.key == key) {
        maps = c.maps;
        hit = true;
        break;
      }
  }
  if (!hit) {
    if (!build_maps(l, maps)) {
      *why = "cuTensorMapEncodeTiled failed (alignment or driver entry point)";
      return cudaErrorInvalidValue;
    }
    std::lock_guard<std::mutex> g(cache_mu);
    MapEntry& c = cache[cache_next];
    cache_next = (cache_next + 1) % 16;
    c.key = key;
    c.maps = maps;
    c.used = true;
  }
  MoeParams p{};
  p.ctrl = l.ctrl;
  p.sorted_ids = l.sorted_ids;
  p.tile_expert = l.tile_expert;
  p.topk_w = l.topk_w;
  p.out_acc = l.out_acc;
  p.act_g = static_cast<__nv_bfloat16*>(l.act_g);
  p.done = l.done;
  p.job_counter = l.job_counter;
  p.gbar = l.job_counter + 1;
  p.acc_a = l.acc_a;
  p.split_cnt = l.split_cnt;
  p.x = static_cast<const __nv_bfloat16*>(l.x);
  p.x_sorted = static_cast<__nv_bfloat16*>(l.x_sorted);
  p.out = static_cast<__nv_bfloat16*>(l.out);
  p.w1_sf = l.w1_sf;
  p.w2_sf = l.w2_sf;
  p.x_q = static_cast<uint8_t*>(l.x_q);
  p.x_sf = l.x_sf;
  p.act_q = static_cast<uint8_t*>(l.act_q);
  p.act_sf = l.act_sf;
  p.xq_in = l.xq_in;
  p.xsf_in = l.xsf_in;
  // token-row strides: of xq_in when the tokens come pre-quantised, else of x
  const int64_t x_dense = l.xq_in ? l.H : 2 * (int64_t)l.H;
  p.x_row16 = (l.x_stride ? l.x_stride : x_dense) / 16;
  p.sf_row4 = (l.sf_stride ? l.sf_stride : l.H / 32) / 4;
  p.w_stride = l.w_stride;
  p.table = l.table;
  p.S = l.S;
  p.H = l.H;
  p.I = l.I;
  p.E = l.E;
  p.top_k = l.top_k;
  p.n_assign = l.S * l.top_k;
  p.prof = g_prof_buffer;
  // Programmatic dependent launch: the megakernel's prologue (barrier init,
  // TMEM allocation, descriptor prefetch) may overlap the route kernel's tail.
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sm_count_cached());
  cfg.blockDim = dim3(kMoeThreads);
  cfg.dynamicSmemBytes = kSmemLimit;
  cfg.stream = stream;
  cfg.attrs = pdl;
  cfg.numAttrs = pdl_mode() ? 1 : 0;
  err = l.fp8 ? cudaLaunchKernelEx(&cfg, fused_moe_kernel<true>, maps, p)
              : cudaLaunchKernelEx(&cfg, fused_moe_kernel<false>, maps, p);
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

}  // namespace ramp
