// Host launcher of the persistent fused MoE megakernel: builds the three TMA
// tensor maps (tokens for gather4, W1, W2), then launches one CTA per SM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "fused_moe.cuh"
#include "launch.h"

namespace ramp {

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

// 2D bf16 row-major [rows, cols] map with a (box_cols x box_rows) SW128 box.
static bool make_map_2d(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                        uint32_t box_cols) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int64_t config_smem_bytes(int bm, int ttn, int stg) {
  if (bm < 1 || bm > kMaxBm || (ttn != 256 && ttn != 512) || stg < 1 || stg > kMaxStages) return 0;
  const int b = moe_smem_bytes(bm, ttn, stg);
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

cudaError_t launch_fused_moe_bf16(const MoeLaunch& l, cudaStream_t stream, const char** why) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t err =
        cudaFuncSetAttribute(fused_moe_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (err != cudaSuccess) return err;
    attr_set = true;
  }
  alignas(64) CUtensorMap tm_x, tm_w1, tm_w2;
  if (!make_map_2d(&tm_x, l.x, l.S, l.H, 1, 64) ||
      !make_map_2d(&tm_w1, l.w1, (uint64_t)l.E * 2 * l.I, l.H, 128, 64) ||
      !make_map_2d(&tm_w2, l.w2, (uint64_t)l.E * l.H, l.I, 128, 64)) {
    *why = "cuTensorMapEncodeTiled failed (alignment or driver entry point)";
    return cudaErrorInvalidValue;
  }
  MoeParams p;
  p.ctrl = l.ctrl;
  p.sorted_ids = l.sorted_ids;
  p.tile_expert = l.tile_expert;
  p.topk_w = l.topk_w;
  p.out_acc = l.out_acc;
  p.table = l.table;
  p.S = l.S;
  p.H = l.H;
  p.I = l.I;
  p.E = l.E;
  p.top_k = l.top_k;
  p.n_assign = l.S * l.top_k;
  fused_moe_bf16_kernel<<<sm_count_cached(), kMoeThreads, kSmemLimit, stream>>>(tm_x, tm_w1, tm_w2, p);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  const int64_t n = (int64_t)l.S * l.H;
  int blocks = (int)((n / 4 + 255) / 256);
  if (blocks > 4 * sm_count_cached()) blocks = 4 * sm_count_cached();
  if (blocks < 1) blocks = 1;
  finalize_bf16_kernel<<<blocks, 256, 0, stream>>>(l.out_acc, static_cast<__nv_bfloat16*>(l.out), n);
  return cudaGetLastError();
}

}  // namespace ramp
