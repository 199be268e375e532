// Persistent fused MoE megakernel for sm_100a (north_star (2)).
//
// One work item = (M-tile of bm aligned assignments of one expert) x (stripe
// of n_i = ttn/2 intermediate features).  For each work item one CTA runs the
// paper's three phases without touching HBM in
// between:
//   P1  acc1[ttn x bm] = W1[e][gate|up stripe] . X[gathered tokens]^T
//       TMA (weights, 128x64 SW128 boxes) + TMA gather4 (token rows) ->
//       tcgen05.mma kind::f16, M=128 weight rows, N=bm tokens ("swap-AB":
//       the weights are the M operand so bm can be 4..128), fp32 in TMEM.
//   P2  act = silu(gate) * up, TMEM -> registers -> bf16 in shared memory,
//       written directly in the SW128 K-major layout the next MMA reads.
//   P3  for every 128-row chunk of H: acc3 = W2[e][chunk, stripe] . act^T
//       (double-buffered in TMEM), then the epilogue scales by the top-k
//       weight and scatter-reduces into the fp32 output (red.global.add).
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM
// allocator, w3 spare, w4-7 epilogue (one TMEM lane = one weight row each).
// The tile config (bm, ttn, stg, group_m) is read from device memory, so the
// dispatcher's choice needs no host round trip.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../../include/ramp_b200.h"
#include "launch.h"
#include "ptx.cuh"

namespace ramp {

constexpr int kMoeThreads = 256;
constexpr int kCtrlBytes = 4096;        // barriers + per-tile metadata
constexpr int kSubTileBytes = 128 * 128;  // 128 rows x 64 bf16 (one SW128 box)
constexpr int kMaxStages = 8;
constexpr int kSmemLimit = 232448;      // 227 KB opt-in per CTA on sm_100

__host__ __device__ inline int bm_mma(int bm) { return bm <= 16 ? 16 : (bm + 15) / 16 * 16; }
__host__ __device__ inline int stage_bytes(int bm, int ttn) {
  const int raw = (ttn / 128) * kSubTileBytes + bm_mma(bm) * 128;
  return (raw + 1023) / 1024 * 1024;
}
__host__ __device__ inline int act_bytes(int bm, int ttn) { return bm_mma(bm) * ttn; }
// Total dynamic shared memory (including 1 KB alignment slack); the B200
// counterpart of smem_usage() (ramp/config_space.py:122-124).
__host__ __device__ inline int moe_smem_bytes(int bm, int ttn, int stg) {
  return 1024 + kCtrlBytes + stg * stage_bytes(bm, ttn) + act_bytes(bm, ttn);
}

struct MoeParams {
  const int32_t* ctrl;         // route output: [0] cfg, [1] n_post_pad, [2] n_mtiles
  const int32_t* sorted_ids;   // [n_post_pad]
  const int32_t* tile_expert;  // [n_mtiles]
  const float* topk_w;         // [S*top_k]
  float* out_acc;              // [S, H] fp32, zeroed by the route kernel
  ramp_table_t table;
  int32_t S, H, I, E, top_k, n_assign;
};

struct CtrlSmem {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t acc1_full;
  uint64_t act_full;
  uint64_t acc3_full[2];
  uint64_t acc3_empty[2];
  uint32_t tmem_base;
  int32_t prod_rows[kMaxBm];
  int32_t epi_tok[kMaxBm];
  float epi_w[kMaxBm];
};
static_assert(sizeof(CtrlSmem) <= kCtrlBytes, "control block overflow");

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.0f + __expf(-g)) * u; }

__global__ void __launch_bounds__(kMoeThreads, 1)
    fused_moe_bf16_kernel(const __grid_constant__ CUtensorMap tm_x,
                          const __grid_constant__ CUtensorMap tm_w1,
                          const __grid_constant__ CUtensorMap tm_w2, const MoeParams p) {
  extern __shared__ unsigned char smem_raw[];
  // 1 KB alignment for the SW128 operand tiles.
  const uint32_t raw_addr = smem_u32(smem_raw);
  const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
  unsigned char* base = smem_raw + (base_addr - raw_addr);
  CtrlSmem& cs = *reinterpret_cast<CtrlSmem*>(base);
  const uint32_t ring_addr = base_addr + kCtrlBytes;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // --- runtime tile config chosen by the dispatcher
  const int cfg = p.ctrl[0];
  const int n_post_pad = p.ctrl[1];
  const int bm = p.table.bm[cfg];
  const int ttn = p.table.ttn[cfg];
  const int stg = p.table.stg[cfg];
  const int group_m = p.table.group_m[cfg];
  const int bmN = bm_mma(bm);
  const int nA = ttn / 128;       // M=128 MMA tiles per phase-1 k-block (gate + up halves)
  const int n_i = ttn / 2;        // intermediate features per stripe
  const int stripes = p.I / n_i;
  const int n_mtiles = n_post_pad / bm;
  const int total = n_mtiles * stripes;
  const int kb1 = p.H / 64;       // phase-1 k-blocks
  const int n_hc = p.H / 128;     // phase-3 output chunks
  const int sbytes = stage_bytes(bm, ttn);
  const uint32_t act_addr = ring_addr + stg * sbytes;
  unsigned char* act_ptr = base + kCtrlBytes + stg * sbytes;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_w1);
    tma_prefetch_desc(&tm_w2);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < stg; ++s) {
      mbar_init(smem_u32(&cs.full[s]), 1);
      mbar_init(smem_u32(&cs.empty[s]), 1);
    }
    mbar_init(smem_u32(&cs.acc1_full), 1);
    mbar_init(smem_u32(&cs.act_full), 128);
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&cs.acc3_full[b]), 1);
      mbar_init(smem_u32(&cs.acc3_empty[b]), 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(&cs.tmem_base));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = cs.tmem_base;

  if (warp == 0) {
    // ============================ TMA producer ============================
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    uint32_t stage = 0, phase = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const int m = group_m ? (w % n_mtiles) : (w / stripes);
      const int s = group_m ? (w / n_mtiles) : (w % stripes);
      const int e = p.tile_expert[m];
      const int row0 = m * bm;
      for (int j = lane; j < bmN; j += 32) {
        int tok = 0;
        if (j < bm) {
          const int a = p.sorted_ids[row0 + j];
          if (a < p.n_assign) tok = a / p.top_k;
        }
        cs.prod_rows[j] = tok;
      }
      __syncwarp();
      if (lane == 0) {
        const int gate_row = e * 2 * p.I + s * n_i;
        const int up_row = gate_row + p.I;
        const uint32_t tx1 = nA * kSubTileBytes + bmN * 128;
        for (int kb = 0; kb < kb1; ++kb) {
          const uint32_t full = smem_u32(&cs.full[stage]);
          mbar_wait(smem_u32(&cs.empty[stage]), phase ^ 1);
          mbar_arrive_expect_tx(full, tx1);
          const uint32_t sb = ring_addr + stage * sbytes;
          for (int t = 0; t < nA / 2; ++t) {
            tma_load_2d(sb + t * kSubTileBytes, &tm_w1, full, kb * 64, gate_row + t * 128, pol_w);
            tma_load_2d(sb + (nA / 2 + t) * kSubTileBytes, &tm_w1, full, kb * 64, up_row + t * 128,
                        pol_w);
          }
          const uint32_t xb = sb + nA * kSubTileBytes;
          for (int r = 0; r < bmN; r += 4)
            tma_gather4(xb + r * 128, &tm_x, full, kb * 64, cs.prod_rows[r], cs.prod_rows[r + 1],
                        cs.prod_rows[r + 2], cs.prod_rows[r + 3], pol_x);
          if (++stage == (uint32_t)stg) { stage = 0; phase ^= 1; }
        }
        const uint32_t tx3 = nA * kSubTileBytes;  // n_i/64 == nA boxes of 128 rows
        for (int hc = 0; hc < n_hc; ++hc) {
          const uint32_t full = smem_u32(&cs.full[stage]);
          mbar_wait(smem_u32(&cs.empty[stage]), phase ^ 1);
          mbar_arrive_expect_tx(full, tx3);
          const uint32_t sb = ring_addr + stage * sbytes;
          for (int kk = 0; kk < nA; ++kk)
            tma_load_2d(sb + kk * kSubTileBytes, &tm_w2, full, s * n_i + kk * 64, e * p.H + hc * 128,
                        pol_w);
          if (++stage == (uint32_t)stg) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ============================ MMA issuer =============================
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(128, bmN);
      uint32_t stage = 0, phase = 0, tile_iter = 0;
      uint32_t uses[2] = {0, 0};
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        // acc1 aliases the acc3 buffers: wait until the epilogue drained them
        for (int b = 0; b < 2; ++b)
          if (uses[b]) mbar_wait(smem_u32(&cs.acc3_empty[b]), (uses[b] - 1) & 1);
        tc_fence_after();
        for (int kb = 0; kb < kb1; ++kb) {
          mbar_wait(smem_u32(&cs.full[stage]), phase);
          tc_fence_after();
          const uint32_t sb = ring_addr + stage * sbytes;
          const uint32_t xb = sb + nA * kSubTileBytes;
          for (int t = 0; t < nA; ++t) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              mma_bf16(tmem + t * bmN, sw128_kmajor_desc(sb + t * kSubTileBytes + k * 32),
                       sw128_kmajor_desc(xb + k * 32), idesc, (kb | k) != 0);
            }
          }
          mma_commit(smem_u32(&cs.empty[stage]));
          if (++stage == (uint32_t)stg) { stage = 0; phase ^= 1; }
        }
        mma_commit(smem_u32(&cs.acc1_full));
        mbar_wait(smem_u32(&cs.act_full), tile_iter & 1);
        tc_fence_after();
        for (int hc = 0; hc < n_hc; ++hc) {
          const int b = hc & 1;
          if (uses[b]) mbar_wait(smem_u32(&cs.acc3_empty[b]), (uses[b] - 1) & 1);
          mbar_wait(smem_u32(&cs.full[stage]), phase);
          tc_fence_after();
          const uint32_t sb = ring_addr + stage * sbytes;
          for (int kk = 0; kk < nA; ++kk) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              mma_bf16(tmem + b * bmN, sw128_kmajor_desc(sb + kk * kSubTileBytes + k * 32),
                       sw128_kmajor_desc(act_addr + kk * bmN * 128 + k * 32), idesc, (kk | k) != 0);
            }
          }
          mma_commit(smem_u32(&cs.empty[stage]));
          mma_commit(smem_u32(&cs.acc3_full[b]));
          ++uses[b];
          if (++stage == (uint32_t)stg) { stage = 0; phase ^= 1; }
        }
        ++tile_iter;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ============================ epilogue ===============================
    const int et = threadIdx.x - 128;                       // TMEM lane == weight row
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(et & ~31) << 16);
    uint32_t tile_iter = 0;
    uint32_t uses[2] = {0, 0};
    for (int w = blockIdx.x; w < total; w += gridDim.x) {
      const int m = group_m ? (w % n_mtiles) : (w / stripes);
      const int row0 = m * bm;
      named_bar_sync(1, 128);
      for (int j = et; j < bm; j += 128) {
        const int a = p.sorted_ids[row0 + j];
        const bool valid = a < p.n_assign;
        cs.epi_tok[j] = valid ? a / p.top_k : -1;
        cs.epi_w[j] = valid ? __ldg(p.topk_w + a) : 0.0f;
      }
      named_bar_sync(1, 128);

      // ---- phase 2: SwiGLU into the SW128 K-major act tile
      mbar_wait(smem_u32(&cs.acc1_full), tile_iter & 1);
      tc_fence_after();
      for (int th = 0; th < nA / 2; ++th) {
        const int f = th * 128 + et;  // feature within the stripe == K index of phase 3
        unsigned char* kblk = act_ptr + (f >> 6) * bmN * 128;
        const int chunk = (f & 63) >> 3;
        const int within = (f & 7) * 2;
        for (int j0 = 0; j0 < bmN; j0 += 16) {
          float g[16], u[16];
          tmem_ld16(lane_base + th * bmN + j0, g);
          tmem_ld16(lane_base + (nA / 2 + th) * bmN + j0, u);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int j = j0 + q;
            const __nv_bfloat16 v = __float2bfloat16(silu_mul(g[q], u[q]));
            *reinterpret_cast<__nv_bfloat16*>(kblk + j * 128 + ((chunk ^ (j & 7)) << 4) + within) = v;
          }
        }
      }
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive(smem_u32(&cs.act_full));

      // ---- phase 3 epilogue: weighted scatter-reduce of each H chunk
      for (int hc = 0; hc < n_hc; ++hc) {
        const int b = hc & 1;
        mbar_wait(smem_u32(&cs.acc3_full[b]), uses[b] & 1);
        tc_fence_after();
        float* orow = p.out_acc + hc * 128 + et;
        for (int j0 = 0; j0 < bm; j0 += 16) {
          float v[16];
          tmem_ld16(lane_base + b * bmN + j0, v);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            const int j = j0 + q;
            if (j < bm) {
              const int tok = cs.epi_tok[j];
              if (tok >= 0) red_add_f32(orow + static_cast<size_t>(tok) * p.H, v[q] * cs.epi_w[j]);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(smem_u32(&cs.acc3_empty[b]));
        ++uses[b];
      }
      ++tile_iter;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// fp32 accumulator -> bf16 output.
__global__ void finalize_bf16_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ out,
                                     int64_t n) {
  const int64_t n4 = n / 4;
  const float4* a4 = reinterpret_cast<const float4*>(acc);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = a4[i];
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(out)[i] = pk;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16(acc[i]);
}

}  // namespace ramp
