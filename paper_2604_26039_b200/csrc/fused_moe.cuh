// Persistent fused-MoE megakernel for sm_100a (north_star (2)).
//
// The layer  out[t] = sum_j w[t,j] * W2[e] (silu(W1g[e] x_t) * W1u[e] x_t)
// runs as ONE launch of one CTA per SM that walks a list of jobs.  Phase 0
// gathers the token rows into expert-sorted order (x_sorted; FP8: MXFP8 bytes
// + scale atoms) behind a grid barrier, so every operand tile arrives with a
// single TMA box (token blocks of <= 16 rows skip it: TMA gather4 from x):
//
//   phase 1  acc[ttn x bm] = W1[e][gate|up stripe] . x_sorted[M-tile]^T
//            one 3D TMA box {64, n_i, 2} brings the gate AND up rows of a
//            k-block, one 2D box brings bm token rows; tcgen05.mma kind::f16
//            with M = 128 weight rows, N = bm tokens ("swap-AB", so bm can be
//            4..256), fp32 accumulators in TMEM.
//   phase 2  act = silu(gate) * up   (TMEM -> registers -> bf16)
//   phase 3  acc[128 x bm] = W2[e][h-chunk, :] . act^T, then the epilogue
//            scales by the top-k weight and scatter-reduces into the fp32
//            output with 16-byte vector reductions (red.global.v4.f32).
//
// Two polymorphic modes (a dispatcher-selected config field, in the spirit of
// the paper's "polymorphic modes"):
//   FUSED (mode 0)  one job = (M-tile, I-stripe): all three phases in one CTA,
//                   act kept in shared memory, phase 3 over every H chunk of
//                   the stripe and partial sums reduced across stripes.
//   SPLIT (mode 1)  job A = (M-tile, I-stripe): phases 1-2, act -> L2-resident
//                   global buffer, then a release on done[M-tile];
//                   job B = (M-tile, H-chunk): phase 3 over the full I, gated
//                   by an acquire on done[M-tile] == #stripes.  More, smaller
//                   jobs (better SM fill at decode sizes) and one reduction
//                   per assignment instead of one per stripe.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM
// allocator, w3 spare, w4-11 epilogue (TMEM lane == weight row; warps w and
// w + 4 share a lane quarter and split the columns).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "../../include/ramp_b200.h"

#include "launch.h"
#include "ptx.cuh"

namespace ramp {

// Two groups of 4 epilogue warps (warps 4-7 and 8-11): each TMEM lane
// quarter is read by two warps that split an accumulator's columns, so the
// epilogue (SwiGLU + MXFP8 requantisation, the scatter-reduce) keeps pace
// with the MMAs at large token blocks.
constexpr int kEpiHalves = 2;
constexpr int kEpiThreads = 128 * kEpiHalves;
constexpr int kMoeThreads = 128 + kEpiThreads;
constexpr int kGatherWarps = kMoeThreads / 32 - 2;  // phase 0: every warp but the producer and MMA issuer
constexpr int kCtrlBytes = 4096;                  // barriers + per-job metadata
constexpr int kStageBytesScatter = 16 * 128 * 4;  // 16 tokens x 128 rows fp32 transpose buffer
constexpr int kSubTileBytes = 128 * 128;          // 128 rows x 64 bf16 (one SW128 box)
constexpr int kMaxStages = 12;
constexpr int kSmemLimit = 232448;                // 227 KB opt-in per CTA on sm_100
constexpr int kModeFused = 0;
constexpr int kModeSplit = 1;

__host__ __device__ inline int bm_mma(int bm) { return bm <= 16 ? 16 : (bm + 15) / 16 * 16; }
// One ring stage holds kps consecutive k-blocks: kps x (ttn/128 weight boxes
// of 16 KB) followed by kps token tiles of bm_mma rows x 128 B.  Bigger stages
// raise the per-CTA streaming rate (a CTA completes roughly one stage per
// 0.25 us however small the stage, scripts/hbm_probe.cu), which is what the
// few-CTA decode regime is bound by.
__host__ __device__ inline int stage_bytes(int bm, int ttn, int kps = 1) {
  const int raw = kps * ((ttn >= 256 ? ttn / 128 : 1) * kSubTileBytes + bm_mma(bm) * 128);
  return (raw + 1023) / 1024 * 1024;
}
// FP8 (MXFP8) stages also carry the 512-byte scale-factor atoms of the nA
// weight tiles and of the token tile of each of their kps k-blocks (after all
// operand tiles; split phase 3 uses 2 x kps of them: W2 then act).
__host__ __device__ inline int stage_bytes_fp8(int bm, int ttn, int kps = 1) {
  const int nA = ttn >= 256 ? ttn / 128 : 1;
  const int raw = kps * (nA * kSubTileBytes + bm_mma(bm) * 128 + (nA + 1) * 512);
  return (raw + 1023) / 1024 * 1024;
}
__host__ __device__ inline int act_bytes(int bm, int ttn, int mode) {
  return mode == kModeFused ? bm_mma(bm) * ttn : 0;
}
// Dynamic shared memory of one config (the B200 counterpart of smem_usage(),
// ramp/config_space.py:122-124): 1 KB alignment slack, control block,
// scatter transpose buffer, stg ring stages, fused mode's bf16 act tile.
__host__ __device__ inline int moe_smem_bytes(int bm, int ttn, int stg, int mode, bool fp8 = false, int kps = 1) {
  return 1024 + kCtrlBytes + kStageBytesScatter + stg * (fp8 ? stage_bytes_fp8(bm, ttn, kps) : stage_bytes(bm, ttn, kps)) +
         (fp8 ? 0 : act_bytes(bm, ttn, mode));
}
__host__ __device__ inline int bmn_index(int bmN) { return bmN <= 16 ? 0 : bmN <= 32 ? 1 : bmN <= 64 ? 2 : bmN <= 128 ? 3 : 4; }

struct MoeMaps {
  CUtensorMap xs[5];   // x_sorted [rows, H],  box {64, 16/32/64/128/256}
  CUtensorMap act[5];  // act_g    [rows, I],  box {64, 16/32/64/128/256}
  CUtensorMap w1[3];   // W1 as [2E, I, H],    box {64, n_i, 2} for n_i = 64 / 128 / 256
  CUtensorMap w2;      // W2 as [E*H, I],      box {64, 128}
  CUtensorMap x;       // x [S, H], box {64, 1}: TMA gather4 of token rows (bm <= 16 configs)
  // FP8 path (byte tensors, 128 elements per 128-byte swizzled row)
  CUtensorMap xq[4];   // x_q   [rows, H] e4m3, box {128, 16/32/64/128} (FP8: bm <= 128)
  CUtensorMap actq[4]; // act_q [rows, I] e4m3, box {128, 16/32/64/128}
  CUtensorMap w1q[2];  // W1 e4m3 as [2E, I, H], box {128, n_i, 2} for n_i = 128 / 256
  CUtensorMap w2q;     // W2 e4m3 as [E*H, I],   box {128, 128}
};

struct MoeParams {
  const int32_t* ctrl;         // route output: [0] cfg, [1] n_post_pad, [2] n_mtiles
  const int32_t* sorted_ids;   // [n_post_pad]
  const int32_t* tile_expert;  // [n_mtiles]
  const float* topk_w;         // [S*top_k]
  float* out_acc;              // [S, H] fp32, zeroed by the route kernel
  __nv_bfloat16* act_g;        // [rows, I] split-mode intermediate
  int* done;                   // [n_mtiles] split-mode phase-A completion counters (zeroed by route)
  int* job_counter;            // global job claim counter (zeroed by route)
  int* gbar;                   // [2] grid barriers: rows gathered, all jobs reduced (zeroed by route)
  float* acc_a;                // [rows, 2I] split-K phase-1 partial sums (read and cleared by the finisher)
  int* split_cnt;              // [n_mtiles * stripes] split-K arrival counters (reset by the finisher)
  const __nv_bfloat16* x;      // [S, H] tokens
  __nv_bfloat16* x_sorted;     // [rows, H] expert-sorted token rows (gathered in phase 0)
  __nv_bfloat16* out;          // [S, H] bf16 result
  // FP8 (MXFP8): e4m3 operands + UE8M0 scale atoms [row block][k block][512 B]
  const uint8_t* w1_sf;        // [2E*I/128][H/128][512]
  const uint8_t* w2_sf;        // [E*H/128][I/128][512]
  uint8_t* x_q;                // [rows, H] quantised, expert-sorted tokens (phase 0)
  uint8_t* x_sf;               // [M-tiles][H/128][512]
  uint8_t* act_q;              // [rows, I] quantised SwiGLU activations
  uint8_t* act_sf;             // [M-tiles][I/128][512]
  const uint8_t* xq_in;        // optional: tokens already MXFP8, [S, H] e4m3 (then x is unused)
  const uint8_t* xsf_in;       //           and their scales [S, H/32] UE8M0, row-major
  int64_t x_row16;             // 16-byte chunks between token rows of x / xq_in (H/8 / H/16 when dense)
  int64_t sf_row4;             // 4-byte words between token rows of xsf_in (H/128 when dense)
  int64_t w_stride;            // floats between token rows of topk_w (0: dense [S*top_k])
  ramp_table_t table;
  int32_t S, H, I, E, top_k, n_assign;
  unsigned long long* prof;    // optional per-CTA cycle counters [gridDim][16] (diagnostics)
};

// Start-path stamps (kTsCfg..kTsClaimed) only in -DRAMP_START_STAMPS builds:
// even predicated-off checks in the per-job paths shift the FP8 epilogue's
// register allocation (measured +0.6-0.9 us per layer).
#ifdef RAMP_START_STAMPS
#define START_STAMP(cond, slot)                          \
  do {                                                   \
    if (ts && (cond)) ts[slot] = globaltimer();          \
  } while (0)
#else
#define START_STAMP(cond, slot) \
  do {                          \
  } while (0)
#endif

// Diagnostic counters (cycles, per CTA) written when MoeParams::prof != null.
enum ProfSlot {
  kPrWaitEmpty = 0, kPrIssue, kMmaWaitFull, kMmaWaitAcc, kMmaWaitAct, kEpiWaitAcc, kEpiSwiglu,
  kEpiWaitChunk, kEpiScatter, kTotal, kItems, kEpiMeta, kPrWaitDep,
  kLatTma, kLatRelease, kNumStages,  // RAMP_PROF_LAT builds: stage issue->landed, commit->slot free
  // globaltimer stamps (ns)
  kTsEntry = 16, kTsStart, kTsGathered, kTsProducerDone, kTsEpilogueDone, kTsEndArrive, kTsEndPass, kTsFinal,
  // start path: config known, first job's expert known, first TMA issued, (unused), first acc ready,
  // producer role entered, first job claimed
  kTsCfg, kTsFirstExpert, kTsFirstIssue, kTsUnused27, kTsFirstAcc, kTsRole, kTsClaimed,
  kNumProf = 32
};

struct ProfClock {
  unsigned long long t;
  __device__ __forceinline__ void start() { t = clock64(); }
  __device__ __forceinline__ unsigned long long lap() {
    const unsigned long long n = clock64();
    const unsigned long long d = n - t;
    t = n;
    return d;
  }
};

struct CtrlSmem {
  uint64_t full[kMaxStages];
  uint64_t empty[kMaxStages];
  uint64_t acc_full[2];    // MMA -> epilogue, per TMEM region
  uint64_t acc_empty[2];   // epilogue -> MMA, per TMEM region (split mode)
  uint64_t act_full;       // fused: act tile written
  uint64_t chunk_full[2];  // fused: phase-3 chunk accumulators
  uint64_t chunk_empty[2];
  uint64_t job_full[4];    // dynamic job ring: producer -> MMA + epilogue
  uint64_t job_empty[4];
  int32_t job_slot[4];
  uint32_t tmem_base;
  int32_t fin;  // split-K: this CTA completed the (m, s) reduction
  int32_t epi_tok[256];
  float epi_w[256];
#ifdef RAMP_PROF_LAT
  unsigned long long t_issue[kMaxStages], t_commit[kMaxStages];
#endif
};
static_assert(sizeof(CtrlSmem) <= kCtrlBytes, "control block overflow");

// Kernel-shape fields of one config, packed in a word (staged in smem at entry).
constexpr int kMaxStagedCfgs = 4096;  // 16 KB of the ring
struct CfgFields {
  int bm, ttn, stg, split_k, group_m, mode, kps, h3;
};
__device__ __forceinline__ uint32_t pack_cfg(const ramp_table_t& t, int i) {
  const uint32_t bm = static_cast<uint32_t>(t.bm[i]);            // <= 256: 9 bits
  const uint32_t ttn = static_cast<uint32_t>(t.ttn[i]) >> 7;     // 1, 2, 4
  const uint32_t stg = static_cast<uint32_t>(t.stg[i]);          // <= 15
  const uint32_t sk = static_cast<uint32_t>(t.split_k[i]);       // 1, 2, 4
  const uint32_t gm = t.group_m[i] ? 1u : 0u;
  const uint32_t mode = t.mode ? static_cast<uint32_t>(t.mode[i]) & 1u : static_cast<uint32_t>(kModeFused);
  const int kv = t.kps ? t.kps[i] : 1;
  const uint32_t kps = (kv == 2 || kv == 4) ? static_cast<uint32_t>(kv) : 1u;
  const int hv = t.h3 ? t.h3[i] : 1;
  const uint32_t h3 = (hv == 2 || hv == 4) ? static_cast<uint32_t>(hv) : 1u;
  return (bm & 511u) | (ttn & 7u) << 9 | (stg & 15u) << 12 | (sk & 7u) << 16 | gm << 19 | mode << 20 |
         kps << 21 | h3 << 24;
}
__device__ __forceinline__ CfgFields unpack_cfg(uint32_t w) {
  CfgFields f;
  f.bm = static_cast<int>(w & 511u);
  f.ttn = static_cast<int>((w >> 9) & 7u) << 7;
  f.stg = static_cast<int>((w >> 12) & 15u);
  f.split_k = static_cast<int>((w >> 16) & 7u);
  f.group_m = static_cast<int>((w >> 19) & 1u);
  f.mode = static_cast<int>((w >> 20) & 1u);
  f.kps = static_cast<int>((w >> 21) & 7u);
  f.h3 = static_cast<int>((w >> 24) & 7u);
  return f;
}

// Job decoding, identical in every role.
template <int N>
struct KpsC {
  static constexpr int value = N;
};

// x / d for x >= 0, d > 0 (once per launch): a shift for powers of two (the
// usual bm, stripe and split factors) instead of a ~25-instruction division.
// (BF16 kernel only: in the FP8 kernel the changed register allocation costs
// more in the epilogue than the divisions, measured +0.6-0.9 us per layer)
template <bool kFp8>
__device__ __forceinline__ int pdiv(int x, int d) {
  if constexpr (kFp8) return x / d;
  return (d & (d - 1)) == 0 ? (x >> (__ffs(d) - 1)) : x / d;
}

struct Job {
  int kind;  // 0 = phase 1(+2) of (m, s) [fused: +phase 3], 1 = split phase 3 of (m, hc)
  int m, s, hc;
  int kq;    // split-K slice of the job's reduction dimension (split mode)
};

struct Geometry {
  int mode, bm, bmN, nA, n_i, stripes, n_mtiles, n_hc, kbH, kbI, nJobA, total, group_m, sk, kps;
  int n3, n_hj;  // split phase 3: 128-row H chunks per job (shared act tile), jobs per M-tile
  bool dbl;      // TMEM double buffering across jobs (split mode)
  int dbl_cols;  // jobs whose accumulator fits in this many columns alternate between two buffers
  __device__ __forceinline__ Job job(int j) const {
    Job r;
    if (j < nJobA) {
      const int u = j / sk;  // the sk K-slices of one (m, s) are consecutive jobs
      r.kind = 0;
      r.kq = j % sk;
      r.m = group_m ? (u % n_mtiles) : (u / stripes);
      r.s = group_m ? (u / n_mtiles) : (u % stripes);
      r.hc = 0;
    } else {
      const int jj = j - nJobA, u = jj / sk;
      r.kind = 1;
      r.kq = jj % sk;
      r.m = group_m ? (u % n_mtiles) : (u / n_hj);
      r.hc = group_m ? (u / n_mtiles) : (u % n_hj);  // job index: chunks [hc * n3, hc * n3 + n3)
      r.s = 0;
    }
    return r;
  }
  // TMEM accumulator buffer of the jl-th job of this CTA: jobs whose
  // accumulator fits in dbl_cols columns alternate between buffers 0 and 1
  // (column offset 256), so the epilogue drains one while the MMAs fill the
  // other; wider ones always use buffer 0.  MMA and epilogue roles agree.
  __device__ __forceinline__ int acc_buf(const Job& jb, uint32_t jl) const {
    const int cols = (jb.kind ? n3 : nA) * bmN;
    return dbl && cols <= dbl_cols ? static_cast<int>(jl & 1u) : 0;
  }
  // k-block range [lo, hi) of a job's reduction (H for phase 1, I for phase 3)
  __device__ __forceinline__ int kb_lo(const Job& jb) const { return jb.kq * (jb.kind ? kbI : kbH) / sk; }
  __device__ __forceinline__ int kb_hi(const Job& jb) const { return (jb.kq + 1) * (jb.kind ? kbI : kbH) / sk; }
};

// silu(g) * u; the fast division returns 0 for a huge denominator (g -> -inf),
// which is silu's limit, and its ~2 ulp error is far below the bf16 rounding.
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.0f + __expf(-g)) * u; }

// 4x4 transpose within each lane quad: lane b (= lane & 3) holds x[j] =
// M[b][j] on entry and M[j][b] on exit (two shuffle rounds, 4 shuffles).
__device__ __forceinline__ void quad_transpose(float (&x)[4], int b) {
#pragma unroll
  for (int m = 1; m <= 2; m <<= 1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j & m) continue;
      const bool hi = b & m;
      const float send = hi ? x[j] : x[j + m];
      const float recv = __shfl_xor_sync(0xffffffffu, send, m);
      if (hi) x[j] = recv; else x[j + m] = recv;
    }
  }
}

// Scatter-reduce 16 token columns of a [128 x bm] TMEM accumulator block into
// out (fp32) as 16-byte vector reductions, without shared memory or a
// barrier: thread et holds row h0 + et for tokens j0..j0+15; after scaling by
// the top-k weights, a 4x4 register transpose inside every lane quad gives
// lane 4a+b the rows 4a..4a+3 of its quad for tokens b, b+4, b+8, b+12 --
// four red.global.add.v4.f32 per lane, 128-byte contiguous per token row.
__device__ __forceinline__ void scatter16(const float (&v)[16], int j0, int bm, int et, const CtrlSmem& cs,
                                          float* out, int H, int h0) {
  const int b = et & 3;
  const int hrow = h0 + (et & ~3);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = j0 + 4 * c + j;
      x[j] = v[4 * c + j] * cs.epi_w[q < bm ? q : 0];
    }
    quad_transpose(x, b);
    const int q = j0 + 4 * c + b;
    if (q < bm) {
      const int tok = cs.epi_tok[q];
      if (tok >= 0) red_add_v4_f32(out + static_cast<size_t>(tok) * H + hrow, make_float4(x[0], x[1], x[2], x[3]));
    }
  }
}

template <bool kFp8>
__global__ void __launch_bounds__(kMoeThreads, 1)
    fused_moe_kernel(const __grid_constant__ MoeMaps maps, const MoeParams p) {
  constexpr int kKb = kFp8 ? 128 : 64;  // K elements per 128-byte swizzled row / k-block
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;  // SW128 tiles need 1 KB alignment
  unsigned char* base = smem_raw + (base_addr - raw_addr);
  CtrlSmem& cs = *reinterpret_cast<CtrlSmem*>(base);
  float* tbuf = reinterpret_cast<float*>(base + kCtrlBytes);
  const uint32_t ring_addr = base_addr + kCtrlBytes + kStageBytesScatter;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long* const ts = p.prof ? p.prof + blockIdx.x * kNumProf : nullptr;
  if (ts && threadIdx.x == 0) ts[kTsEntry] = globaltimer();

  // Prologue (overlaps the route kernel's tail under PDL): descriptors,
  // barriers, TMEM.  Nothing here reads the route kernel's outputs.
  if (warp == 0 && lane < 15) {
    // bf16: xs[5], act[5], w1[3], w2, x; fp8: xq[4], actq[4], w1q[2], w2q (contiguous)
    const CUtensorMap* all = kFp8 ? &maps.xq[0] : &maps.xs[0];
    if (!kFp8 || lane < 11) tma_prefetch_desc(all + lane);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(smem_u32(&cs.full[s]), 1);
      mbar_init(smem_u32(&cs.empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&cs.acc_full[b]), 1);
      mbar_init(smem_u32(&cs.acc_empty[b]), kEpiThreads);
      mbar_init(smem_u32(&cs.chunk_full[b]), 1);
      mbar_init(smem_u32(&cs.chunk_empty[b]), kEpiThreads);
    }
    mbar_init(smem_u32(&cs.act_full), kEpiThreads);
    for (int q = 0; q < 4; ++q) {
      mbar_init(smem_u32(&cs.job_full[q]), 1);
      mbar_init(smem_u32(&cs.job_empty[q]), 1 + kEpiThreads);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(smem_u32(&cs.tmem_base));
  // The dispatch table's kernel-shape fields, packed one word per config,
  // staged in the (still unused) ring while the route kernel runs: once the
  // selection is visible the geometry needs no second global round trip.
  uint32_t* const cfg_words = reinterpret_cast<uint32_t*>(base + kCtrlBytes + kStageBytesScatter);
  const bool staged_cfg = p.table.n_cfg <= kMaxStagedCfgs;
  if (staged_cfg)
    for (int i = threadIdx.x; i < p.table.n_cfg; i += blockDim.x) cfg_words[i] = pack_cfg(p.table, i);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = cs.tmem_base;
  pdl_wait();  // the route kernel's selection and alignment are now visible
  // the producer's expert of M-tiles 0..31 (decode-size calls have no
  // others), loaded alongside the selection instead of once per job after it
  // (entries past n_mtiles are never read back)
  const int te_pref = warp == 0 ? __ldcg(p.tile_expert + lane) : 0;
  const int cfg = p.ctrl[0];
  const int n_post_pad = p.ctrl[1];
  if (ts && threadIdx.x == 0) ts[kTsStart] = globaltimer();

  // --- runtime tile config chosen by the dispatcher (no host round trip)
  const CfgFields cf = staged_cfg ? unpack_cfg(cfg_words[cfg]) : unpack_cfg(pack_cfg(p.table, cfg));
  __syncthreads();  // the staged words are dead from here on (the ring is about to be filled)
#ifdef RAMP_START_STAMPS
  if (ts && threadIdx.x == 0) {
    asm volatile("" ::"r"(cf.stg), "r"(n_post_pad));  // stamp after the loads resolved
    ts[kTsCfg] = globaltimer();
  }
#endif
  const int stg = cf.stg;
  Geometry G;
  G.mode = cf.mode;
  G.bm = cf.bm;
  G.bmN = bm_mma(G.bm);
  if (kFp8 && G.bmN > 128) __trap();  // FP8 token blocks are at most 128 rows (one scale atom)
  const int ttn = cf.ttn;
  G.nA = ttn >= 256 ? ttn / 128 : 1;  // ttn = 128: one tile = 64 gate rows + 64 up rows
  G.n_i = ttn / 2;
  G.stripes = pdiv<kFp8>(p.I, G.n_i);
  G.n_mtiles = pdiv<kFp8>(n_post_pad, G.bm);
  G.n_hc = p.H / 128;
  G.kbH = p.H / kKb;
  G.kbI = p.I / kKb;
  G.group_m = cf.group_m;
  G.sk = (G.mode == kModeSplit && cf.split_k > 1) ? cf.split_k : 1;
  G.nJobA = G.n_mtiles * G.stripes * G.sk;
  G.n3 = 1;
  if (!kFp8 && G.mode == kModeSplit) {
    const int h3 = cf.h3;
    if ((h3 == 2 || h3 == 4) && h3 <= G.nA && G.n_hc % h3 == 0) G.n3 = h3;
  }
  G.n_hj = pdiv<kFp8>(G.n_hc, G.n3);
  G.total = G.nJobA + (G.mode == kModeSplit ? G.n_mtiles * G.n_hj * G.sk : 0);
  // every job fits in buffer 0 (columns < 256, disjoint from buffer 1); FP8:
  // buffer 1 (columns 256..) must also stay below the scale-factor columns
  G.dbl = G.mode == kModeSplit && G.nA * G.bmN <= 256;
  G.dbl_cols = kFp8 ? kSfCol - 256 : 256;
  // k-blocks per stage; every job's k-range must split into whole stages
  // (FP8: at most 16 scale atoms per stage)
  G.kps = cf.kps;
  if (G.kps != 2 && G.kps != 4) G.kps = 1;
  if (kFp8 && (G.kps > 2 || G.kps * (G.nA + 1) > 16)) G.kps = 1;  // FP8 roles: kps 1 and 2
  if (pdiv<kFp8>(G.kbH, G.sk) % G.kps != 0 || (G.mode == kModeSplit && pdiv<kFp8>(G.kbI, G.sk) % G.kps != 0)) G.kps = 1;
  const int bmN = G.bmN, nA = G.nA, kps = G.kps;
  const int sbytes = kFp8 ? stage_bytes_fp8(G.bm, ttn, kps) : stage_bytes(G.bm, ttn, kps);
  const int tok_off = kps * nA * kSubTileBytes;  // token tiles follow the stage's weight boxes
  const uint32_t act_addr = ring_addr + stg * sbytes;
  unsigned char* act_ptr = base + kCtrlBytes + kStageBytesScatter + stg * sbytes;
  const CUtensorMap* tm_xs = kFp8 ? &maps.xq[bmn_index(bmN)] : &maps.xs[bmn_index(bmN)];
  const CUtensorMap* tm_act = kFp8 ? &maps.actq[bmn_index(bmN)] : &maps.act[bmn_index(bmN)];
  const CUtensorMap* tm_w1 =
      kFp8 ? &maps.w1q[G.n_i == 256 ? 1 : 0] : &maps.w1[G.n_i == 256 ? 2 : G.n_i == 128 ? 1 : 0];
  const CUtensorMap* tm_w2 = kFp8 ? &maps.w2q : &maps.w2;
  // FP8: scale atoms after the operand tiles; phase 1 atom slot t * kps + q
  // (t < nA: weight tile t, t = nA: tokens; q = k-block within the stage),
  // split phase 3 slot q (W2) and kps + q (act)
  const int sf_off = kps * (nA * kSubTileBytes + bmN * 128);

  // ---- phase 0: gather the token rows of every M-tile into expert-sorted
  // order (warps 2-7 of every CTA, 8 x 16-byte loads in flight per lane),
  // then arrive on grid barrier 0.  The producers stream weights meanwhile
  // and hold back token tiles until all CTAs have arrived.
  // Token blocks of <= 16 rows skip phase 0: their producer gathers the rows
  // straight from x with TMA gather4 (4 rows per instruction), so decode-size
  // calls need no grid barrier before the first MMA.
  const bool direct_x = !kFp8 && bmN == 16;
  if (kFp8 && warp >= 2) {
    // FP8 phase 0, two forms (the host picks by batch size):
    // * the token rows arrive already in MXFP8 (xq_in / xsf_in: the token
    //   quantisation kernel, run once per token ahead of the route kernel for
    //   large batches, or an MXFP8 expert-parallel wire): only move them into
    //   expert-sorted order (x_q, 16-byte chunks) and their row-major scales
    //   into the M-tiles' atoms (x_sf, one k-block per 4-byte word); a warp's
    //   32 rows are flattened into one chunk stream so every lane keeps
    //   kUnroll loads in flight whatever the row length;
    // * small batches: quantise every gathered row here (no extra launch).
    if (p.xq_in != nullptr) {
      constexpr int kUnroll = 16;  // pure copy: 256 B in flight per lane
      const int row16 = p.H / 16;
      const int gw = blockIdx.x * kGatherWarps + (warp - 2), nw = gridDim.x * kGatherWarps;
      const int4* qsrc = reinterpret_cast<const int4*>(p.xq_in);
      for (int r0 = gw; r0 < n_post_pad; r0 += 32 * nw) {
        const int rl = r0 + lane * nw;
        const int asg_l = rl < n_post_pad ? __ldcg(p.sorted_ids + rl) : p.n_assign;
        const int src_l = asg_l < p.n_assign ? asg_l / p.top_k : -1;  // token row, -1 = padding
        const int nrows = min(32, (n_post_pad - r0 + nw - 1) / nw);
        const int nch = nrows * row16;
        for (int b0 = 0; b0 < nch; b0 += 32 * kUnroll) {  // warp-uniform trip count (shuffles inside)
          int4 v[kUnroll];
          int dst_row[kUnroll], cc[kUnroll];
  #pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int c = b0 + lane + 32 * u;
            const int q = min(c / row16, nrows - 1);
            cc[u] = c - q * row16;
            const int src = __shfl_sync(0xffffffffu, src_l, q);
            dst_row[u] = c < nch && src >= 0 ? r0 + q * nw : -1;  // padding rows: never read back
            v[u] = make_int4(0, 0, 0, 0);
            if (c < nch && src >= 0) v[u] = __ldg(qsrc + src * p.x_row16 + cc[u]);
          }
  #pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (dst_row[u] >= 0)
              reinterpret_cast<int4*>(p.x_q + static_cast<int64_t>(dst_row[u]) * p.H)[cc[u]] = v[u];
        }
        const int nsw = nrows * G.kbH;
        for (int b0 = 0; b0 < nsw; b0 += 32) {
          const int c0 = b0 + lane;
          const int q = min(c0 / G.kbH, nrows - 1), kb = c0 - q * G.kbH;
          const int src = __shfl_sync(0xffffffffu, src_l, q);
          if (c0 < nsw) {
            const uint32_t sc =
                src < 0 ? 0u : __ldg(reinterpret_cast<const uint32_t*>(p.xsf_in) + src * p.sf_row4 + kb);
            const int r = r0 + q * nw, m = r / G.bm, jr = r - m * G.bm;
            *reinterpret_cast<uint32_t*>(p.x_sf + (static_cast<int64_t>(m) * G.kbH + kb) * 512 + (jr & 31) * 16 +
                                         (jr >> 5) * 4) = sc;
          }
        }
      }
    } else {
      constexpr int kUnroll = 8;
      const int row_vec = p.H / 8;  // multiple of 16 (H % 128 == 0)
      const int gw = blockIdx.x * kGatherWarps + (warp - 2), nw = gridDim.x * kGatherWarps;
      const int4* xv = reinterpret_cast<const int4*>(p.x);
      for (int r0 = gw; r0 < n_post_pad; r0 += 32 * nw) {
        const int rl = r0 + lane * nw;
        const int asg_l = rl < n_post_pad ? __ldcg(p.sorted_ids + rl) : p.n_assign;
        const int nrows = min(32, (n_post_pad - r0 + nw - 1) / nw);
        for (int q = 0; q < nrows; ++q) {
          const int asg = __shfl_sync(0xffffffffu, asg_l, q);
          // padding rows are skipped: their MMA columns / act rows are never
          // scattered, and every column of an MMA depends only on its own row
          if (asg >= p.n_assign) continue;  // warp-uniform
          const int r = r0 + q * nw;
          const int m = r / G.bm, jr = r - m * G.bm;
          const int4* src = xv + (asg / p.top_k) * p.x_row16;
          uint8_t* dst = p.x_q + static_cast<int64_t>(r) * p.H;
          uint8_t* sf_row = p.x_sf + static_cast<int64_t>(m) * G.kbH * 512 + (jr & 31) * 16 + (jr >> 5) * 4;
          for (int c0 = lane; c0 < row_vec; c0 += 32 * kUnroll) {
            int4 v[kUnroll];
  #pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              v[u] = make_int4(0, 0, 0, 0);
              if (c0 + 32 * u < row_vec && asg < p.n_assign) v[u] = __ldg(src + c0 + 32 * u);
            }
  #pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
              const int c = c0 + 32 * u;
              if (c - lane >= row_vec) break;  // warp-uniform
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
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
              const bool in = c < row_vec;  // row_vec may be an odd multiple of 16
              if (in) *reinterpret_cast<uint2*>(dst + c * 8) = qv;
              // the 4 group exponents of this lane's k-block (lanes 16h .. 16h+15)
              const int b16 = lane & 16;
              const uint32_t e0 = __shfl_sync(0xffffffffu, ex + 127, b16);
              const uint32_t e1 = __shfl_sync(0xffffffffu, ex + 127, b16 + 4);
              const uint32_t e2 = __shfl_sync(0xffffffffu, ex + 127, b16 + 8);
              const uint32_t e3 = __shfl_sync(0xffffffffu, ex + 127, b16 + 12);
              if (in && (lane & 15) == 0)
                *reinterpret_cast<uint32_t*>(sf_row + static_cast<int64_t>(c >> 4) * 512) =
                    e0 | (e1 << 8) | (e2 << 16) | (e3 << 24);
            }
          }
        }
      }
    }
    __threadfence();
    named_bar_sync(2, 32 * kGatherWarps);
    if (warp == 2 && lane == 0) atomicAdd(p.gbar, 1);
  }
  if (!kFp8 && warp >= 2 && !direct_x) {
    constexpr int kUnroll = 8;
    const int row_vec = p.H / 8;  // 16-byte vectors per row
    const int gw = blockIdx.x * kGatherWarps + (warp - 2), nw = gridDim.x * kGatherWarps;
    const int4* xv = reinterpret_cast<const int4*>(p.x);
    int4* dv = reinterpret_cast<int4*>(p.x_sorted);
    // This warp's rows are gw, gw + nw, ...: one coalesced load fetches the
    // assignments of the next 32 of them (no per-row dependent load), and two
    // rows move per iteration (16 x 16 B in flight per lane).
    for (int r0 = gw; r0 < n_post_pad; r0 += 32 * nw) {
      const int rl = r0 + lane * nw;
      const int asg_l = rl < n_post_pad ? __ldcg(p.sorted_ids + rl) : p.n_assign;
      const int nrows = min(32, (n_post_pad - r0 + nw - 1) / nw);
      for (int q = 0; q < nrows; q += 2) {
        const int a0 = __shfl_sync(0xffffffffu, asg_l, q);
        const int a1 = __shfl_sync(0xffffffffu, asg_l, (q + 1) & 31);
        const bool two = q + 1 < nrows;
        const int4* s0 = xv + (a0 < p.n_assign ? a0 / p.top_k : 0) * p.x_row16;
        const int4* s1 = xv + (a1 < p.n_assign ? a1 / p.top_k : 0) * p.x_row16;
        int4* d0 = dv + static_cast<int64_t>(r0 + q * nw) * row_vec;
        int4* d1 = dv + static_cast<int64_t>(r0 + (q + 1) * nw) * row_vec;
        for (int c0 = lane; c0 < row_vec; c0 += 32 * kUnroll) {
          int4 v0[kUnroll], v1[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const bool in = c0 + 32 * u < row_vec;
            v0[u] = v1[u] = make_int4(0, 0, 0, 0);
            if (in && a0 < p.n_assign) v0[u] = __ldg(s0 + c0 + 32 * u);
            if (in && two && a1 < p.n_assign) v1[u] = __ldg(s1 + c0 + 32 * u);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            if (c0 + 32 * u < row_vec) {  // padding rows are skipped (never read back)
              if (a0 < p.n_assign) d0[c0 + 32 * u] = v0[u];
              if (two && a1 < p.n_assign) d1[c0 + 32 * u] = v1[u];
            }
          }
        }
      }
    }
    __threadfence();
    named_bar_sync(2, 32 * kGatherWarps);
    if (warp == 2 && lane == 0) atomicAdd(p.gbar, 1);
  }

  if (warp == 0) {
    auto role = [&](auto kc) {
    // ============================ TMA producer ============================
    // The whole warp walks the schedule (so every operand is warp-uniform and
    // stays on the uniform datapath); one elected lane issues each TMA.
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    const int u_stg = warp_uniform(stg), u_sbytes = warp_uniform(sbytes);
    constexpr int u_kps = decltype(kc)::value;  // compile-time: runtime trip counts slow the issue loops
    const int u_tok = warp_uniform(tok_off);
    uint32_t stage = 0, phase = 0;
    unsigned long long c_wait = 0, c_issue = 0, c_dep = 0, t_begin = clock64();
    ProfClock pc;
    pc.start();
    auto next = [&]() {
#ifdef RAMP_PROF_LAT
      if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&cs.t_issue[stage]) = clock64();
#endif
      if (++stage == (uint32_t)u_stg) {
        stage = 0;
        phase ^= 1;
      }
    };
#ifdef RAMP_PROF_LAT
    unsigned long long c_rel = 0;
#endif
    auto acquire = [&]() {
      c_issue += pc.lap();
      mbar_wait(smem_u32(&cs.empty[stage]), phase ^ 1);
      c_wait += pc.lap();
#ifdef RAMP_PROF_LAT
      if (phase) c_rel += clock64() - *reinterpret_cast<volatile unsigned long long*>(&cs.t_commit[stage]);
#endif
    };
    uint32_t js = 0, jph = 0;
    bool first_job = true, first_stamp = true;
    START_STAMP(lane == 0, kTsRole);
    // direct_x gathers its token rows straight from x (no phase-0 barrier)
    bool gathered = direct_x;
    while (true) {
      // claim the next job (dynamic, in global order) and publish it to the ring
      // the first job is static (job = CTA index: no claim round trip before
      // the first loads); later ones are claimed past the static wave
      int j = static_cast<int>(blockIdx.x);
      if (!first_job && lane == 0) j = static_cast<int>(gridDim.x) + atomicAdd(p.job_counter, 1);
      first_job = false;
      j = warp_uniform(j);
      if (j >= G.total) j = -1;
      mbar_wait(smem_u32(&cs.job_empty[js]), jph ^ 1);
      if (elect_one()) {
        cs.job_slot[js] = j;
        mbar_arrive(smem_u32(&cs.job_full[js]));
      }
      __syncwarp();
      if (++js == 4) { js = 0; jph ^= 1; }
      if (j < 0) break;
      START_STAMP(lane == 0 && first_stamp, kTsClaimed);
      const Job jb = G.job(j);
      const int e = warp_uniform(jb.m < 32 ? __shfl_sync(0xffffffffu, te_pref, jb.m) : __ldcg(p.tile_expert + jb.m));
#ifdef RAMP_START_STAMPS
      if (ts && lane == 0 && first_stamp) {
        asm volatile("" ::"r"(e));
        ts[kTsFirstExpert] = globaltimer();
      }
#endif
      const int row0 = jb.m * G.bm;
      if (jb.kind == 0) {
        // direct_x gathers only the token block's bm rows (4 per gather4): the
        // MMA's padding columns bm..15 read stale shared memory, and column n
        // of the product depends on token row n alone, so every consumer
        // (SwiGLU stores, split-K partials, scatter) stops at bm
        const int n_g4 = direct_x ? warp_uniform(min(16, (G.bm + 3) & ~3)) : 16;
        const uint32_t tx1 = u_kps * (nA * kSubTileBytes + (direct_x ? n_g4 : bmN) * 128 + (kFp8 ? (nA + 1) * 512 : 0));
        const int wrow = jb.s * G.n_i;
        const int kb0 = G.kb_lo(jb), kb1 = G.kb_hi(jb);
        int first_pending = 0, npend = 0;
        int trow[16];  // direct_x: token row of each of the 16 MMA columns
        bool have_trow = false;
        auto ensure_trow = [&]() {  // whole warp; only once sorted_ids are final
          if (!direct_x || have_trow) return;
          int mine = 0;
          if (lane < G.bm) {
            const int a = __ldcg(p.sorted_ids + row0 + lane);
            mine = a < p.n_assign ? a / p.top_k : 0;
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) trow[q] = __shfl_sync(0xffffffffu, mine, q);
          have_trow = true;
        };
        auto gather_tokens = [&](uint32_t sb, uint32_t full, int kb) {  // direct_x token loads of one stage
          for (int u = 0; u < u_kps; ++u) {
#pragma unroll
            for (int q = 0; q < 16; q += 4)
              if (q < n_g4)  // (constant trow indices: the array stays in registers)
                tma_gather4(sb + u_tok + u * 16 * 128 + q * 128, &maps.x, full, (kb + u) * 64, trow[q], trow[q + 1],
                          trow[q + 2], trow[q + 3], pol_x);
          }
        };
        if (gathered) ensure_trow();
        // token-side loads of one stage (tiles + FP8 scale atom), deferrable
        auto load_tokens = [&](uint32_t sb, uint32_t full, int kb) {
          for (int q = 0; q < u_kps; ++q)
            tma_load_2d(sb + u_tok + q * bmN * 128, tm_xs, full, (kb + q) * kKb, row0, pol_x);
          if constexpr (kFp8)
            bulk_g2s(sb + sf_off + nA * u_kps * 512, p.x_sf + (static_cast<int64_t>(jb.m) * G.kbH + kb) * 512,
                     u_kps * 512, full);
        };
        START_STAMP(lane == 0 && first_stamp, kTsFirstIssue);  // first stage slot is free
        first_stamp = false;
        for (int kb = kb0; kb < kb1; kb += u_kps) {
          acquire();
          if (elect_one()) {
            const uint32_t full = smem_u32(&cs.full[stage]);
            const uint32_t sb = ring_addr + stage * u_sbytes;
            mbar_arrive_expect_tx(full, tx1);
            for (int q = 0; q < u_kps; ++q)
              tma_load_3d(sb + q * nA * kSubTileBytes, tm_w1, full, (kb + q) * kKb, wrow, 2 * e, pol_w);
            if constexpr (kFp8) {
              for (int t = 0; t < nA; ++t) {
                const int half = nA / 2;
                const int64_t rb = (static_cast<int64_t>(e) * 2 * p.I + (t < half ? 0 : p.I) + wrow +
                                    (t % half) * 128) / 128;
                bulk_g2s(sb + sf_off + t * u_kps * 512, p.w1_sf + (rb * G.kbH + kb) * 512, u_kps * 512, full);
              }
            }
            if (gathered) {
              if (direct_x) gather_tokens(sb, full, kb);
              else load_tokens(sb, full, kb);
            }
          }
          __syncwarp();
          if (!gathered) {
            // weights stream while phase 0 finishes; token rows follow once
            // every CTA has published its slice of x_sorted
            if (npend == 0) first_pending = kb;
            ++npend;
            if (npend == u_stg || kb + u_kps >= kb1) {
              pc.lap();
              while (ld_acquire_gpu(p.gbar) < (int)gridDim.x) __nanosleep(32);
              fence_proxy_async_global();
              c_dep += pc.lap();
              gathered = true;
              ensure_trow();
              if (ts && lane == 0) ts[kTsGathered] = globaltimer();
              if (elect_one()) {
                for (int q = 0; q < npend; ++q) {
                  const uint32_t st = (stage + u_stg - (npend - 1) + q) % u_stg;
                  if (direct_x) gather_tokens(ring_addr + st * u_sbytes, smem_u32(&cs.full[st]), first_pending + q * u_kps);
                  else load_tokens(ring_addr + st * u_sbytes, smem_u32(&cs.full[st]), first_pending + q * u_kps);
                }
              }
              __syncwarp();
            }
          }
          next();
        }
        if (G.mode == kModeFused) {
          for (int hc = 0; hc < G.n_hc; ++hc) {
            acquire();
            if (elect_one()) {
              const uint32_t full = smem_u32(&cs.full[stage]);
              const uint32_t sb = ring_addr + stage * u_sbytes;
              mbar_arrive_expect_tx(full, nA * kSubTileBytes);  // n_i/64 == nA boxes
              for (int kk = 0; kk < nA; ++kk)
                tma_load_2d(sb + kk * kSubTileBytes, tm_w2, full, jb.s * G.n_i + kk * 64, e * p.H + hc * 128,
                            pol_w);
            }
            __syncwarp();
            next();
          }
        }
      } else {
        // Split phase 3: weights stream immediately; the act rows wait for
        // every phase-1 job of this M-tile (release/acquire on done[m]).
        const int n3 = warp_uniform(G.n3);
        const uint32_t tx = u_kps * (n3 * kSubTileBytes + bmN * 128 + (kFp8 ? 2 * 512 : 0));
        const int wrow = e * p.H + jb.hc * n3 * 128;
        const int kb0 = G.kb_lo(jb), kb1 = G.kb_hi(jb);
        // act tiles sit after the stage's weight area
        const int a_off = u_tok;
        int first_pending = 0, npend = 0;
        bool ready = false;
        // Pull this job's whole W2 slice toward L2 now: while the act rows are
        // still being produced by the phase-1 jobs, HBM keeps streaming weights,
        // and once the dependency resolves the slice arrives from L2.
        if (ld_acquire_gpu(p.done + jb.m) < G.stripes) {
          for (int t = 0; t < n3; ++t)
            for (int kb = kb0 + u_stg * u_kps + lane; kb < kb1; kb += 32) tma_prefetch_2d(tm_w2, kb * kKb, wrow + t * 128);
        }
        __syncwarp();
        auto load_act = [&](uint32_t sb, uint32_t full, int kb) {
          for (int q = 0; q < u_kps; ++q)
            tma_load_2d(sb + a_off + q * bmN * 128, tm_act, full, (kb + q) * kKb, row0, pol_x);
          if constexpr (kFp8)
            bulk_g2s(sb + sf_off + u_kps * 512, p.act_sf + (static_cast<int64_t>(jb.m) * G.kbI + kb) * 512,
                     u_kps * 512, full);
        };
        for (int kb = kb0; kb < kb1; kb += u_kps) {
          acquire();
          if (elect_one()) {
            const uint32_t full = smem_u32(&cs.full[stage]);
            const uint32_t sb = ring_addr + stage * u_sbytes;
            mbar_arrive_expect_tx(full, tx);
            if (n3 == 1) {  // the common case keeps its compile-time trip count
              for (int q = 0; q < u_kps; ++q)
                tma_load_2d(sb + q * kSubTileBytes, tm_w2, full, (kb + q) * kKb, wrow, pol_w);
            } else {
              for (int q = 0; q < u_kps; ++q)
                for (int t = 0; t < n3; ++t)
                  tma_load_2d(sb + (q * n3 + t) * kSubTileBytes, tm_w2, full, (kb + q) * kKb, wrow + t * 128, pol_w);
            }
            if constexpr (kFp8)
              bulk_g2s(sb + sf_off, p.w2_sf + (static_cast<int64_t>(wrow / 128) * G.kbI + kb) * 512, u_kps * 512, full);
            if (ready) load_act(sb, full, kb);
          }
          __syncwarp();
          if (!ready) {
            if (npend == 0) first_pending = kb;
            ++npend;
            if (npend == u_stg || kb + u_kps >= kb1) {
              pc.lap();
              while (ld_acquire_gpu(p.done + jb.m) < G.stripes) __nanosleep(64);
              fence_proxy_async_global();
              c_dep += pc.lap();
              ready = true;
              if (elect_one()) {
                // the pending k-blocks sit in the npend stages ending at `stage`
                for (int q = 0; q < npend; ++q) {
                  const uint32_t st = (stage + u_stg - (npend - 1) + q) % u_stg;
                  load_act(ring_addr + st * u_sbytes, smem_u32(&cs.full[st]), first_pending + q * u_kps);
                }
              }
              __syncwarp();
            }
          }
          next();
        }
      }
    }
    if (p.prof && lane == 0) {
      unsigned long long* pr = p.prof + blockIdx.x * kNumProf;
      pr[kTsProducerDone] = globaltimer();
      pr[kPrWaitEmpty] = c_wait;
      pr[kPrIssue] = c_issue + pc.lap();
      pr[kPrWaitDep] = c_dep;
      pr[kTotal] = clock64() - t_begin;
#ifdef RAMP_PROF_LAT
      pr[kLatRelease] = c_rel;
#endif
    }
    };
    // kps is chosen on the device per call: one compiled copy of the role per
    // value (a runtime trip count in these loops costs ~30 % of the issue rate)
    if (!kFp8 && kps == 4) {
      role(KpsC<4>{});
    } else if (kps == 2) {
      role(KpsC<2>{});
    } else {
      role(KpsC<1>{});
    }
  } else if (warp == 1) {
    auto role = [&](auto kc) {
    // ============================ MMA issuer =============================
    // Whole warp iterates; one elected lane issues the tcgen05 instructions.
    const uint32_t idesc = idesc_bf16(128, warp_uniform(bmN));
    const int u_stg = warp_uniform(stg), u_sbytes = warp_uniform(sbytes);
    constexpr int u_kps = decltype(kc)::value;  // compile-time: runtime trip counts slow the issue loops
    const int u_tok = warp_uniform(tok_off);
    const uint32_t u_tmem = warp_uniform(tmem);
    const uint64_t act_desc = sw128_kmajor_desc(act_addr);
    const int a_step = warp_uniform(bmN) * 128 >> 4;  // act K-block stride in descriptor units
    uint32_t stage = 0, phase = 0, jl = 0, act_iter = 0;
    uint32_t acc_cnt[2] = {0, 0}, chunk_cnt[2] = {0, 0};
    unsigned long long c_full = 0, c_acc = 0, c_act = 0, items = 0;
    ProfClock pc;
    pc.start();
#ifdef RAMP_PROF_LAT
    unsigned long long c_lat = 0, n_st = 0;
#endif
    auto wait_full = [&]() -> uint32_t {
      pc.lap();
      mbar_wait(smem_u32(&cs.full[stage]), phase);
      c_full += pc.lap();
#ifdef RAMP_PROF_LAT
      c_lat += clock64() - *reinterpret_cast<volatile unsigned long long*>(&cs.t_issue[stage]);
      ++n_st;
#endif
      tc_fence_after();
      return ring_addr + stage * u_sbytes;
    };
    auto release = [&]() {
      if (elect_one()) mma_commit(smem_u32(&cs.empty[stage]));
#ifdef RAMP_PROF_LAT
      if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&cs.t_commit[stage]) = clock64();
#endif
      __syncwarp();
      if (++stage == (uint32_t)u_stg) {
        stage = 0;
        phase ^= 1;
      }
    };
    uint32_t js = 0, jph = 0;
    for (;; ++jl) {
      mbar_wait(smem_u32(&cs.job_full[js]), jph);
      const int j = warp_uniform(cs.job_slot[js]);
      if (elect_one()) mbar_arrive(smem_u32(&cs.job_empty[js]));
      __syncwarp();
      if (++js == 4) { js = 0; jph ^= 1; }
      if (j < 0) break;
      ++items;
      const Job jb = G.job(j);
      const int r = G.acc_buf(jb, jl);
      const uint32_t acc = u_tmem + r * 256;
      pc.lap();
      if (G.mode == kModeSplit) {
        if (acc_cnt[r]) mbar_wait(smem_u32(&cs.acc_empty[r]), (acc_cnt[r] - 1) & 1);
      } else {
        for (int b = 0; b < 2; ++b)
          if (chunk_cnt[b]) mbar_wait(smem_u32(&cs.chunk_empty[b]), (chunk_cnt[b] - 1) & 1);
      }
      c_acc += pc.lap();
      tc_fence_after();
      const int kb0 = G.kb_lo(jb), kb1 = G.kb_hi(jb);
      if (jb.kind == 0) {
        for (int kb = kb0; kb < kb1; kb += u_kps) {
          const uint32_t sb = wait_full();
          const uint64_t da = sw128_kmajor_desc(sb);
          const uint64_t db = sw128_kmajor_desc(sb + u_tok);
          if (elect_one()) {
            if constexpr (kFp8) {
              // scale atoms smem -> TMEM; in-order with the MMAs that read them
              const int n_atoms = (nA + 1) * u_kps;
              for (int a = 0; a < n_atoms; ++a) tmem_cp_sf(u_tmem + kSfCol + 4 * a, sf_atom_desc(sb + sf_off + a * 512));
              for (int q = 0; q < u_kps; ++q)
                for (int t = 0; t < nA; ++t) {
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_mxf8(acc + t * bmN, da + ((((q * nA + t) * kSubTileBytes) + k * 32) >> 4),
                             db + ((q * bmN * 128 + k * 32) >> 4), idesc_mxf8(128, bmN, k), ((kb - kb0) | q | k) != 0,
                             (uint32_t(k) << 30) | (u_tmem + kSfCol + 4 * (t * u_kps + q)),
                             (uint32_t(k) << 30) | (u_tmem + kSfCol + 4 * (nA * u_kps + q)));
                }
            } else {
              for (int q = 0; q < u_kps; ++q)
                for (int t = 0; t < nA; ++t) {
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_bf16(acc + t * bmN, da + ((((q * nA + t) * kSubTileBytes) + k * 32) >> 4),
                             db + ((q * bmN * 128 + k * 32) >> 4), idesc, ((kb - kb0) | q | k) != 0);
                }
            }
          }
          __syncwarp();
          release();
        }
        if (elect_one()) mma_commit(smem_u32(&cs.acc_full[r]));
        __syncwarp();
        ++acc_cnt[r];
        if (G.mode == kModeFused) {
          pc.lap();
          mbar_wait(smem_u32(&cs.act_full), act_iter & 1);
          c_act += pc.lap();
          ++act_iter;
          tc_fence_after();
          for (int hc = 0; hc < G.n_hc; ++hc) {
            const int b = hc & 1;
            pc.lap();
            if (chunk_cnt[b]) mbar_wait(smem_u32(&cs.chunk_empty[b]), (chunk_cnt[b] - 1) & 1);
            c_acc += pc.lap();
            const uint32_t sb = wait_full();
            const uint64_t da = sw128_kmajor_desc(sb);
            if (elect_one()) {
              for (int kk = 0; kk < nA; ++kk) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16(u_tmem + b * bmN, da + ((kk * kSubTileBytes + k * 32) >> 4),
                           act_desc + kk * a_step + ((k * 32) >> 4), idesc, (kk | k) != 0);
              }
            }
            __syncwarp();
            release();
            if (elect_one()) mma_commit(smem_u32(&cs.chunk_full[b]));
            __syncwarp();
            ++chunk_cnt[b];
          }
        }
      } else {
        const int n3 = warp_uniform(G.n3);
        for (int kb = kb0; kb < kb1; kb += u_kps) {
          const uint32_t sb = wait_full();
          const uint64_t da = sw128_kmajor_desc(sb);
          const uint64_t db = sw128_kmajor_desc(sb + u_tok);
          if (elect_one()) {
            if constexpr (kFp8) {
              for (int a = 0; a < 2 * u_kps; ++a) tmem_cp_sf(u_tmem + kSfCol + 4 * a, sf_atom_desc(sb + sf_off + a * 512));
              for (int q = 0; q < u_kps; ++q) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_mxf8(acc, da + ((q * kSubTileBytes + k * 32) >> 4), db + ((q * bmN * 128 + k * 32) >> 4),
                           idesc_mxf8(128, bmN, k), ((kb - kb0) | q | k) != 0,
                           (uint32_t(k) << 30) | (u_tmem + kSfCol + 4 * q),
                           (uint32_t(k) << 30) | (u_tmem + kSfCol + 4 * (u_kps + q)));
              }
            } else if (n3 == 1) {  // the common case keeps its compile-time trip count
              for (int q = 0; q < u_kps; ++q) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16(acc, da + ((q * kSubTileBytes + k * 32) >> 4), db + ((q * bmN * 128 + k * 32) >> 4), idesc,
                           ((kb - kb0) | q | k) != 0);
              }
            } else {
              for (int q = 0; q < u_kps; ++q)
                for (int t = 0; t < n3; ++t) {
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_bf16(acc + t * bmN, da + ((((q * n3 + t) * kSubTileBytes) + k * 32) >> 4),
                             db + ((q * bmN * 128 + k * 32) >> 4), idesc, ((kb - kb0) | q | k) != 0);
                }
            }
          }
          __syncwarp();
          release();
        }
        if (elect_one()) mma_commit(smem_u32(&cs.acc_full[r]));
        __syncwarp();
        ++acc_cnt[r];
      }
    }
    if (p.prof && lane == 0) {
      unsigned long long* pr = p.prof + blockIdx.x * kNumProf;
      pr[kMmaWaitFull] = c_full;
      pr[kMmaWaitAcc] = c_acc;
      pr[kMmaWaitAct] = c_act;
      pr[kItems] = items;
#ifdef RAMP_PROF_LAT
      pr[kLatTma] = c_lat;
      pr[kNumStages] = n_st;
#endif
    }
    };
    // kps is chosen on the device per call: one compiled copy of the role per
    // value (a runtime trip count in these loops costs ~30 % of the issue rate)
    if (!kFp8 && kps == 4) {
      role(KpsC<4>{});
    } else if (kps == 2) {
      role(KpsC<2>{});
    } else {
      role(KpsC<1>{});
    }
  } else if (warp >= 4) {
    // ============================ epilogue ===============================
    const int et2 = threadIdx.x - 128;  // 0 .. kEpiThreads-1
    const int et = et2 & 127;           // TMEM lane == weight row of the 128-row MMA tile
    const int half = et2 >> 7;          // which of the two column halves this warp serves
    const uint32_t lane_off = static_cast<uint32_t>(et & ~31) << 16;
    // the bar.sync id / smem slice private to this half (nA == 1 SwiGLU exchange)
    const uint32_t hbar = 4 + half;
    float* const hbuf = tbuf + half * 1024;
    uint32_t jl = 0, acc_cnt[2] = {0, 0}, chunk_cnt[2] = {0, 0};
    unsigned long long c_meta = 0, c_wacc = 0, c_swiglu = 0, c_wchunk = 0, c_scatter = 0;
    ProfClock pc;
    pc.start();
    uint32_t js = 0, jph = 0;
    for (;; ++jl) {
      mbar_wait(smem_u32(&cs.job_full[js]), jph);
      const int j = cs.job_slot[js];
      mbar_arrive(smem_u32(&cs.job_empty[js]));
      if (++js == 4) { js = 0; jph ^= 1; }
      if (j < 0) break;
      const Job jb = G.job(j);
      const int r = G.acc_buf(jb, jl);
      const uint32_t acc = tmem + lane_off + r * 256;
      const int row0 = jb.m * G.bm;
      pc.lap();
      // token rows and top-k weights of the M-tile, for the jobs that
      // scatter (split mode's phase-1 jobs only write act: no setup)
      if (jb.kind == 1 || G.mode == kModeFused) {
        named_bar_sync(1, kEpiThreads);  // previous job's readers of epi_tok / epi_w are done
        for (int q = et2; q < G.bm; q += kEpiThreads) {
          const int a = p.sorted_ids[row0 + q];
          const bool valid = a < p.n_assign;
          const int t = a / p.top_k;
          cs.epi_tok[q] = valid ? t : -1;
          cs.epi_w[q] = valid ? __ldg(p.topk_w + (p.w_stride ? t * p.w_stride + (a - t * p.top_k) : a)) : 0.0f;
        }
        named_bar_sync(1, kEpiThreads);
      }
      c_meta += pc.lap();
      mbar_wait(smem_u32(&cs.acc_full[r]), acc_cnt[r] & 1);
      START_STAMP(jl == 0 && et2 == 0, kTsFirstAcc);
      ++acc_cnt[r];
      c_wacc += pc.lap();
      tc_fence_after();

      if (jb.kind == 0) {
        // ---- phase 2: SwiGLU -> bf16 act (fused: SW128 K-major smem tile that
        // phase 3 reads; split: L2-resident global rows read by phase-3 jobs)
        auto store_act = [&](int f, int j0, const float (&g)[16], const float (&u)[16]) {
          if constexpr (kFp8) {
            // MXFP8 act for the FP8 phase-3 MMA: the warp's 32 lanes hold 32
            // consecutive features = one scale group per token
            // (one redux per token for the group amax; the 16 x 32 bytes are
            // transposed through this warp's 512 B of tbuf so that every lane
            // stores 16 contiguous bytes of one token row)
            const int l = et & 31;
            const int col0 = jb.s * G.n_i + f - l;  // first feature of the warp's group
            uint8_t* wbuf = reinterpret_cast<uint8_t*>(tbuf) + (et2 >> 5) * 512;
            uint32_t my_sf = 0;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const float a = silu_mul(g[q], u[q]);
              const int ex = mx_exponent(warp_amax_bits(a));
              wbuf[q * 32 + l] = e4m3_from_float(a * mx_inv_scale(ex));
              if (l == q) my_sf = static_cast<uint32_t>(ex + 127);
            }
            __syncwarp();
            const int tq = l >> 1;
            if (j0 + tq < G.bm)
              *reinterpret_cast<int4*>(p.act_q + static_cast<int64_t>(row0 + j0 + tq) * p.I + col0 + (l & 1) * 16) =
                  *reinterpret_cast<const int4*>(wbuf + tq * 32 + (l & 1) * 16);
            if (l < 16 && j0 + l < G.bm)
              p.act_sf[(static_cast<int64_t>(jb.m) * G.kbI + (col0 >> 7)) * 512 + ((j0 + l) & 31) * 16 +
                       ((j0 + l) >> 5) * 4 + ((col0 >> 5) & 3)] = static_cast<uint8_t>(my_sf);
            __syncwarp();
            return;
          }
          if (G.mode == kModeFused) {
            unsigned char* kblk = act_ptr + (f >> 6) * bmN * 128;
            const int chunk = (f & 63) >> 3, within = (f & 7) * 2;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              const int jj = j0 + q;
              *reinterpret_cast<__nv_bfloat16*>(kblk + jj * 128 + ((chunk ^ (jj & 7)) << 4) + within) =
                  __float2bfloat16(silu_mul(g[q], u[q]));
            }
          } else {
            // lanes (f, f+1) swap one value per token pair so each lane writes
            // a packed bf16x2 (4 B) instead of two 2-byte stores
            const bool odd = f & 1;
            __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
                p.act_g + static_cast<size_t>(row0 + j0) * p.I + jb.s * G.n_i + (f & ~1));
#pragma unroll
            for (int m2 = 0; m2 < 8; ++m2) {
              const float a0 = silu_mul(g[2 * m2], u[2 * m2]);
              const float a1 = silu_mul(g[2 * m2 + 1], u[2 * m2 + 1]);
              const float recv = __shfl_xor_sync(0xffffffffu, odd ? a0 : a1, 1);
              const int q = 2 * m2 + (odd ? 1 : 0);
              if (j0 + q < G.bm)
                dst[static_cast<size_t>(q) * (p.I / 2)] = odd ? __floats2bfloat162_rn(recv, a1)
                                                             : __floats2bfloat162_rn(a0, recv);
            }
          }
        };
        if (G.sk == 1) {
          if (nA == 1) {
            // ttn = 128: lanes 0-63 hold gate rows, lanes 64-127 the matching up rows
            // (the halves take alternate 16-column groups)
            for (int j0 = 16 * half; j0 < bmN; j0 += 32) {
              float g[16], u[16];
              tmem_ld16(acc + j0, g);
              tmem_ld_wait();
              if (et >= 64) {
#pragma unroll
                for (int q = 0; q < 16; ++q) hbuf[q * 64 + (et - 64)] = g[q];
              }
              named_bar_sync(hbar, 128);
              if (et < 64) {
#pragma unroll
                for (int q = 0; q < 16; ++q) u[q] = hbuf[q * 64 + et];
                store_act(et, j0, g, u);
              }
              named_bar_sync(hbar, 128);
            }
          } else {
            // Thread et owns features f = th*128 + et of the stripe; the
            // (th, 32-column) items alternate between the two halves.
            const int nj = (bmN + 31) / 32;
            for (int it = half; it < (nA / 2) * nj; it += kEpiHalves) {
              const int th = it / nj, j0 = (it % nj) * 32;
              const int f = th * 128 + et;
              {  // two 16-column chunks per TMEM round trip
                float g[16], u[16], g1[16], u1[16];
                const bool two = j0 + 16 < bmN;
                tmem_ld16(acc + th * bmN + j0, g);
                tmem_ld16(acc + (nA / 2 + th) * bmN + j0, u);
                if (two) {
                  tmem_ld16(acc + th * bmN + j0 + 16, g1);
                  tmem_ld16(acc + (nA / 2 + th) * bmN + j0 + 16, u1);
                }
                tmem_ld_wait();
                store_act(f, j0, g, u);
                if (two) store_act(f, j0 + 16, g1, u1);
              }
            }
          }
        } else {
          // split-K slice: reduce this job's partial gate/up sums into acc_a
          // (fp32, L2-resident) with 16-byte vector reductions; the last
          // slice to arrive applies SwiGLU below.
          const int two_i = 2 * p.I;
          auto col_of = [&](int t, int lane_row) {
            if (nA == 1) return lane_row < 64 ? jb.s * 64 + lane_row : p.I + jb.s * 64 + (lane_row - 64);
            return (t < nA / 2 ? 0 : p.I) + jb.s * G.n_i + (t % (nA / 2)) * 128 + lane_row;
          };
          // (same quad register transpose as scatter16: no smem, no barrier)
          const int b4 = et & 3;
          const int nj = (G.bm + 15) / 16;
          for (int it = half; it < nA * nj; it += kEpiHalves) {
            const int t = it / nj, j0 = (it % nj) * 16;
            const int c4 = col_of(t, et & ~3);
            {
              float v[16];
              tmem_ld16(acc + t * bmN + j0, v);
              tmem_ld_wait();
#pragma unroll
              for (int cq = 0; cq < 4; ++cq) {
                float x4[4] = {v[4 * cq], v[4 * cq + 1], v[4 * cq + 2], v[4 * cq + 3]};
                quad_transpose(x4, b4);
                const int jj = j0 + 4 * cq + b4;
                if (jj < G.bm)
                  red_add_v4_f32(p.acc_a + static_cast<size_t>(row0 + jj) * two_i + c4,
                                 make_float4(x4[0], x4[1], x4[2], x4[3]));
              }
            }
          }
        }
        tc_fence_before();
        if (G.mode == kModeFused) {
          fence_proxy_async_smem();
          mbar_arrive(smem_u32(&cs.act_full));
          c_swiglu += pc.lap();
          // ---- phase 3 (fused): every 128-row chunk of H for this stripe
          for (int hc = 0; hc < G.n_hc; ++hc) {
            const int b = hc & 1;
            mbar_wait(smem_u32(&cs.chunk_full[b]), chunk_cnt[b] & 1);
            c_wchunk += pc.lap();
            tc_fence_after();
            bool freed = false;
            // two 16-column chunks per TMEM round trip; the halves alternate
            for (int j0 = 32 * half; j0 < G.bm; j0 += 32 * kEpiHalves) {
              float v[16], v1[16];
              const bool two = j0 + 16 < G.bm;
              tmem_ld16(tmem + lane_off + b * bmN + j0, v);
              if (two) tmem_ld16(tmem + lane_off + b * bmN + j0 + 16, v1);
              tmem_ld_wait();
              if (j0 + 32 * kEpiHalves >= G.bm) {  // this half's last TMEM read of the chunk
                tc_fence_before();
                mbar_arrive(smem_u32(&cs.chunk_empty[b]));
                freed = true;
              }
              scatter16(v, j0, G.bm, et, cs, p.out_acc, p.H, hc * 128);
              if (two) scatter16(v1, j0 + 16, G.bm, et, cs, p.out_acc, p.H, hc * 128);
            }
            if (!freed) {  // no columns for this half
              tc_fence_before();
              mbar_arrive(smem_u32(&cs.chunk_empty[b]));
            }
            ++chunk_cnt[b];
            c_scatter += pc.lap();
          }
        } else {
          mbar_arrive(smem_u32(&cs.acc_empty[r]));
          bool publish = true;
          if (G.sk > 1) {
            // count this slice in; the last of the sk slices finishes the stripe
            __threadfence();
            named_bar_sync(1, kEpiThreads);
            if (et2 == 0) {
              int* cnt = p.split_cnt + jb.m * G.stripes + jb.s;
              const int old = atomicAdd(cnt, 1);
              cs.fin = old == G.sk - 1;
              if (cs.fin) *cnt = 0;  // every slice has arrived: reset for the next call
              __threadfence();
            }
            named_bar_sync(1, kEpiThreads);
            publish = cs.fin != 0;
            if (publish) {
              const int two_i = 2 * p.I;
              for (int f = et; f < G.n_i; f += 128) {
                for (int j0 = 16 * half; j0 < G.bm; j0 += 16 * kEpiHalves) {
                  float g[16], u[16];
#pragma unroll
                  for (int q = 0; q < 16; ++q) {
                    g[q] = u[q] = 0.f;
                    if (j0 + q < G.bm) {
                      float* rowp = p.acc_a + static_cast<size_t>(row0 + j0 + q) * two_i + jb.s * G.n_i + f;
                      g[q] = __ldcg(rowp);
                      u[q] = __ldcg(rowp + p.I);
                      rowp[0] = 0.f;  // leave acc_a cleared for the next call
                      rowp[p.I] = 0.f;
                    }
                  }
                  store_act(f, j0, g, u);
                }
              }
            }
          }
          if (publish) {
            // publish phase-1 completion of this (m, s) stripe for the phase-3 jobs
            named_bar_sync(1, kEpiThreads);
            if (et2 == 0) {
              __threadfence();
              atomicAdd(p.done + jb.m, 1);
            }
          }
          c_swiglu += pc.lap();
        }
      } else {
        // ---- split phase 3 epilogue: n3 128-row chunks, full I reduced in TMEM
        // (two 16-column chunks per TMEM round trip)
        // (the halves take alternate (chunk, 32-column) items)
        const int nj = (G.bm + 31) / 32, n_it = G.n3 * nj;
        bool freed = false;
        for (int it = half; it < n_it; it += kEpiHalves) {
          const int t = it / nj, j0 = (it % nj) * 32;
          const int col0 = (jb.hc * G.n3 + t) * 128;
          float v[16], v1[16];
          const bool two = j0 + 16 < G.bm;
          tmem_ld16(acc + t * G.bmN + j0, v);
          if (two) tmem_ld16(acc + t * G.bmN + j0 + 16, v1);
          tmem_ld_wait();
          if (it + kEpiHalves >= n_it) {  // this half's last TMEM read of the job
            tc_fence_before();
            mbar_arrive(smem_u32(&cs.acc_empty[r]));
            freed = true;
          }
          scatter16(v, j0, G.bm, et, cs, p.out_acc, p.H, col0);
          if (two) scatter16(v1, j0 + 16, G.bm, et, cs, p.out_acc, p.H, col0);
        }
        if (!freed) {
          tc_fence_before();
          mbar_arrive(smem_u32(&cs.acc_empty[r]));
        }
        c_scatter += pc.lap();
      }
    }
    if (p.prof && et2 == 0) {
      unsigned long long* pr = p.prof + blockIdx.x * kNumProf;
      pr[kTsEpilogueDone] = globaltimer();
      pr[kEpiMeta] = c_meta;
      pr[kEpiWaitAcc] = c_wacc;
      pr[kEpiSwiglu] = c_swiglu;
      pr[kEpiWaitChunk] = c_wchunk;
      pr[kEpiScatter] = c_scatter;
    }
  }

  // ---- grid barrier 1: every job's reductions have landed; then convert
  // the fp32 accumulator to bf16 and clear it for the next call.
  // The next route kernel (a PDL secondary) may be scheduled from here on; it
  // waits for this grid's completion before it reads or writes anything.
  pdl_launch_dependents();
  __threadfence();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
  if (threadIdx.x == 0) {
    if (ts) ts[kTsEndArrive] = globaltimer();
    atomicAdd(p.gbar + 1, 1);
    while (ld_acquire_gpu(p.gbar + 1) < (int)gridDim.x) __nanosleep(64);
    if (ts) ts[kTsEndPass] = globaltimer();
  }
  __syncthreads();
  {
    const int64_t n4 = static_cast<int64_t>(p.S) * p.H / 4;  // H % 128 == 0
    float4* a4 = reinterpret_cast<float4*>(p.out_acc);
    uint2* o2 = reinterpret_cast<uint2*>(p.out);
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(a4 + i);
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      o2[i] = pk;
      a4[i] = z;
    }
  }
  if (ts && threadIdx.x == 0) ts[kTsFinal] = globaltimer();
}

}  // namespace ramp
