// Host-side launchers shared between the translation units of libramp_b200.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/ramp_b200.h"

namespace ramp {

constexpr int kMaxBm = 256;  // largest token block the megakernel supports (256: BF16, ttn <= 256)
inline int bm_mma_host(int bm) { return bm <= 16 ? 16 : (bm + 15) / 16 * 16; }
// TMEM columns kSfCol..511 hold the FP8 MMAs' scale factors (4 columns per
// 512-byte atom, up to 16 atoms per stage); FP8 accumulators stay below.
constexpr int kSfCol = 448;

struct RouteArgs {
  const int32_t* topk_ids;
  int64_t ids_stride;    // int32s between consecutive tokens' ids; 0 = dense [S, top_k]
  int64_t n_assign;
  int32_t E;
  int32_t forced_cfg;
  ramp_table_t table;
  int32_t* ctrl;         // [16]: cfg, n_post_pad, n_mtiles, n_eval, bad_ids, -, -, job counter, grid barriers
  int32_t* hist_out;     // [E] or null
  int32_t* sorted_ids;   // [capacity]
  int32_t* tile_expert;  // [capacity]
  int32_t* sel_out;      // [4] or null
  int32_t* n_eval_out;   // or null
  int64_t* grid_out;     // [n_cfg] or null
  double* pred_out;      // [n_cfg] or null
  int* done;             // split-mode per-M-tile counters, zeroed by block 0
  unsigned long long* prof;  // optional globaltimer stamps (diagnostics)
  int32_t S, H, top_k;
  int32_t pdl_prev;      // launched as a PDL secondary of the previous kernel: 1 = waits before reading
                         // its inputs, 2 = reads nothing of it (waits only before completing)
  int32_t pdl_early;     // trigger the dependent launch at entry (1) or after the alignment (0)
  // router fusion: when logits != null the route kernel first computes the
  // softmax top-k into topk_ids (== ids_out) and w_out
  const void* logits;    // [S, E] fp32 or bf16
  int32_t logits_bf16, renorm;
  float* w_out;          // [S, top_k]
};

int pdl_mode();          // RAMP_PDL: 0 off, 1 trigger at route entry (default), 2 trigger at route exit

cudaError_t launch_route(const RouteArgs& a, cudaStream_t stream);
cudaError_t launch_align(const int32_t* ids, int64_t n, int E, int bm, int32_t* hist, int32_t* sorted_ids,
                         int32_t* tile_expert, int32_t* n_post_pad, cudaStream_t stream);
cudaError_t launch_select(const int32_t* hist, int E, const ramp_table_t& t, int32_t* cfg_out,
                          int32_t* n_eval_out, int64_t* grid_out, double* pred_out,
                          cudaStream_t stream);

struct MoeLaunch {
  const void* x;
  const void* w1;
  const void* w2;
  const float* topk_w;
  const int32_t* ctrl;
  const int32_t* sorted_ids;
  const int32_t* tile_expert;
  float* out_acc;
  void* out;
  void* x_sorted;   // [rows, H] bf16
  void* act_g;      // [rows, I] bf16
  int* done;        // [rows] split-mode counters
  int* job_counter; // dynamic scheduler claim counter (zeroed by the route kernel)
  float* acc_a;     // [rows, 2I] split-K partial sums
  int* split_cnt;   // [rows] split-K arrival counters
  bool fp8;         // MXFP8 path: w1/w2 are e4m3 with tiled UE8M0 scale atoms
  const uint8_t* w1_sf;
  const uint8_t* w2_sf;
  void* x_q;        // [rows, H] e4m3
  uint8_t* x_sf;    // [M-tiles][H/128][512]
  void* act_q;      // [rows, I] e4m3
  uint8_t* act_sf;  // [M-tiles][I/128][512]
  const uint8_t* xq_in;   // optional pre-quantised tokens [S, H] e4m3 (FP8 path)
  const uint8_t* xsf_in;  // and their row-major scales [S, H/32]
  // token-row strides (0 = dense): bytes between rows of x / xq_in and of
  // xsf_in, floats between rows of topk_w (e.g. the rows of an expert-parallel
  // message: ramp_ep_row_layout)
  int64_t x_stride, sf_stride, w_stride;
  int64_t rows;     // capacity of x_sorted / act_g
  ramp_table_t table;
  int32_t S, H, I, E, top_k;
};

bool pdl_prev_enabled();       // RAMP_PDL_PREV (default 0, measured neutral): route as PDL secondary of the previous kernel

extern unsigned long long* g_prof_buffer;  // diagnostics, see ramp_set_profile_buffer

cudaError_t launch_fused_moe(const MoeLaunch& l, cudaStream_t stream, const char** why);

// expert-parallel exchange kernels (csrc/ep.cu)
struct EpPackArgs {
  const int32_t* ids;   // [S, k] global expert ids (outside [0, E): ignored)
  const float* w;       // [S, k]
  const void* x;        // [S, H] bf16
  int32_t S, H, k, E, world, cap;
  uint8_t* send;        // [world][cap][row_bytes] messages (ep_row_layout): the token (bf16, or e4m3
                        // + UE8M0 scales at off_sf), its k rank-local ids at off_ids (-1 = another
                        // rank's slot / padding row) and weights at off_w
  int32_t off_sf, off_ids, off_w, row_bytes;
  int32_t* pos;         // [S][world] send row of (token, rank), -1 = not sent
  int32_t* counts;      // [world] rows sent to each rank
  int32_t* overflow;    // set to 1 when a rank needs more than cap rows (those pairs are dropped)
};
// {off_sf (-1: bf16 wire), off_ids, off_w, row_bytes} of one wire row
void ep_row_layout(int32_t H, int32_t k, bool fp8_wire, int32_t out4[4]);
cudaError_t launch_ep_pack(const EpPackArgs& a, bool fp8_wire, cudaStream_t stream);
cudaError_t launch_ep_combine(const void* back, const int32_t* pos, int32_t S, int32_t H, int32_t world,
                              int32_t cap, void* out, cudaStream_t stream);
// NCCL, loaded at run time (dlopen of the process's libnccl.so.2: torch's when torch is loaded)
struct NcclApi;
const NcclApi* nccl_api(const char** why);
int nccl_unique_id(unsigned char out[128], const char** why);
void* nccl_comm_init(const unsigned char id[128], int world, int rank, const char** why);
int nccl_comm_destroy(void* comm);
// grouped send/recv of `world` equal blocks of `block_bytes` (block d of
// send goes to rank d, block s of recv comes from rank s); n_bufs pairs in one group
int nccl_all_to_all(void* comm, int world, const void* const* send, void* const* recv, const size_t* block_bytes,
                    int n_bufs, cudaStream_t stream, const char** why);
int64_t config_smem_bytes(int bm, int ttn, int stg, int mode, bool fp8, int kps = 1);
// MXFP8 quantisation of token rows [S, H] bf16 -> e4m3 [S, H] + UE8M0 [S, H/32] (row-major)
cudaError_t launch_mx_quant_tokens(const void* x, int64_t S, int32_t H, uint8_t* q, uint8_t* sf,
                                   cudaStream_t stream);

}  // namespace ramp
