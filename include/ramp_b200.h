/*
 * ramp_b200.h -- C ABI of the B200-native RaMP fused-MoE hot path.
 *
 * The reference (arxiv 2604.26039, /root/reference/pkg/src/ramp) is a Python
 * package with no FFI; its hot path is the online selector
 *   select_config(table, hist, cache, step_id)      ramp/dispatch.py:89-122
 *   pool_grids(pool, hist)                          ramp/routing.py:206-216
 *   predict_batch(a, b, c, d, g, sm_count)          ramp/cost_model.py:104-114
 * plus the fused kernel it only simulates (simulate_pool_times,
 * ramp/oracle.py:197-254; kernel semantics PAPER.md:155-169, :719-754).
 * Each entry point below replaces one of those; the Python mirror in
 * paper_2604_26039_b200/ binds them with ctypes.
 *
 * Conventions
 *   - every pointer argument is DEVICE memory unless the name ends in _host;
 *     buffers are owned by the caller (torch allocates them);
 *   - every call is stream-ordered on `stream` (a cudaStream_t, 0 = legacy
 *     default stream) and never synchronises the host;
 *   - return value: 0 on success, a RAMP_E* code otherwise; ramp_last_error()
 *     returns a thread-local message for the last failure on this thread.
 */
#ifndef RAMP_B200_H
#define RAMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RAMP_OK 0
#define RAMP_EINVAL 1  /* bad shape / argument  (reference raises ValueError)   */
#define RAMP_ECUDA 2   /* CUDA runtime / driver failure                           */
#define RAMP_ENOSYS 3  /* not built for this configuration (e.g. no sm_100a GPU)  */

/* Dispatch table: the pool's per-config integer fields plus the four fitted
 * floats per config (ramp/dispatch.py:57-86, "4 floats per config",
 * PAPER.md:701-703).  All arrays are device arrays of length n_cfg, except
 * ubm (n_ubm distinct bm values, ascending) and ubm_index (n_cfg entries into
 * ubm), which let the device share the ceil-divs per distinct bm exactly like
 * pool_grids' np.unique (ramp/routing.py:212-214). */
typedef struct ramp_table {
  int32_t n_cfg;
  int32_t n_ubm;
  int32_t N;        /* geometry N (= 2 * d_ff for the up/gate GEMM)            */
  int32_t kappa_ok; /* region_variables(geom).kappa >= 48 (ramp/dispatch.py:86) */
  int32_t sm_count; /* DispatchTable.sm_count                                   */
  int32_t reserved[3];
  const int32_t* bm;
  const int32_t* ttn;
  const int32_t* stg;
  const int32_t* split_k;
  const int32_t* group_m;
  const int32_t* mode;    /* megakernel mode: 0 fused (act in smem), 1 split (act in L2); may be null = 0 */
  const int32_t* ubm;
  const int32_t* ubm_index;
  const double* a;
  const double* b;
  const double* c;
  const double* d;
  /* Optional generalisations (the reference behaviour when null / <= 0):
   * ntile[i]   work tiles per M-tile of config i, replacing ceil(N/ttn) in
   *            g = M-tiles * ntile * split_k -- the B200 megakernel's split
   *            mode runs I-stripe jobs AND H-chunk jobs per M-tile;
   * omega_max  split-K gate threshold (reference: 0.2, ramp/dispatch.py:31);
   * lam[i]     B200 L2-reuse factor of config i (variant "B4"): the traffic
   *            terms c*g and d*ln(g+1) see the HBM-equivalent grid
   *            g_l = ntile*split_k*(n_act + lam*(M-tiles - n_act)), n_act =
   *            active experts, while the wave term keeps the job grid g.
   *            null: g_l = g (the reference model). */
  const int32_t* ntile;
  double omega_max;
  const double* lam;
  /* kps[i]     k-blocks (64 K-elements each) per pipeline stage of config i,
   *            1, 2 or 4 (BF16 megakernel; null = 1).  Larger stages raise the
   *            per-CTA weight-streaming rate of the decode configs. */
  const int32_t* kps;
  /* step_cache  optional device-resident StepCache (ramp/dispatch.py:40-54):
   *             int32 [3 + 2*cap] = {current step, cached step, n, (M, cfg) x cap}.
   *             The caller advances the step by writing [0] (graph-capturable);
   *             the dispatcher resets the entries when [1] != [0], reuses the
   *             selection cached for this step's M = hist total, and appends on
   *             a miss.  null = no cache. */
  int32_t* step_cache;
  int32_t step_cache_cap;
  /* h3[i]      split-mode phase-3 jobs of config i cover h3 128-row chunks of
   *            d_model sharing one act tile: 1, 2 or 4, at most ttn/128 (BF16
   *            megakernel; null = 1).  Halves/quarters the act re-reads and the
   *            phase-3 job count of the prefill configs. */
  const int32_t* h3;
} ramp_table_t;

/* Library version (major*10000 + minor*100 + patch) and sm_100a build flag. */
int ramp_version(void);
/* Thread-local message for the last non-zero return on this thread. */
const char* ramp_last_error(void);
/* 1 if a device of compute capability 10.0 is visible and the kernels can run. */
int ramp_device_ok(void);

/* Expert histogram + moe_align_block_size (north_star (1); SURVEY 8a rows a1,
 * a19).  Stable counting sort of the flattened topk_ids by expert, each
 * expert padded to a multiple of bm.
 *   hist[E]            bincount(topk_ids, minlength=E)
 *   sorted_ids[cap]    flat assignment indices grouped by expert, ascending
 *                      within an expert, padding = n_assign; cap must be
 *                      >= ramp_align_capacity(n_assign, E, bm)
 *   tile_expert[cap/bm] expert of each bm-row M-tile
 *   n_post_pad[1]      total padded length (sum_e ceil(c_e/bm)*bm)
 * E <= 512.
 * Replaces: the M-tile count inside grid_size / m_tile_counts
 * (ramp/routing.py:191-203) and the routing bincount of PAPER.md:761-762. */
int ramp_moe_align(const int32_t* topk_ids, int64_t n_assign, int32_t E, int32_t bm,
                   int32_t* hist, int32_t* sorted_ids, int32_t* tile_expert, int32_t* n_post_pad,
                   void* stream);
int64_t ramp_align_capacity(int64_t n_assign, int32_t E, int32_t bm);

/* Routing-aware dispatcher on a device histogram (north_star (3)).
 * Evaluates T(g) = a + b*ceil(g/SM) + c*g + d*ln(g+1) in fp64 in numpy's
 * operation order, masks split-K configs failing the gate
 * (g/split_k)/SM < 0.2 with kappa >= 48, and writes the first argmin.
 *   cfg_out[1]         selected config id         (select_config's return)
 *   n_eval_out[1]      number of kept configs     (DispatchTable.evaluations increment)
 *   grid_out[n_cfg]    optional, pool_grids       (ramp/routing.py:206-216)
 *   pred_out[n_cfg]    optional, predict_batch    (ramp/cost_model.py:104-114), +inf if masked
 * Replaces select_config (ramp/dispatch.py:89-122) minus the host StepCache. */
int ramp_dispatch_select(const int32_t* hist, int32_t E, const ramp_table_t* table,
                         int32_t* cfg_out, int32_t* n_eval_out, int64_t* grid_out, double* pred_out,
                         void* stream);

/* Fused MoE layer forward, BF16 (north_star (2)):
 *   out[t] = sum_j topk_w[t,j] * W2[e] (silu(W1[e,:I] x_t) * (W1[e,I:] x_t)),  e = topk_ids[t,j]
 * x[S,H] bf16, w1[E,2I,H] bf16 (gate rows first), w2[E,H,I] bf16, topk_w[S,k]
 * fp32, topk_ids[S,k] int32, out[S,H] bf16.  One call = route kernel
 * (histogram -> dispatcher -> align -> accumulator clear) + persistent
 * tcgen05 megakernel + bf16 finalize; no host synchronisation.
 *   forced_cfg < 0   select on device from the live histogram (routing-aware)
 *   forced_cfg >= 0  run that config id (static dispatch / exhaustive sweep)
 *   sel_out          optional device int32[4]: {cfg, n_post_pad, n_work, n_eval}
 * workspace: >= ramp_fused_moe_workspace_size(S, ...) bytes of device memory,
 *            zero-filled once before its first use.  The regions are laid out
 *            for the largest S the buffer holds (not for this call's S), so a
 *            workspace can serve every smaller batch; when the geometry
 *            (H, I, E, top_k) or workspace_bytes change between calls on the
 *            same buffer, the library re-zeroes it (stream-ordered memset)
 *            before use.  int32 word 4 of the workspace is set to 1 by a call
 *            whose topk_ids held an id outside [0, E) other than -1 (such
 *            slots are skipped; the reference's ExpertHistogram raises
 *            ValueError for them, ramp/routing.py:45-50).
 * Replaces the kernel that simulate_pool_times stands in for
 * (ramp/oracle.py:197-254) together with the select_config call before it. */
size_t ramp_fused_moe_workspace_size(int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k);
int ramp_fused_moe_bf16(const void* x, const void* w1, const void* w2, const float* topk_w,
                        const int32_t* topk_ids, int32_t S, int32_t H, int32_t I, int32_t E,
                        int32_t top_k, const ramp_table_t* table, int32_t forced_cfg, void* out,
                        int32_t* sel_out, void* workspace, size_t workspace_bytes, void* stream);

/* The two launches of ramp_fused_moe_bf16 separately, on the same arguments
 * and workspace: phases = 1 runs only the route kernel (histogram, dispatch,
 * alignment), 2 only the megakernel (which reads the route kernel's outputs
 * from the workspace), 3 both.  Lets a caller time the megakernel alone or
 * reuse one routing decision for several layers that share the histogram. */
int ramp_fused_moe_bf16_ex(const void* x, const void* w1, const void* w2, const float* topk_w,
                           const int32_t* topk_ids, int32_t S, int32_t H, int32_t I, int32_t E,
                           int32_t top_k, const ramp_table_t* table, int32_t forced_cfg, void* out,
                           int32_t* sel_out, void* workspace, size_t workspace_bytes, int32_t phases,
                           void* stream);

/* Router fusion: the BF16 layer straight from the router's
 * logits, vLLM's fused_moe(hidden_states, w1, w2, gating_output, topk,
 * renormalize) contract.  The route kernel first takes the softmax top-k of
 * router_logits[S,E] (fp32, or bf16 when logits_bf16) per token: the k
 * highest probabilities, ties to the lower expert id; weights = the softmax
 * probabilities (fp32), divided by their sum over the k picks when
 * renormalize.  It writes them to topk_w_out[S,k] / topk_ids_out[S,k]
 * (device) and continues exactly as ramp_fused_moe_bf16 on them -- the
 * routing decision never round-trips through another kernel.
 * Needs top_k <= 32 and S * top_k <= 16384. */
int ramp_fused_moe_gating_bf16(const void* x, const void* w1, const void* w2, const void* router_logits,
                               int32_t logits_bf16, int32_t renormalize, float* topk_w_out, int32_t* topk_ids_out,
                               int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k, const ramp_table_t* table,
                               int32_t forced_cfg, void* out, int32_t* sel_out, void* workspace,
                               size_t workspace_bytes, void* stream);

/* Fused MoE layer forward, block-scaled FP8 (MXFP8: E4M3 operands with one
 * UE8M0 scale per 32 K elements, kind::mxf8f6f4.block_scale MMAs).
 * w1_q [E,2I,H] / w2_q [E,H,I] e4m3; w1_sf / w2_sf their scale atoms tiled as
 * [rows/128][K/128][512 B] (paper_2604_26039_b200/quant.py tile_scales);
 * tokens arrive in bf16 and are quantised on the fly (per token, per 32).
 * The table must hold FP8 configs (split mode, ttn >= 256,
 * ramp_config_smem_bytes_fp8_kps > 0).  d_ff must be a multiple of 256.
 * Replaces the W8A8 FP8 kernel of the paper. */
int ramp_fused_moe_fp8(const void* x, const void* w1_q, const uint8_t* w1_sf, const void* w2_q,
                       const uint8_t* w2_sf, const float* topk_w, const int32_t* topk_ids, int32_t S, int32_t H,
                       int32_t I, int32_t E, int32_t top_k, const ramp_table_t* table, int32_t forced_cfg,
                       void* out, int32_t* sel_out, void* workspace, size_t workspace_bytes, int32_t phases,
                       void* stream);
/* Same layer with the tokens already in MXFP8 -- x_q [S,H] e4m3 and x_sf
 * [S,H/32] UE8M0 row-major, e.g. straight off the RAMP_EP_WIRE_MXFP8
 * exchange: the megakernel's phase 0 moves them instead of quantising. */
int ramp_fused_moe_fp8_prequant(const uint8_t* x_q, const uint8_t* x_sf, const void* w1_q, const uint8_t* w1_sf,
                                const void* w2_q, const uint8_t* w2_sf, const float* topk_w, const int32_t* topk_ids,
                                int32_t S, int32_t H, int32_t I, int32_t E, int32_t top_k, const ramp_table_t* table,
                                int32_t forced_cfg, void* out, int32_t* sel_out, void* workspace,
                                size_t workspace_bytes, int32_t phases, void* stream);
/* Token-row strides of the per-token inputs (0 = dense), for tokens that sit
 * inside wider rows -- e.g. the received rows of an expert-parallel message
 * (ramp_ep_row_layout), where x, its scales, the ids and the weights of one
 * token share a row.  x_stride: bytes between rows of x (multiple of 16);
 * sf_stride: bytes between rows of x_sf (multiple of 4); ids_stride / w_stride:
 * elements between rows of topk_ids / topk_w (>= top_k). */
typedef struct {
  int64_t x_stride;
  int64_t sf_stride;
  int64_t ids_stride;
  int64_t w_stride;
} ramp_row_strides_t;
/* ramp_fused_moe_bf16_ex / ramp_fused_moe_fp8 / ramp_fused_moe_fp8_prequant
 * with row-strided token inputs: BF16 when w1_sf is null; else MXFP8, the
 * tokens bf16 when x_sf is null, already MXFP8 (x = e4m3 bytes) when not. */
int ramp_fused_moe_strided(const void* x, const uint8_t* x_sf, const void* w1, const uint8_t* w1_sf, const void* w2,
                           const uint8_t* w2_sf, const float* topk_w, const int32_t* topk_ids,
                           const ramp_row_strides_t* strides, int32_t S, int32_t H, int32_t I, int32_t E,
                           int32_t top_k, const ramp_table_t* table, int32_t forced_cfg, void* out, int32_t* sel_out,
                           void* workspace, size_t workspace_bytes, int32_t phases, void* stream);
int64_t ramp_config_smem_bytes_fp8(int32_t bm, int32_t ttn, int32_t stg);
/* Same with kps k-blocks (128 K-elements each) per stage (1 or 2); 0 if not realisable. */
int64_t ramp_config_smem_bytes_fp8_kps(int32_t bm, int32_t ttn, int32_t stg, int32_t kps);

/* Shared-memory bytes the megakernel needs for (bm, ttn, stg, mode); 0 if the
 * configuration is not realisable on this part (pool admissibility test,
 * the B200 counterpart of smem_usage/is_valid, ramp/config_space.py:122-138). */
int64_t ramp_config_smem_bytes(int32_t bm, int32_t ttn, int32_t stg, int32_t mode);
/* Same with kps k-blocks per stage (1, 2 or 4); 0 if not realisable. */
int64_t ramp_config_smem_bytes_kps(int32_t bm, int32_t ttn, int32_t stg, int32_t mode, int32_t kps);

/* Diagnostics: when dev_buf is non-null, every later megakernel launch writes
 * 32 per-CTA slots (cycle counters of the producer / MMA / epilogue roles and
 * globaltimer stamps of the kernel's phases, see ProfSlot in
 * csrc/fused_moe.cuh) to dev_buf[blockIdx * 32 + slot], and the route kernel
 * writes globaltimer stamps to dev_buf[148 * 32 + 0..15]; from
 * dev_buf[149 * 32] on, each CTA logs its first 16 jobs as
 * {job id, claimed, loads issued, epilogue done} (4 entries per job)
 * (buffer: >= 149 * 32 + 148 * 16 * 4 entries).
 * Pass null to switch it off.  Not used on the timed path. */
void ramp_set_profile_buffer(unsigned long long* dev_buf);

/* ---------------------------------------------------------------------------
 * Expert parallelism (north_star (4); SURVEY.md 8b ramp_ep_dispatch/combine,
 * replacing the eager torch exchange the reference-side integration would
 * otherwise write).  Rank r of `world` owns experts [r*E/world, (r+1)*E/world).
 * Every exchange moves fixed-capacity blocks -- `cap` rows per destination
 * (cap = S never drops a pair) -- so no split size is read on the host and
 * the layer is CUDA-graph capturable.  A row is one self-contained message
 * of row_bytes (ramp_ep_row_layout), so a dispatch is ONE send / receive per
 * peer:
 *   send     [world][cap][row_bytes]; row = the token (H bf16, or H e4m3 +
 *            H/32 UE8M0 scales at off_sf: RAMP_EP_WIRE_MXFP8, 0.52x the
 *            bytes, consumed as is by the FP8 megakernel), its top_k
 *            rank-local expert ids at off_ids (int32, -1 = another rank's slot
 *            or a padding row: skipped by the route kernel, no work) and their
 *            fp32 weights at off_w (0 on -1 slots)
 *   pos      [S][world] row of (token, rank) in the send blocks, -1 = none
 *   counts   [world] rows sent; *overflow = 1 if some rank needed > cap rows
 * The receive buffer has the same shape (block s came from rank s); the local
 * layer reads it in place through ramp_fused_moe_strided (all four strides =
 * row_bytes).
 */
#define RAMP_EP_WIRE_BF16 0
#define RAMP_EP_WIRE_MXFP8 1
typedef struct ramp_ep_comm ramp_ep_comm;

/* Row layout of the wire: out4 = {off_sf (-1 for bf16), off_ids, off_w,
 * row_bytes}, every offset and row_bytes a multiple of 16 (off_w: of 4). */
int ramp_ep_row_layout(int32_t H, int32_t top_k, int32_t wire, int32_t* out4);
/* pack only (the exchange is left to the caller, e.g. torch.distributed) */
int ramp_ep_pack(const void* x, const int32_t* topk_ids, const float* topk_w, int32_t S, int32_t H, int32_t E,
                 int32_t top_k, int32_t world, int32_t cap, int32_t wire, void* send, int32_t* pos, int32_t* counts,
                 int32_t* overflow, void* stream);
/* out[t] = sum over ranks d (in rank order) of back[d][pos[t][d]] (fp32 sum, bf16 out) */
int ramp_ep_reduce(const void* back, const int32_t* pos, int32_t S, int32_t H, int32_t world, int32_t cap,
                   void* out, void* stream);
/* NCCL communicator (libnccl.so.2 loaded at run time): rank 0 gets the
 * 128-byte id, every rank passes it to ramp_ep_comm_init. */
int ramp_ep_get_unique_id(unsigned char* out128);
int ramp_ep_comm_init(ramp_ep_comm** comm, const unsigned char* id128, int32_t world, int32_t rank);
int ramp_ep_comm_destroy(ramp_ep_comm* comm);
/* pack + one grouped NCCL all-to-all of the row blocks (one send and one
 * receive per peer) */
int ramp_ep_dispatch(ramp_ep_comm* comm, const void* x, const int32_t* topk_ids, const float* topk_w, int32_t S,
                     int32_t H, int32_t E, int32_t top_k, int32_t cap, int32_t wire, void* send, int32_t* pos,
                     int32_t* counts, int32_t* overflow, void* recv, void* stream);
/* NCCL all-to-all of the partial outputs [world*cap][H] bf16 back into
 * back[world][cap][H], then ramp_ep_reduce into out[S][H] */
int ramp_ep_combine(ramp_ep_comm* comm, const void* partial, void* back, const int32_t* pos, int32_t S, int32_t H,
                    int32_t cap, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RAMP_B200_H */
