// Expert-parallel exchange kernels (north_star (4)).
//
// Rank r of a P-rank group owns experts [r*E/P, (r+1)*E/P).  A layer call
// exchanges fixed-capacity buffers, so nothing on the path needs the
// per-destination counts on the host (no device -> host read, graph
// capturable):
//
//   pack     x[S,H], topk_ids/w[S,k] -> for every destination rank d a block
//            of `cap` rows: the tokens with at least one expert on d, in
//            token order (one row per unique (token, rank) pair: the
//            "pre-reduce per (token, rank)" of SURVEY 8e), their top-k slots
//            as d-local expert ids (-1 for slots owned by other ranks) and
//            weights (0 there); rows past the count carry ids -1 (the route
//            kernel skips them: no work).  Token rows travel as bf16 or as
//            MXFP8 (E4M3 + one UE8M0 scale per 32 features, the FP8
//            megakernel's operand format).  A row is one self-contained
//            message -- token, scales, ids, weights at fixed offsets
//            (ep_row_layout) -- so the exchange is one send / receive per
//            peer and the receiver's megakernel reads the rows in place
//            (row-strided inputs).  pos[t][d] remembers the row.
//   (all-to-all of the P blocks: NCCL, or torch.distributed in the tests)
//   combine  the per-(token, rank) partial outputs that came back, summed in
//            fp32 in rank order into out[S,H] bf16 (deterministic).
//
// Both kernels are HBM/L2-bound byte movers: x is read once per token and
// written once per (token, rank) pair with 16-byte vectors.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "launch.h"
#include "ptx.cuh"

namespace ramp {

constexpr int kEpThreads = 256;
constexpr int kEpMaxWorld = 32;

void ep_row_layout(int32_t H, int32_t k, bool fp8_wire, int32_t out4[4]) {
  auto up16 = [](int32_t v) { return (v + 15) & ~15; };
  const int32_t tok = fp8_wire ? H + H / 32 : 2 * H;
  out4[0] = fp8_wire ? H : -1;
  out4[1] = up16(tok);
  out4[2] = out4[1] + 4 * k;
  out4[3] = up16(out4[2] + 4 * k);
}

// per = experts per rank; shift = log2(per) when per is a power of two
// (every model here), else -1 (integer division)
__device__ __forceinline__ int ep_owner(int id, int per, int shift) { return shift >= 0 ? id >> shift : id / per; }

__device__ __forceinline__ uint32_t ep_mask(const int32_t* ids, int t, int k, int E, int per, int shift) {
  uint32_t m = 0;
  for (int j = 0; j < k; ++j) {
    const int id = __ldg(ids + static_cast<int64_t>(t) * k + j);
    if (id >= 0 && id < E) m |= 1u << ep_owner(id, per, shift);
  }
  return m;
}

template <bool kFp8>
__global__ void __launch_bounds__(kEpThreads) ep_pack_kernel(EpPackArgs a) {
  __shared__ int s_before[kEpMaxWorld], s_total[kEpMaxWorld];
  __shared__ int s_warp[kEpMaxWorld][kEpThreads / 32];
  __shared__ uint32_t s_mask[kEpThreads];
  __shared__ int s_pos[kEpThreads][8];  // first 8 destinations' rows of this block's tokens (pos[] has all)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = a.world, per = a.E / a.world;
  const int shift = (per & (per - 1)) == 0 ? __ffs(per) - 1 : -1;
  const int T = (a.S + gridDim.x - 1) / gridDim.x;  // tokens per block (<= kEpThreads)
  const int t0 = min(a.S, static_cast<int>(blockIdx.x) * T), t1 = min(a.S, t0 + T);
  if (tid < kEpMaxWorld) s_before[tid] = s_total[tid] = 0;
  // this block's token rows start streaming into L2 now; the row copies of
  // step (4) wait for the counts and the scan, not for HBM
  if (tid < t1 - t0) bulk_prefetch_l2(static_cast<const uint8_t*>(a.x) + static_cast<int64_t>(t0 + tid) * a.H * 2,
                                      static_cast<uint32_t>(a.H) * 2);
  __syncthreads();
  // (1) how many tokens before this block's chunk go to each rank, and in
  // total; the destination masks of the block's own tokens are kept
  for (int base = 0; base < a.S; base += kEpThreads) {
    const int t = base + tid;
    const uint32_t m = t < a.S ? ep_mask(a.ids, t, a.k, a.E, per, shift) : 0u;
    if (t >= t0 && t < t1) s_mask[t - t0] = m;
    for (int d = 0; d < P; ++d) {
      const uint32_t b = __ballot_sync(0xffffffffu, (m >> d) & 1u);
      const uint32_t bb = __ballot_sync(0xffffffffu, ((m >> d) & 1u) && t < t0);
      if (lane == 0 && b) {
        atomicAdd(&s_total[d], __popc(b));
        if (bb) atomicAdd(&s_before[d], __popc(bb));
      }
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {  // written, not accumulated: no zero-fill needed before the launch
    int o = 0;
    for (int d = 0; d < P; ++d) {
      a.counts[d] = min(s_total[d], a.cap);
      o |= s_total[d] > a.cap;  // the caller's capacity is too small: the pairs past it are dropped
    }
    *a.overflow = o;
  }
  // (2) rows of this block's tokens: block-wide exclusive scan per rank
  const int t = t0 + tid;
  const uint32_t m = t < t1 ? s_mask[tid] : 0u;
  for (int d = 0; d < P; ++d) {
    const uint32_t b = __ballot_sync(0xffffffffu, (m >> d) & 1u);
    if (lane == 0) s_warp[d][warp] = __popc(b);
  }
  __syncthreads();
  if (tid < P) {
    int run = s_before[tid];
    for (int w = 0; w < kEpThreads / 32; ++w) {
      const int c = s_warp[tid][w];
      s_warp[tid][w] = run;
      run += c;
    }
  }
  __syncthreads();
  for (int d = 0; d < P; ++d) {
    const bool hit = (m >> d) & 1u;
    const uint32_t b = __ballot_sync(0xffffffffu, hit);
    int row = hit ? s_warp[d][warp] + __popc(b & ((1u << lane) - 1u)) : -1;
    if (row >= a.cap) row = -1;  // dropped (overflow flagged above)
    if (t < t1) {
      a.pos[static_cast<int64_t>(t) * P + d] = row;
      if (d < 8) s_pos[tid][d] = row;
    }
  }
  __syncthreads();
  // (3) the slots of every row: one (token, slot) per thread, so each
  // thread's two loads are in flight together (no load-after-store chain)
  for (int it = tid; it < (t1 - t0) * a.k; it += kEpThreads) {
    const int q = it / a.k, j = it - q * a.k;
    const int64_t src = static_cast<int64_t>(t0 + q) * a.k + j;
    const int id = __ldg(a.ids + src);
    const float wv = __ldg(a.w + src);
    const int own_d = id >= 0 && id < a.E ? ep_owner(id, per, shift) : -1;
    for (int d = 0; d < P; ++d) {
      const int row = d < 8 ? s_pos[q][d] : __ldcg(a.pos + static_cast<int64_t>(t0 + q) * P + d);
      if (row < 0) continue;
      uint8_t* msg = a.send + (static_cast<int64_t>(d) * a.cap + row) * a.row_bytes;
      reinterpret_cast<int32_t*>(msg + a.off_ids)[j] = own_d == d ? id - d * per : -1;
      reinterpret_cast<float*>(msg + a.off_w)[j] = own_d == d ? wv : 0.0f;
    }
  }
  // rows past each rank's count: ids -1 / weights 0 (no work on arrival)
  const int64_t n_rows = static_cast<int64_t>(P) * a.cap;
  for (int64_t i = blockIdx.x * (int64_t)kEpThreads + tid; i < n_rows; i += (int64_t)gridDim.x * kEpThreads) {
    const int d = static_cast<int>(i / a.cap), row = static_cast<int>(i % a.cap);
    if (row >= s_total[d]) {
      uint8_t* msg = a.send + i * a.row_bytes;
      for (int j = 0; j < a.k; ++j) {
        reinterpret_cast<int32_t*>(msg + a.off_ids)[j] = -1;
        reinterpret_cast<float*>(msg + a.off_w)[j] = 0.0f;
      }
    }
  }
  __syncthreads();
  // (4) token rows: (token, row segment) items over the block's warps -- a
  // segment is 32 x kUnroll 16-byte chunks, read once (kUnroll loads in
  // flight per lane) and written to every destination rank; a block holds
  // few tokens when S is small, so rows are split across warps
  constexpr int kUnroll = 4;
  const int row_vec = a.H / 8;  // 16-byte chunks of 8 bf16
  const int n_seg = (row_vec + 32 * kUnroll - 1) / (32 * kUnroll);
  const int4* xv = reinterpret_cast<const int4*>(a.x);
  for (int item = warp; item < (t1 - t0) * n_seg; item += kEpThreads / 32) {
    const int q = item / n_seg, seg = item - q * n_seg;
    const int tt = t0 + q;
    const uint32_t mq = s_mask[q];
    if (!mq) continue;
    {
      const int c0 = seg * 32 * kUnroll + lane;
      int4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (c0 + 32 * u < row_vec) v[u] = __ldg(xv + static_cast<int64_t>(tt) * row_vec + c0 + 32 * u);
      if constexpr (!kFp8) {
        for (int d = 0; d < P; ++d) {
          if (!((mq >> d) & 1u)) continue;
          const int row = d < 8 ? s_pos[q][d] : a.pos[static_cast<int64_t>(tt) * P + d];
          if (row < 0) continue;
          int4* dst = reinterpret_cast<int4*>(a.send + (static_cast<int64_t>(d) * a.cap + row) * a.row_bytes);
#pragma unroll
          for (int u = 0; u < kUnroll; ++u)
            if (c0 + 32 * u < row_vec) dst[c0 + 32 * u] = v[u];
        }
      } else {
        // MXFP8: 4 lanes (32 features) share one UE8M0 scale
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int c = c0 + 32 * u;
          if (c - lane >= row_vec) break;  // warp-uniform
          const bool in = c < row_vec;
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
          float f[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 p2 = in ? __bfloat1622float2(h2[i]) : make_float2(0.f, 0.f);
            f[2 * i] = p2.x;
            f[2 * i + 1] = p2.y;
          }
          uint32_t am = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) am = max(am, __float_as_uint(fabsf(f[i])));
          am = max(am, __shfl_xor_sync(0xffffffffu, am, 1));
          am = max(am, __shfl_xor_sync(0xffffffffu, am, 2));
          const int ex = mx_exponent(am);
          const float inv = mx_inv_scale(ex);
          uint2 qv;
          qv.x = static_cast<uint32_t>(e4m3x2_from_float(f[0] * inv, f[1] * inv)) |
                 (static_cast<uint32_t>(e4m3x2_from_float(f[2] * inv, f[3] * inv)) << 16);
          qv.y = static_cast<uint32_t>(e4m3x2_from_float(f[4] * inv, f[5] * inv)) |
                 (static_cast<uint32_t>(e4m3x2_from_float(f[6] * inv, f[7] * inv)) << 16);
          if (!in) continue;
          for (int d = 0; d < P; ++d) {
            if (!((mq >> d) & 1u)) continue;
            const int row = d < 8 ? s_pos[q][d] : a.pos[static_cast<int64_t>(tt) * P + d];
            if (row < 0) continue;
            uint8_t* msg = a.send + (static_cast<int64_t>(d) * a.cap + row) * a.row_bytes;
            *reinterpret_cast<uint2*>(msg + c * 8) = qv;
            if ((lane & 3) == 0) msg[a.off_sf + (c >> 2)] = static_cast<uint8_t>(ex + 127);
          }
        }
      }
    }
  }
}

// out[t] = sum over ranks d (in order) of back[d][pos[t][d]], fp32 -> bf16.
__global__ void __launch_bounds__(kEpThreads) ep_combine_kernel(const __nv_bfloat16* back, const int32_t* pos,
                                                                int32_t S, int32_t H, int32_t P, int32_t cap,
                                                                __nv_bfloat16* out) {
  const int row_vec = H / 8;
  const int64_t n = static_cast<int64_t>(S) * row_vec;
  const int4* bv = reinterpret_cast<const int4*>(back);
  int4* ov = reinterpret_cast<int4*>(out);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int t = static_cast<int>(i / row_vec), c = static_cast<int>(i % row_vec);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int d = 0; d < P; ++d) {
      const int row = __ldg(pos + static_cast<int64_t>(t) * P + d);
      if (row < 0) continue;
      const int4 v = __ldg(bv + (static_cast<int64_t>(d) * cap + row) * row_vec + c);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h2[q]);
        acc[2 * q] += f.x;
        acc[2 * q + 1] += f.y;
      }
    }
    int4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int q = 0; q < 4; ++q) o2[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
    ov[i] = o;
  }
}

static int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

cudaError_t launch_ep_pack(const EpPackArgs& a, bool fp8, cudaStream_t st) {
  // S == 0 still launches: the empty rank's blocks must carry ids -1, and
  // counts / overflow are written
  // up to two blocks per SM (both resident): at decode / small-batch sizes a
  // block holds one or two tokens, whose row segments then fit one round of
  // its 8 warps
  const int blocks = max(1, max(min(2 * sm_count(), a.S), (a.S + kEpThreads - 1) / kEpThreads));
  if (fp8)
    ep_pack_kernel<true><<<blocks, kEpThreads, 0, st>>>(a);
  else
    ep_pack_kernel<false><<<blocks, kEpThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_ep_combine(const void* back, const int32_t* pos, int32_t S, int32_t H, int32_t P, int32_t cap,
                              void* out, cudaStream_t st) {
  if (S == 0) return cudaSuccess;
  const int64_t n = static_cast<int64_t>(S) * (H / 8);
  // one 16-byte chunk per thread: every thread's pos -> row loads are its
  // only dependent pair (a grid-stride loop would chain two of them)
  const int64_t want = (n + kEpThreads - 1) / kEpThreads, cap_blocks = 64 * sm_count();
  const int blocks = static_cast<int>(want < cap_blocks ? want : cap_blocks);
  ep_combine_kernel<<<blocks, kEpThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(back), pos, S, H, P, cap,
                                                   static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

// ---------------------------------------------------------------- NCCL
// Loaded at run time: libramp_b200.so has no link-time NCCL dependency, and
// inside a torch process it binds to the libnccl.so.2 torch already loaded
// (one NCCL per process).  Only the C types of nccl.h are restated here.
namespace {
using NcclComm = void*;
struct NcclUid {
  char internal[128];
};
using FnGetUid = int (*)(NcclUid*);
using FnInit = int (*)(NcclComm*, int, NcclUid, int);
using FnDestroy = int (*)(NcclComm);
using FnGroup = int (*)();
using FnSend = int (*)(const void*, size_t, int, int, NcclComm, cudaStream_t);
using FnRecv = int (*)(void*, size_t, int, int, NcclComm, cudaStream_t);
using FnErr = const char* (*)(int);
constexpr int kNcclUint8 = 1;  // ncclUint8 in nccl.h's ncclDataType_t
}  // namespace

struct NcclApi {
  FnGetUid get_uid;
  FnInit init;
  FnDestroy destroy;
  FnGroup group_start, group_end;
  FnSend send;
  FnRecv recv;
  FnErr err;
};

const NcclApi* nccl_api(const char** why) {
  static NcclApi api{};
  static const char* fail = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      fail = "libnccl.so.2 not found";
      return;
    }
    api.get_uid = reinterpret_cast<FnGetUid>(dlsym(h, "ncclGetUniqueId"));
    api.init = reinterpret_cast<FnInit>(dlsym(h, "ncclCommInitRank"));
    api.destroy = reinterpret_cast<FnDestroy>(dlsym(h, "ncclCommDestroy"));
    api.group_start = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupEnd"));
    api.send = reinterpret_cast<FnSend>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<FnRecv>(dlsym(h, "ncclRecv"));
    api.err = reinterpret_cast<FnErr>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_uid || !api.init || !api.destroy || !api.group_start || !api.group_end || !api.send || !api.recv ||
        !api.err)
      fail = "libnccl.so.2 lacks a required symbol";
  });
  if (fail) {
    if (why) *why = fail;
    return nullptr;
  }
  return &api;
}

int nccl_unique_id(unsigned char out[128], const char** why) {
  const NcclApi* a = nccl_api(why);
  if (!a) return -1;
  NcclUid uid;
  const int rc = a->get_uid(&uid);
  if (rc != 0) {
    if (why) *why = a->err(rc);
    return -1;
  }
  std::memcpy(out, uid.internal, 128);
  return 0;
}

void* nccl_comm_init(const unsigned char id[128], int world, int rank, const char** why) {
  const NcclApi* a = nccl_api(why);
  if (!a) return nullptr;
  NcclUid uid;
  std::memcpy(uid.internal, id, 128);
  NcclComm comm = nullptr;
  const int rc = a->init(&comm, world, uid, rank);
  if (rc != 0) {
    if (why) *why = a->err(rc);
    return nullptr;
  }
  return comm;
}

int nccl_comm_destroy(void* comm) {
  const NcclApi* a = nccl_api(nullptr);
  return a && comm ? a->destroy(comm) : 0;
}

int nccl_all_to_all(void* comm, int world, const void* const* send, void* const* recv, const size_t* block_bytes,
                    int n_bufs, cudaStream_t st, const char** why) {
  const NcclApi* a = nccl_api(why);
  if (!a) return -1;
  int rc = a->group_start();
  for (int b = 0; b < n_bufs && rc == 0; ++b) {
    for (int d = 0; d < world && rc == 0; ++d) {
      rc = a->send(static_cast<const char*>(send[b]) + d * block_bytes[b], block_bytes[b], kNcclUint8, d, comm, st);
      if (rc == 0)
        rc = a->recv(static_cast<char*>(recv[b]) + d * block_bytes[b], block_bytes[b], kNcclUint8, d, comm, st);
    }
  }
  const int rc2 = a->group_end();
  if (rc == 0) rc = rc2;
  if (rc != 0 && why) *why = a->err(rc);
  return rc == 0 ? 0 : -1;
}

}  // namespace ramp
