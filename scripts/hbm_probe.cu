// Per-SM HBM streaming probe (development tool, not product code).
//
// How fast can G CTAs pull weight tiles from HBM with TMA?  Each CTA streams
// its own region of a [rows, 2048] bf16 matrix (4 KB rows, the OLMoE W1
// layout) in the megakernel's access order: a box of {64 cols, R rows} per
// stage, k-blocks advancing along the row.  Variants: R rows per box, stages
// in flight, boxes per stage (consecutive k-blocks), CTAs in the grid.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_probe hbm_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    auto e = (x);                                                              \
    if (e != 0) {                                                              \
      printf("error %d at %s:%d\n", (int)e, __FILE__, __LINE__);               \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t b) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_spin(uint32_t bar, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nS_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra S_%=;\n}" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// mode 0: 2D boxes {64, R} x nb per stage; mode 1: 1D contiguous bulk copies of 16 KB x nb
__global__ void probe(const __grid_constant__ CUtensorMap map, const char* base, int mode, int R, int nb, int stg,
                      int rows_per_cta, int kblocks, unsigned long long* cyc, int spin) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[16];
  const uint32_t ring = (smem_u32(sm) + 1023) & ~1023u;
  const uint32_t sbytes = 128u * R * nb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stg; ++s) mbar_init(smem_u32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = clock64();
  const int row0 = blockIdx.x * rows_per_cta;
  // job list: for each R-row band of this CTA's rows, kblocks k-blocks (groups of nb)
  const int bands = rows_per_cta / R, steps_per_band = kblocks / nb;
  const int total = mode == 0 ? bands * steps_per_band : (1 << 20) / sbytes;
  auto issue = [&](int it, int s) {
    const uint32_t bar = smem_u32(&full[s]);
    mbar_expect(bar, sbytes);
    const int band = it / steps_per_band, kb = (it % steps_per_band) * nb;
    if (mode == 0) {
      for (int q = 0; q < nb; ++q) tma2d(ring + s * sbytes + q * 128 * R, &map, bar, (kb + q) * 64, row0 + band * R);
    } else {
      const char* src = base + (static_cast<size_t>(row0) * 4096) + static_cast<size_t>(it) * sbytes;
      for (int q = 0; q < nb; ++q) bulk1d(ring + s * sbytes + q * 128 * R, src + q * 128 * R, 128 * R, bar);
    }
  };
  for (int s = 0; s < stg && s < total; ++s) issue(s, s);
  for (int it = 0; it < total; ++it) {
    const int s = it % stg;
    if (spin) mbar_spin(smem_u32(&full[s]), (it / stg) & 1);
    else mbar_wait(smem_u32(&full[s]), (it / stg) & 1);
    if (it + stg < total) issue(it + stg, s);
  }
  cyc[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t rows = 148 * 1024;  // 148 CTAs x up to 1024 rows x 4 KB = 606 MB
  const size_t bytes = rows * 4096;
  char* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  char* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  unsigned long long* cyc;
  CK(cudaMalloc(&cyc, 148 * 8));
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", (void**)&enc, 12000, cudaEnableDefault, &q));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Case {
    int mode, R, nb, stg, ctas, rows_per_cta, kblocks, spin;
  };
  std::vector<Case> cases;
  const char* env = getenv("PROBE_SET");
  if (env && env[0] == '3') {
    for (int spin : {0, 1})
      for (int ctas : {1, 48})
        for (int kb : {8, 16, 32, 64})
          for (int stg : {2, 4, 6}) {
            const int R = kb * 1024 / 128;
            if (kb * 1024 * stg > 200 * 1024) continue;
            cases.push_back({1, R, 1, stg, ctas, 256, 32, spin});
            cases.push_back({0, R > 256 ? 256 : R, R > 256 ? R / 256 : 1, stg, ctas, 256, 32, spin});
          }
  } else if (env && env[0] == '2') {
    for (int ctas : {1, 148})
      for (int kb : {4, 8, 16, 32, 64})
        for (int nb : {1, 2, 4})
          for (int stg : {1, 2, 3, 4, 6}) {
            const int R = kb * 1024 / 128 / nb;
            if (kb * 1024 * stg > 200 * 1024) continue;
            if (256 % (R * nb) != 0 && (R * nb) % 256 != 0) continue;
            cases.push_back({1, R, nb, stg, ctas, 256, 32, 0});
          }
  } else {
  // per-CTA bytes fixed at 1 MB (a ttn=256 phase-1 job of OLMoE): R*kblocks*128 B
  for (int ctas : {1, 24, 48, 96, 148})
    for (int R : {64, 128, 256})
      for (int nb : {1, 2})
        for (int stg : {4, 6, 8, 12}) {
          if (128 * R * nb * stg > 200 * 1024) continue;
          cases.push_back({0, R, nb, stg, ctas, 256, 32, 0});
        }
  }
  printf("mode R nb stg ctas  us  GB/s_total GB/s_per_cta\n");
  for (auto& c : cases) {
    CUtensorMap map;
    cuuint64_t dims[2] = {2048, rows};
    cuuint64_t strides[1] = {4096};
    cuuint32_t box[2] = {64, (cuuint32_t)c.R > 256 ? 256u : (cuuint32_t)c.R};
    cuuint32_t es[2] = {1, 1};
    CK(enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    const int smem = 128 * c.R * c.nb * c.stg + 1024;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaMemsetAsync(flush, rep, 512 << 20));
      cudaEventRecord(e0);
      probe<<<c.ctas, 32, smem>>>(map, buf, c.mode, c.R, c.nb, c.stg, c.rows_per_cta, c.kblocks, cyc, c.spin);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    CK(cudaGetLastError());
    std::vector<unsigned long long> hc(c.ctas);
    CK(cudaMemcpy(hc.data(), cyc, 8 * c.ctas, cudaMemcpyDeviceToHost));
    unsigned long long mx = 0;
    for (auto v : hc) mx = v > mx ? v : mx;
    const double per = 1048576.0;
    const double us = best * 1e3;
    const double kus = mx / 1965.0;
    printf("spin%d %d %3d %d %2d %3d %7.2f %8.1f %7.1f | in-kernel %7.2f us %7.1f GB/s/cta\n", c.spin, c.mode, c.R, c.nb, c.stg,
           c.ctas, us, per * c.ctas / us / 1e3, per / us / 1e3, kus, per / kus / 1e3);
  }
  return 0;
}
