// ubench_tma_gather.cu -- does TMA tile::gather4 (sm_100a) add random-gather
// throughput beyond the LSU path?  (research microbenchmark, not product)
//
// Table: 4 MiB of bytes viewed as a [262144][16] uint8 tensor.  Each gather4
// fetches 4 random 16-byte rows into shared memory.  Modes:
//   tma  : every warp's lanes issue gather4s (4 rows each), STAGES deep
//   ldg  : plain random 1-byte LDG gathers (baseline)
//   mix  : warps 0..TW-1 issue gather4s, the other warps LDG gathers
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int STAGES = 4;
constexpr int WARPS = 8;

// per warp: STAGES x 32 lanes x 128 bytes = 16 KB; 8 warps = 128 KB
struct __align__(128) Smem {
  uint8_t buf[WARPS][STAGES][32][128];  // 128-byte aligned TMA destinations
  uint64_t bar[WARPS][STAGES];
};

__global__ void __launch_bounds__(WARPS * 32)
k_gather(const __grid_constant__ CUtensorMap tmap, const uint8_t *__restrict__ tab, uint32_t nrows,
         uint64_t iters, int tma_warps, uint64_t tma_iters, unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t raw[];
  Smem &sm = *reinterpret_cast<Smem *>(raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * WARPS + warp;
  unsigned long long acc = 0;
  if (warp < tma_warps) {
    if (lane == 0)
      for (int s = 0; s < STAGES; ++s)
        asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&sm.bar[warp][s])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    // iterations: each lane issues one gather4 per stage (4 rows = 4 gathers)
    const uint64_t n = tma_iters / 4;
    for (uint64_t it = 0; it < n + STAGES; ++it) {
      const int s = (int)(it % STAGES);
      const uint32_t parity = (uint32_t)((it / STAGES) & 1);
      if (it >= STAGES) {  // consume stage s (issued STAGES iterations ago)
        const uint32_t bar = smem_u32(&sm.bar[warp][s]);
        uint32_t done = 0;
        for (uint32_t spin = 0; !done; ++spin) {
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                       : "=r"(done) : "r"(bar), "r"(parity ^ 1u) : "memory");
          if (spin > (1u << 22)) {  // never hang the box: report and bail out
            if (lane == 0) atomicAdd(sink, 1ull << 32);
            return;
          }
        }
        const uint8_t *b = sm.buf[warp][s][lane];
        acc += b[0] + b[16] + b[32] + b[48];
        __syncwarp();
      }
      if (it < n) {
        const uint32_t bar = smem_u32(&sm.bar[warp][s]);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(32 * 64)
                       : "memory");
        __syncwarp();
        const uint32_t base = mix((gw << 20) ^ (uint32_t)(it * 32 + lane));
        int32_t r0 = mix(base) % nrows, r1 = mix(base + 1) % nrows, r2 = mix(base + 2) % nrows,
                r3 = mix(base + 3) % nrows;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(sm.buf[warp][s][lane])),
            "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
            : "memory");
      }
    }
  } else {
    const uint32_t mask = nrows * 16 - 1;
    for (uint64_t it = 0; it < iters; it += 8) {
      uint32_t v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(tab + (mix((gw << 20) ^ (uint32_t)(it + u) * 32 + lane) & mask));
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
  }
  if (acc == 42) *sink = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint32_t nrows = 1u << 18;  // 4 MiB
  uint8_t *tab;
  CK(cudaMalloc(&tab, (size_t)nrows * 16));
  CK(cudaMemset(tab, 1, (size_t)nrows * 16));
  unsigned long long *sink;
  CK(cudaMalloc(&sink, 8));

  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = (EncodeFn)fn;
  CUtensorMap tmap;
  cuuint64_t gdim[2] = {16, nrows};
  cuuint64_t gstride[1] = {16};
  cuuint32_t box[2] = {16, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, tab, gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode box{16,1} -> %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;

  CK(cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const uint64_t iters = 1 << 14;  // gathers per lane
  for (int blocks_per_sm : {1}) {
    for (int cfg = 0; cfg < 9; ++cfg) {
      const int tws[9] = {0, 8, 1, 1, 1, 2, 2, 2, 4};
      const double frac[9] = {0, 1, 0.5, 0.8, 1.2, 0.3, 0.4, 0.5, 0.2};
      const int tw = tws[cfg];
      const uint64_t tma_iters = ((uint64_t)(iters * frac[cfg]) + 3) & ~3ull;
      const int grid = sms * blocks_per_sm;
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        k_gather<<<grid, WARPS * 32, sizeof(Smem)>>>(tmap, tab, nrows, iters, tw, tma_iters, sink);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        unsigned long long hs;
        CK(cudaMemcpy(&hs, sink, 8, cudaMemcpyDeviceToHost));
        if (hs >> 32) { printf("TMA wait timed out (%llu warps)\n", hs >> 32); return 2; }
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      const double gathers = (double)grid * 32 * ((WARPS - tw) * (double)iters + tw * (double)tma_iters);
      printf("tma_warps=%d/%d tma_iters=%.2fx: %.3f ms  %.1f Ggathers/s\n", tw, WARPS, frac[cfg],
             best, gathers / best / 1e6);
    }
  }
  return 0;
}
