// ubench_gather.cu -- microbenchmarks that size the VBDR estimate and scan
// kernels on B200 (not part of the product; run by tools/ubench.sh on a box).
//
//  gather_ldg    : random 1-byte LDG gathers from a T-byte table (the estimate's
//                  access pattern, table = regmax)
//  gather_dsmem  : the table packed 6 x 5-bit entries per u32 word and spread
//                  over the shared memory of a C-CTA cluster; random loads via
//                  ld.shared::cluster (mapa)
//  gather_smem   : random loads from the CTA's own shared memory (upper bound)
//  red_max       : random atomicMax (RED) at u32 addresses in an array of A
//                  bytes (the scan's update pattern; BASELINE.md random-RED ceiling)
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du; x ^= x >> 15; x *= 0x846CA68Bu; x ^= x >> 16;
  return x;
}

// NQ independent gathers per lane per iteration (like k_estimate with g=128)
template <int NQ>
__global__ void __launch_bounds__(256) gather_ldg(const uint8_t *__restrict__ t, uint32_t mask,
                                                  uint64_t n_items, unsigned long long *sink) {
  unsigned long long acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_items; i += stride) {
    uint32_t v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = __ldg(t + (mix((uint32_t)i * NQ + q) & mask));
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc += 1ull << (25 - (v[q] & 15));
  }
  if (acc == 42) *sink = acc;
}

template <int NQ>
__global__ void __launch_bounds__(256) gather_dsmem(const uint32_t *__restrict__ packed,
                                                    uint32_t words_per_cta, uint32_t local_bits,
                                                    uint64_t n_items, unsigned long long *sink) {
  extern __shared__ uint32_t tab[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  const uint32_t csize = cl.num_blocks();
  for (uint32_t w = threadIdx.x; w < words_per_cta; w += blockDim.x)
    tab[w] = packed[(uint64_t)rank * words_per_cta + w];
  cl.sync();
  unsigned long long acc = 0;
  const uint32_t lmask = (1u << local_bits) - 1u;
  const uint64_t n_clusters = gridDim.x / csize;
  const uint64_t cid = blockIdx.x / csize;
  const uint64_t stride = n_clusters * csize * blockDim.x;
  for (uint64_t i = (cid * csize + rank) * blockDim.x + threadIdx.x; i < n_items; i += stride) {
    uint32_t v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t p = mix((uint32_t)i * NQ + q);
      const uint32_t owner = (p >> local_bits) & (csize - 1);
      const uint32_t li = p & lmask;
      const uint32_t word = li / 6u, sh = 5u * (li - word * 6u);
      const uint32_t *remote = cl.map_shared_rank(tab + word, owner);
      v[q] = (*remote >> sh) & 31u;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc += 1ull << (25 - (v[q] & 15));
  }
  cl.sync();
  if (acc == 42) *sink = acc;
}

template <int NQ>
__global__ void __launch_bounds__(256) gather_smem(const uint32_t *__restrict__ packed,
                                                   uint32_t words, uint64_t n_items,
                                                   unsigned long long *sink) {
  extern __shared__ uint32_t tab[];
  for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) tab[w] = packed[w];
  __syncthreads();
  unsigned long long acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_items; i += stride) {
    uint32_t v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t li = mix((uint32_t)i * NQ + q) % (words * 6u);
      const uint32_t word = li / 6u, sh = 5u * (li - word * 6u);
      v[q] = (tab[word] >> sh) & 31u;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc += 1ull << (25 - (v[q] & 15));
  }
  if (acc == 42) *sink = acc;
}

__global__ void __launch_bounds__(256) red_max(uint32_t *a, uint32_t mask, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t h = mix((uint32_t)i ^ 0x9E3779B9u);
    atomicMax(a + (h & mask), (uint32_t)(i & 0xFFFF));
  }
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  unsigned long long *sink;
  CK(cudaMalloc(&sink, 8));
  const uint64_t n_gathers = 64ull << 20;  // the caida estimate: 500k hosts x 128
  uint8_t *tab;
  CK(cudaMalloc(&tab, 256u << 20));
  CK(cudaMemset(tab, 3, 256u << 20));
  void *flush;
  CK(cudaMalloc(&flush, 512u << 20));

  for (uint32_t tbytes : {4u << 20, 64u << 20, 256u << 20}) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemset(flush, rep, 512u << 20));
      CK(cudaEventRecord(e0));
      gather_ldg<4><<<sms * 8, 256>>>(tab, tbytes - 1, n_gathers / 4, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      if (rep) printf("gather_ldg table=%uMiB: %.3f ms  %.1f Ggathers/s\n", tbytes >> 20,
                      time_ms(e0, e1), n_gathers / time_ms(e0, e1) / 1e6);
    }
  }

  // DSMEM: table of 2^22 entries, 5 bits each, 6 per word
  for (int csize : {8, 16}) {
    const uint32_t entries = 1u << 22;
    const uint32_t local_bits = 22 - (csize == 16 ? 4 : 3);
    const uint32_t words_per_cta = ((1u << local_bits) + 5) / 6;
    const size_t smem = words_per_cta * 4ull;
    if (smem > 227 * 1024) {
      printf("gather_dsmem cluster=%d: table needs %zu KB per CTA (> 227 KB), skipped\n", csize,
             smem / 1024);
      continue;
    }
    uint32_t *packed;
    CK(cudaMalloc(&packed, (size_t)words_per_cta * csize * 4));
    CK(cudaMemset(packed, 0x11, (size_t)words_per_cta * csize * 4));
    auto kern = gather_dsmem<4>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (csize > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int max_clusters = 0;
    cfg.gridDim = dim3(csize);
    CK(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
    for (int blocks_mult : {1, 2}) {
      for (int threads : {256, 512, 1024}) {
        if (threads > 256) continue;  // launch bounds
        cfg.gridDim = dim3(max_clusters * csize * blocks_mult);
        if (blocks_mult > 1) continue;
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          CK(cudaEventRecord(e0));
          CK(cudaLaunchKernelEx(&cfg, kern, (const uint32_t *)packed, words_per_cta, local_bits,
                                n_gathers / 4, sink));
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms = time_ms(e0, e1);
          if (ms < best) best = ms;
        }
        printf("gather_dsmem cluster=%d max_active_clusters=%d (%d SMs) smem=%zuKB: %.3f ms  "
               "%.1f Ggathers/s\n", csize, max_clusters, max_clusters * csize, smem / 1024, best,
               n_gathers / best / 1e6);
      }
    }
    CK(cudaFree(packed));
  }

  {
    const uint32_t words = 40000;  // 160 KB
    uint32_t *packed;
    CK(cudaMalloc(&packed, words * 4));
    CK(cudaMemset(packed, 0x11, words * 4));
    CK(cudaFuncSetAttribute(gather_smem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            words * 4));
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(e0));
      gather_smem<4><<<sms, 256, words * 4>>>(packed, words, n_gathers / 4, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = time_ms(e0, e1);
      if (ms < best) best = ms;
    }
    printf("gather_smem local 160KB: %.3f ms  %.1f Ggathers/s\n", best, n_gathers / best / 1e6);
  }

  uint32_t *arr;
  CK(cudaMalloc(&arr, 1ull << 30));
  CK(cudaMemset(arr, 0, 1ull << 30));
  const uint64_t n_red = 100ull << 20;
  for (uint64_t abytes : {16ull << 20, 48ull << 20, 256ull << 20, 1ull << 30}) {
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaMemset(flush, rep, 512u << 20));
      CK(cudaEventRecord(e0));
      red_max<<<sms * 8, 256>>>(arr, (uint32_t)(abytes / 4 - 1), n_red);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      if (rep) printf("red_max array=%lluMiB: %.3f ms  %.1f Gatomics/s\n",
                      (unsigned long long)(abytes >> 20), time_ms(e0, e1),
                      n_red / time_ms(e0, e1) / 1e6);
    }
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
