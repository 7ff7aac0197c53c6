// ubench_plan.cu -- can a plan-based estimate beat the L2 gather ceiling?
// (research microbenchmark, not product)
//
// 148 persistent CTAs x 512 threads.  Each thread owns SLOTS hosts whose
// packed sums (S | V << 40) live in shared memory.  The 4 MiB register table
// is streamed through shared memory in 64 KB blocks (TMA bulk copies, double
// buffered); per block, each warp reads its padded, lane-interleaved plan
// entries (offset | slot << 16, 0xFFFFFFFF = padding), gathers the register
// from shared memory and adds into the owning thread's accumulator.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

#ifndef UNR
#define UNR 4
#endif
constexpr int THREADS = 512, WARPS = THREADS / 32, SLOTS = 7, BLOCK = 1 << 16, PHASES = 64;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

struct __align__(128) Smem {
  uint8_t tab[2][BLOCK];
  unsigned long long acc[SLOTS][THREADS];
  uint64_t bar[2];
};

__global__ void __launch_bounds__(THREADS, 1)
k_plan(const uint8_t *__restrict__ table, const uint32_t *__restrict__ entries,
       const uint32_t *__restrict__ base, const uint16_t *__restrict__ kmax, uint32_t L,
       unsigned long long *out) {
  extern __shared__ __align__(128) uint8_t raw[];
  Smem &sm = *reinterpret_cast<Smem *>(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int s = 0; s < SLOTS; ++s) sm.acc[s][tid] = 0ull;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int ph) {
    const int b = ph & 1;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.bar[b])),
                 "r"(BLOCK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sm.tab[b])), "l"(table + (size_t)ph * BLOCK), "r"(BLOCK),
                 "r"(smem_u32(&sm.bar[b])) : "memory");
  };
  if (tid == 0) issue(0);
  for (int ph = 0; ph < PHASES; ++ph) {
    const int b = ph & 1;
    if (tid == 0 && ph + 1 < PHASES) issue(ph + 1);
    const uint32_t parity = (ph >> 1) & 1;
    uint32_t done = 0;
    for (uint32_t spin = 0; !done; ++spin) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(done) : "r"(smem_u32(&sm.bar[b])), "r"(parity) : "memory");
      if (spin > (1u << 24)) { if (tid == 0) atomicAdd(out, 1ull << 40); return; }
    }
    const size_t key = ((size_t)blockIdx.x * PHASES + ph) * WARPS + warp;
    const uint32_t *e = entries + base[key] + lane;
    const uint32_t kk = kmax[key];
    const uint8_t *tab = sm.tab[b];
    uint32_t k = 0;
    for (; k + UNR <= kk; k += UNR) {
      uint32_t v[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) v[u] = __ldcs(e + (k + u) * 32);
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (v[u] != 0xFFFFFFFFu) {
          const uint32_t M = tab[v[u] & 0xFFFFu];
          sm.acc[v[u] >> 16][tid] += (1ull << (L - M)) + ((unsigned long long)(M == 0) << 40);
        }
    }
    for (; k < kk; ++k) {
      const uint32_t v = __ldcs(e + k * 32);
      if (v != 0xFFFFFFFFu) {
        const uint32_t M = tab[v & 0xFFFFu];
        sm.acc[v >> 16][tid] += (1ull << (L - M)) + ((unsigned long long)(M == 0) << 40);
      }
    }
    __syncthreads();  // buffer b is refilled two phases later
  }
  unsigned long long t = 0;
  for (int s = 0; s < SLOTS; ++s) t += sm.acc[s][tid];
  if (t == 42) *out = t;
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t table_bytes = (size_t)PHASES * BLOCK;  // 4 MiB
  uint8_t *table;
  CK(cudaMalloc(&table, table_bytes));
  std::vector<uint8_t> ht(table_bytes);
  for (size_t i = 0; i < table_bytes; ++i) ht[i] = (uint8_t)(1 + (i * 2654435761u >> 28) % 6);
  CK(cudaMemcpy(table, ht.data(), table_bytes, cudaMemcpyHostToDevice));
  // synthetic plan: 64M real entries over sms*PHASES*WARPS warps, lane counts ~Poisson(mean)
  const double total = 64.0 * (1 << 20);
  const double per_lane = total / ((double)sms * PHASES * THREADS);
  const size_t nkeys = (size_t)sms * PHASES * WARPS;
  std::vector<uint32_t> base(nkeys);
  std::vector<uint16_t> kmax(nkeys);
  std::vector<uint32_t> ent;
  ent.reserve((size_t)(total * 1.8));
  uint64_t rng = 88172645463325252ull;
  auto rnd = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
  auto poisson = [&](double lam) {  // Knuth, fine for lam ~ 14
    double L = exp(-lam), p = 1.0;
    int k = 0;
    do { ++k; p *= (double)(rnd() >> 11) * 0x1.0p-53; } while (p > L);
    return k - 1;
  };
  size_t real = 0;
  for (size_t key = 0; key < nkeys; ++key) {
    int c[32], mx = 0;
    for (int l = 0; l < 32; ++l) { c[l] = poisson(per_lane); mx = c[l] > mx ? c[l] : mx; }
    base[key] = (uint32_t)ent.size();
    kmax[key] = (uint16_t)mx;
    for (int k = 0; k < mx; ++k)
      for (int l = 0; l < 32; ++l) {
        if (k < c[l]) {
          ent.push_back((uint32_t)(rnd() & 0xFFFFu) | (uint32_t)((rnd() % SLOTS) << 16));
          ++real;
        } else {
          ent.push_back(0xFFFFFFFFu);
        }
      }
  }
  printf("entries: %zu real, %zu padded (%.2fx), %.1f MB\n", real, ent.size(),
         (double)ent.size() / real, ent.size() * 4.0 / 1e6);
  uint32_t *d_ent, *d_base;
  uint16_t *d_k;
  unsigned long long *out;
  CK(cudaMalloc(&d_ent, ent.size() * 4));
  CK(cudaMalloc(&d_base, nkeys * 4));
  CK(cudaMalloc(&d_k, nkeys * 2));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(out, 0, 8));
  CK(cudaMemcpy(d_ent, ent.data(), ent.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_base, base.data(), nkeys * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_k, kmax.data(), nkeys * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  void *flush;
  CK(cudaMalloc(&flush, 512u << 20));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(flush, rep, 512u << 20));
    CK(cudaEventRecord(e0));
    k_plan<<<sms, THREADS, sizeof(Smem)>>>(table, d_ent, d_base, d_k, 25, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    unsigned long long h;
    CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
    if (h >> 40) { printf("mbarrier timeout\n"); return 2; }
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("plan estimate (L2 flushed): %.3f ms = %.1f G real gathers/s\n", ms, real / ms / 1e6);
  }
  return 0;
}
