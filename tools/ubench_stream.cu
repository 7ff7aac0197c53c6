// ubench_stream.cu -- what bounds the staged plan's block stream (round 2).
// 148 persistent CTAs (one per SM), one producer lane issuing TMA bulk copies
// of a table block (from a 4 MiB L2-resident array, the same block for every
// CTA in a phase, as in k_estimate_plan) and of the CTA's own entry chunk
// (from a 300 MB DRAM array, each CTA a contiguous region) into S stages;
// 16 consumer warps wait for each stage, optionally touch it (one 4-byte
// shared load per lane per 128 B: TOUCH=1), and release it.  L2 is flushed
// before every timed launch.  Prints us per launch for the (T, E, S) given.
// usage: ubench_stream T_bytes E_bytes stages phases [touch]
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mwait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                 : "=r"(done) : "r"(su32(bar)), "r"(parity) : "memory");
}

constexpr int kW = 16;

__global__ void __launch_bounds__(kW * 32 + 32, 1)
k_stream(const uint8_t *tab, const uint8_t *ent, uint32_t T, uint32_t E, uint32_t S,
         uint32_t phases, int touch, unsigned long long *sink) {
  // touch = 2: the entries are NOT staged; the consumer warps read their
  // share of each phase's entry chunk straight from global memory (16-byte
  // loads), the producer prefetches the next chunk into L2
  const bool ldg = touch == 2;
  const uint32_t Es = ldg ? 0u : E;
  extern __shared__ __align__(128) uint8_t raw[];
  uint64_t *full = reinterpret_cast<uint64_t *>(raw);
  uint64_t *empty = full + 16;
  uint8_t *buf = raw + 256;
  const uint32_t stage = ((T + (touch == 2 ? 0u : E)) + 127u) & ~127u;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (uint32_t b = 0; b < S; ++b) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[b])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(&empty[b])), "r"(kW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t *my_ent = ent + (uint64_t)blockIdx.x * phases * E;
  if (w == kW) {
    if (lane == 0) {
      for (uint32_t ph = 0; ph < phases; ++ph) {
        const uint32_t b = ph % S;
        if (ph >= S) mwait(&empty[b], ((ph / S) + 1u) & 1u);
        const uint32_t fb = su32(&full[b]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb), "r"(T + Es) : "memory");
        uint8_t *dst = buf + (size_t)b * stage;
        if (T)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(dst)), "l"(tab + (uint64_t)(ph % 64) * T), "r"(T), "r"(fb) : "memory");
        if (Es)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(dst + T)), "l"(my_ent + (uint64_t)ph * E), "r"(E), "r"(fb) : "memory");
        if (ldg && ph + 1 < phases)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(my_ent + (uint64_t)(ph + 1) * E),
                       "r"(E) : "memory");
      }
    }
    return;
  }
  uint32_t acc = 0;
  for (uint32_t ph = 0; ph < phases; ++ph) {
    const uint32_t b = ph % S;
    mwait(&full[b], (ph / S) & 1u);
    if (ldg) {
      const uint4 *q = reinterpret_cast<const uint4 *>(my_ent + (uint64_t)ph * E);
      const uint32_t n16 = E / 16u;
#pragma unroll 4
      for (uint32_t i = w * 32 + lane; i < n16; i += kW * 32) {
        const uint4 v = __ldcs(q + i);
        acc += v.x ^ v.w;
      }
    } else if (touch) {
      const uint32_t *p = reinterpret_cast<const uint32_t *>(buf + (size_t)b * stage);
      for (uint32_t i = w * 32 + lane; i < (T + E) / 128u; i += kW * 32) acc += p[i * 32];
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&empty[b])) : "memory");
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}


// Decoupled rings (round 2): table blocks in ST stages, entry chunks in SE
// stages, each with its own full/empty barriers, so the DRAM-bound entry
// stream can run further ahead than the L2-bound table stream.
__global__ void __launch_bounds__(kW * 32 + 32, 1)
k_stream2(const uint8_t *tab, const uint8_t *ent, uint32_t T, uint32_t E, uint32_t ST,
          uint32_t SE, uint32_t phases, unsigned long long *sink) {
  extern __shared__ __align__(128) uint8_t raw[];
  uint64_t *tfull = reinterpret_cast<uint64_t *>(raw), *tempty = tfull + 8;
  uint64_t *efull = tfull + 16, *eempty = tfull + 24;
  uint8_t *tbuf = raw + 256;
  const uint32_t estage = (E + 127u) & ~127u;
  uint8_t *ebuf = tbuf + (size_t)ST * T;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (uint32_t b = 0; b < ST; ++b) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&tfull[b])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(&tempty[b])), "r"(kW));
    }
    for (uint32_t b = 0; b < SE; ++b) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&efull[b])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(&eempty[b])), "r"(kW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t *my_ent = ent + (uint64_t)blockIdx.x * phases * E;
  if (w == kW) {
    if (lane == 0) {
      // entries run up to SE phases ahead, tables up to ST
      uint32_t te = 0, tt = 0;
      while (tt < phases) {
        while (te < phases && te < tt + SE) {
          const uint32_t b = te % SE;
          if (te >= SE) mwait(&eempty[b], ((te / SE) + 1u) & 1u);
          const uint32_t fb = su32(&efull[b]);
          asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb), "r"(E) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(ebuf + (size_t)b * estage)), "l"(my_ent + (uint64_t)te * E), "r"(E), "r"(fb) : "memory");
          ++te;
        }
        const uint32_t b = tt % ST;
        if (tt >= ST) mwait(&tempty[b], ((tt / ST) + 1u) & 1u);
        const uint32_t fb = su32(&tfull[b]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb), "r"(T) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(tbuf + (size_t)b * T)), "l"(tab + (uint64_t)(tt % 64) * T), "r"(T), "r"(fb) : "memory");
        ++tt;
      }
    }
    return;
  }
  uint32_t acc = 0;
  for (uint32_t ph = 0; ph < phases; ++ph) {
    mwait(&tfull[ph % ST], (ph / ST) & 1u);
    mwait(&efull[ph % SE], (ph / SE) & 1u);
    acc += tbuf[(size_t)(ph % ST) * T + lane] + ebuf[(size_t)(ph % SE) * estage + lane];
    __syncwarp();
    if (lane == 0) {
      asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&tempty[ph % ST])) : "memory");
      asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(su32(&eempty[ph % SE])) : "memory");
    }
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

// plain streaming read of `bytes` with 16-byte loads, UNROLL in flight per thread
__global__ void __launch_bounds__(1024) k_ldg(const uint4 *p, uint64_t n16, unsigned long long *sink) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x ^ v[u].w;
  }
  for (; i < n16; i += stride) acc += __ldcs(p + i).y;
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char **argv) {
  if (argc > 1 && argv[1][0] == 'R') {  // R T E ST SE phases: decoupled rings
    const uint32_t T = atoi(argv[2]), E = atoi(argv[3]), ST = atoi(argv[4]), SE = atoi(argv[5]),
                   phases = atoi(argv[6]);
    uint8_t *tab, *ent, *flush;
    unsigned long long *sink;
    CK(cudaMalloc(&tab, 64ull * T));
    CK(cudaMalloc(&ent, 148ull * phases * E));
    CK(cudaMalloc(&flush, 512ull << 20));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(tab, 1, 64ull * T));
    CK(cudaMemset(ent, 2, 148ull * phases * E));
    const size_t smem = 256 + (size_t)ST * T + (size_t)SE * ((E + 127u) & ~127u);
    CK(cudaFuncSetAttribute(k_stream2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float sum = 0;
    for (int r = 0; r < 12; ++r) {
      CK(cudaMemsetAsync(flush, r, 512ull << 20));
      CK(cudaEventRecord(a));
      k_stream2<<<148, kW * 32 + 32, smem>>>(tab, ent, T, E, ST, SE, phases, sink);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (r >= 2) sum += ms;
    }
    CK(cudaGetLastError());
    printf("rings T=%u x %u, E=%u x %u, phases=%u, smem=%zu: %.1f us\n", T, ST, E, SE, phases, smem,
           1e3 * sum / 10);
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'L') {  // L <bytes>: the LDG read rate
    const uint64_t bytes = strtoull(argv[2], nullptr, 10);
    uint8_t *src, *flush;
    unsigned long long *sink;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMalloc(&flush, 512ull << 20));
    CK(cudaMalloc(&sink, 8));
    CK(cudaMemset(src, 3, bytes));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float sum = 0;
    for (int r = 0; r < 12; ++r) {
      CK(cudaMemsetAsync(flush, r, 512ull << 20));
      CK(cudaEventRecord(a));
      k_ldg<<<148 * 2, 1024>>>(reinterpret_cast<const uint4 *>(src), bytes / 16, sink);
      CK(cudaEventRecord(b));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (r >= 2) sum += ms;
    }
    printf("LDG read %llu B: %.1f us, %.2f TB/s\n", (unsigned long long)bytes, 1e3 * sum / 10,
           bytes / (sum / 10 * 1e-3) / 1e12);
    return 0;
  }
  const uint32_t T = atoi(argv[1]), E = atoi(argv[2]), S = atoi(argv[3]), phases = atoi(argv[4]);
  const int touch = argc > 5 ? atoi(argv[5]) : 0;
  const int ctas = 148;
  uint8_t *tab, *ent, *flush;
  unsigned long long *sink;
  CK(cudaMalloc(&tab, 64ull * (T ? T : 1)));
  CK(cudaMalloc(&ent, (uint64_t)ctas * phases * (E ? E : 1)));
  CK(cudaMalloc(&flush, 512ull << 20));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(tab, 1, 64ull * (T ? T : 1)));
  CK(cudaMemset(ent, 2, (uint64_t)ctas * phases * (E ? E : 1)));
  const uint32_t stage = ((T + (touch == 2 ? 0u : E)) + 127u) & ~127u;
  const size_t smem = 256 + (size_t)S * stage;
  CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  float best = 1e30f, sum = 0;
  const int reps = 10;
  for (int r = 0; r < reps + 2; ++r) {
    CK(cudaMemsetAsync(flush, r, 512ull << 20));
    CK(cudaEventRecord(a));
    k_stream<<<ctas, kW * 32 + 32, smem>>>(tab, ent, T, E, S, phases, touch, sink);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (r >= 2) {
      sum += ms;
      if (ms < best) best = ms;
    }
  }
  CK(cudaGetLastError());
  const double bytes = (double)ctas * phases * (T + E);
  printf("T=%u E=%u S=%u phases=%u touch=%d smem=%zu: %.1f us (best %.1f), %.2f TB/s into SMs, entries %.2f TB/s\n",
         T, E, S, phases, touch, smem, 1e3 * sum / reps, 1e3 * best, bytes / (sum / reps * 1e-3) / 1e12,
         (double)ctas * phases * E / (sum / reps * 1e-3) / 1e12);
  return 0;
}
