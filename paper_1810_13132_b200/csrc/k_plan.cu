// k_plan.cu -- plan-based estimation for a fixed host list (sm_100a),
// compiled with -fmad=false like k_estimate.cu (same fp64 finish).
//
// The gather estimate (k_estimate.cu) is bound by the SM's L1-to-L2 request
// rate: one 32-byte sector request per 1-byte register read.  For pools whose
// register array is small (n_phys <= 2^22, 4 MiB) the same sums can be formed
// from shared memory instead:
//   * a PLAN, built once per host list, assigns every host to one thread of
//     one of `ctas` persistent CTAs (host h -> thread h % T, slot h / T) and
//     lists, for every (CTA, register block of 2^16) phase, the entries
//     (offset in block | slot << 16) of each thread's (host, i) gathers that
//     fall in that block (Alg.5 / Alg.3 indices, precomputed);
//   * per slice, each CTA streams the register array through shared memory
//     one 64 KB block at a time (TMA bulk copies, double buffered, mbarrier),
//     together with its entries for that block, and every thread adds
//     2^(L - M) (or M for LogLog/PCSA) and the zero count into its hosts'
//     packed accumulators (S | V << 40) in shared memory -- no atomics, no
//     L2 gathers.  The last step is the fp64 finish of k_estimate.
// Integer sums make the result bit-identical to the gather kernel.
#include "vbdr_dev.cuh"

using namespace vbdr_dev;
using vbdr_launch::EstParams;
using vbdr_launch::PlanLayout;

namespace {

constexpr int kT = vbdr_launch::kPlanThreads;  // 512
constexpr int kSlots = vbdr_launch::kPlanSlots;  // 7
constexpr int kCap = vbdr_launch::kPlanEntCap;   // entries per (CTA, phase) buffer
constexpr int kStride = kT + 4;                  // run starts per key, 16-byte padded

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---------------------------------------------------------------- build
struct BuildArgs {
  const uint32_t *hosts;
  uint64_t n;
  uint32_t g, A0, mask, block_log2, phases, ctas;
  uint32_t *counts;      // [ctas * phases * kT]
  uint32_t *starts;      // [ctas * phases * kStride]
  uint32_t *range_base;  // [ctas * phases + 1]
  uint32_t *entries;
  uint32_t *max_range;   // scalar
};

__device__ __forceinline__ void locate_entry(const BuildArgs &a, uint64_t h, uint32_t i,
                                             uint64_t &key, uint32_t &thread, uint32_t &val) {
  const uint64_t T = (uint64_t)a.ctas * kT;
  const uint64_t t = h % T;
  const uint32_t slot = (uint32_t)(h / T);
  const uint32_t cta = (uint32_t)(t / kT);
  thread = (uint32_t)(t % kT);
  const uint32_t s1 = fmix32(i ^ a.A0);                         // Alg.3
  const uint32_t pidx = fmix32(__ldg(a.hosts + h) ^ s1) & a.mask;  // Alg.3
  const uint32_t phase = pidx >> a.block_log2;
  key = (uint64_t)cta * a.phases + phase;
  val = (pidx & ((1u << a.block_log2) - 1u)) | (slot << 16);
}

__global__ void k_plan_count(BuildArgs a) {
  const uint64_t total = a.n * a.g;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    uint64_t key;
    uint32_t thread, val;
    locate_entry(a, x / a.g, (uint32_t)(x % a.g), key, thread, val);
    atomicAdd(a.counts + key * kT + thread, 1u);
  }
}

// One block per key: exclusive scan of the kT thread counts -> run starts;
// the key's total (padded to a multiple of 4 entries: 16-byte ranges).
__global__ void __launch_bounds__(kT) k_plan_starts(BuildArgs a, uint32_t *range_size) {
  __shared__ uint32_t warp_sum[kT / 32];
  const uint64_t key = blockIdx.x;
  const uint32_t c = a.counts[key * kT + threadIdx.x];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= (uint32_t)off) x += y;
  }
  if (lane == 31) warp_sum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t v = lane < kT / 32 ? warp_sum[lane] : 0u;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= (uint32_t)off) v += y;
    }
    if (lane < kT / 32) warp_sum[lane] = v;
  }
  __syncthreads();
  const uint32_t incl = x + (w > 0 ? warp_sum[w - 1] : 0u);
  a.starts[key * kStride + threadIdx.x] = incl - c;
  if (threadIdx.x == kT - 1) {
    a.starts[key * kStride + kT] = incl;
    range_size[key] = (incl + 3u) & ~3u;
    atomicMax(a.max_range, incl);
  }
  a.counts[key * kT + threadIdx.x] = 0u;  // reused as fill cursors
}

// Single block: exclusive scan of the range sizes -> range_base (u32 entries).
__global__ void __launch_bounds__(1024) k_plan_bases(BuildArgs a, const uint32_t *range_size,
                                                     uint64_t nkeys) {
  __shared__ uint32_t carry;
  __shared__ uint32_t warp_sum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (uint64_t base = 0; base < nkeys; base += 1024) {
    const uint64_t k = base + threadIdx.x;
    const uint32_t c = k < nkeys ? range_size[k] : 0u;
    uint32_t x = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= (uint32_t)off) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t v = warp_sum[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= (uint32_t)off) v += y;
      }
      warp_sum[lane] = v;
    }
    __syncthreads();
    const uint32_t incl = x + (w > 0 ? warp_sum[w - 1] : 0u);
    if (k < nkeys) a.range_base[k] = carry + incl - c;
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.range_base[nkeys] = carry;
}

__global__ void k_plan_fill(BuildArgs a) {
  const uint64_t total = a.n * a.g;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    uint64_t key;
    uint32_t thread, val;
    locate_entry(a, x / a.g, (uint32_t)(x % a.g), key, thread, val);
    const uint32_t k = atomicAdd(a.counts + key * kT + thread, 1u);
    a.entries[a.range_base[key] + a.starts[key * kStride + thread] + k] = val;
  }
}

// --------------------------------------------------------------- estimate
__device__ __forceinline__ double hll_finish(double agg, double D, double lc, uint64_t V,
                                             double s) {
  double E = __ddiv_rn(agg, D);
  if (E <= lc && V > 0) E = __dmul_rn(s, log(__ddiv_rn(s, (double)V)));
  return E;
}

template <int BLOCK_LOG2>
struct __align__(128) PlanSmem {
  uint8_t tab[2][1 << BLOCK_LOG2];
  uint32_t ent[2][kCap];
  uint32_t start[2][kStride];
  unsigned long long acc[kSlots][kT];
  uint64_t bar[2];
  double etot_z;
};

template <int BLOCK_LOG2, bool SUMS>
__global__ void __launch_bounds__(kT, 1)
k_estimate_plan(EstParams e, PlanLayout pl, uint64_t n, double *__restrict__ out,
                unsigned long long *__restrict__ outS, uint32_t *__restrict__ outV,
                unsigned long long *__restrict__ err) {
  constexpr uint32_t BLOCK = 1u << BLOCK_LOG2;
  pdl_wait();
  extern __shared__ __align__(128) uint8_t raw[];
  PlanSmem<BLOCK_LOG2> &sm = *reinterpret_cast<PlanSmem<BLOCK_LOG2> *>(raw);
  const int tid = threadIdx.x;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) sm.acc[s][tid] = 0ull;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!SUMS) {
      const unsigned long long St = e.acc[0], Vt = e.acc[1];
      double Et;
      if (e.est == 0u) {
        Et = hll_finish(e.azz, __dmul_rn((double)St, e.inv2L), e.lc_z, Vt, e.z);
      } else {
        Et = __dmul_rn(e.coef_z, exp2(__ddiv_rn((double)St, e.z)));
      }
      sm.etot_z = __ddiv_rn(Et, e.z);
    }
  }
  __syncthreads();
  const uint32_t phases = pl.phases;
  auto bulk = [&](void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
  };
  auto issue = [&](uint32_t ph) {
    const int b = ph & 1;
    const uint64_t key = (uint64_t)blockIdx.x * phases + ph;
    const uint32_t e0 = pl.range_base[key], e1 = pl.range_base[key + 1];
    const uint32_t ebytes = (e1 - e0) * 4u;  // ranges are multiples of 4 entries
    const uint32_t sbytes = kStride * 4u;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.bar[b])),
                 "r"(BLOCK + ebytes + sbytes)
                 : "memory");
    bulk(sm.tab[b], e.regmax + (uint64_t)ph * BLOCK, BLOCK, &sm.bar[b]);
    if (ebytes) bulk(sm.ent[b], pl.entries + e0, ebytes, &sm.bar[b]);
    bulk(sm.start[b], pl.starts + key * kStride, sbytes, &sm.bar[b]);
  };
  if (tid == 0) issue(0);
  for (uint32_t ph = 0; ph < phases; ++ph) {
    const int b = ph & 1;
    if (tid == 0 && ph + 1 < phases) issue(ph + 1);  // buffer freed by the sync of phase ph-1
    const uint32_t parity = (ph >> 1) & 1u;
    uint32_t done = 0;
    for (uint32_t spin = 0; !done; ++spin) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
          : "=r"(done)
          : "r"(smem_u32(&sm.bar[b])), "r"(parity)
          : "memory");
      if (spin > (1u << 26)) {  // a lost transfer must not hang the GPU: report and stop
        if (tid == 0) atomicAdd(err, 1ull);
        return;
      }
    }
    const uint8_t *tab = sm.tab[b];
    const uint32_t k0 = sm.start[b][tid], k1 = sm.start[b][tid + 1];
    for (uint32_t k = k0; k < k1; ++k) {
      const uint32_t v = sm.ent[b][k];
      const uint32_t M = tab[v & (BLOCK - 1u)];
      const unsigned long long c =
          e.est == 0u ? 1ull << (e.L - M) : (unsigned long long)M;  // HLL / LogLog, PCSA
      sm.acc[v >> 16][tid] += c + ((unsigned long long)(M == 0u) << 40);
    }
    __syncthreads();
  }
  pdl_trigger();
  const uint64_t T = (uint64_t)gridDim.x * kT;
  const uint64_t t = (uint64_t)blockIdx.x * kT + tid;
  const double g = (double)e.g;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    const uint64_t h = (uint64_t)s * T + t;
    if (h >= n) break;
    const unsigned long long packed = sm.acc[s][tid];
    const unsigned long long S = packed & ((1ull << 40) - 1ull);
    const uint32_t V = (uint32_t)(packed >> 40);
    if constexpr (SUMS) {
      outS[h] = S;
      outV[h] = V;
    } else {
      double Es;
      if (e.est == 0u) {
        Es = hll_finish(e.agg, __dmul_rn((double)S, e.inv2L), e.lc_g, V, g);
      } else {
        Es = __dmul_rn(e.coef_g, exp2(__ddiv_rn((double)S, g)));
      }
      const double est = __dmul_rn(e.C, __dsub_rn(__ddiv_rn(Es, g), sm.etot_z));
      out[h] = est > 0.0 ? est : 0.0;
    }
  }
}

template <int BL>
cudaError_t launch_est(const EstParams &e, const PlanLayout &pl, uint64_t n, double *out,
                       unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  const size_t smem = sizeof(PlanSmem<BL>);
  auto kern = outS ? k_estimate_plan<BL, true> : k_estimate_plan<BL, false>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  return launch(kern, dim3(pl.ctas), dim3(kT), smem, s, e, pl, n, out, outS, outV, pl.error);
}

}  // namespace

namespace vbdr_launch {

cudaError_t plan_build(const PlanLayout &pl, const uint32_t *hosts, uint64_t n, uint32_t g,
                       uint32_t A0, uint32_t mask, uint32_t *range_size_scratch,
                       cudaStream_t s) {
  BuildArgs a{};
  a.hosts = hosts;
  a.n = n;
  a.g = g;
  a.A0 = A0;
  a.mask = mask;
  a.block_log2 = pl.block_log2;
  a.phases = pl.phases;
  a.ctas = pl.ctas;
  a.counts = pl.counts;
  a.starts = pl.starts;
  a.range_base = pl.range_base;
  a.entries = pl.entries;
  a.max_range = pl.max_range;
  const uint64_t nkeys = (uint64_t)pl.ctas * pl.phases;
  cudaError_t e = cudaMemsetAsync(pl.counts, 0, nkeys * kT * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pl.max_range, 0, 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pl.error, 0, 8, s);
  if (e != cudaSuccess) return e;
  const uint64_t total = n * g;
  const uint32_t grid = (uint32_t)((total + 255) / 256 < 148ull * 16 ? (total + 255) / 256 : 148ull * 16);
  k_plan_count<<<grid ? grid : 1, 256, 0, s>>>(a);
  k_plan_starts<<<(uint32_t)nkeys, kT, 0, s>>>(a, range_size_scratch);
  k_plan_bases<<<1, 1024, 0, s>>>(a, range_size_scratch, nkeys);
  k_plan_fill<<<grid ? grid : 1, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t estimate_plan(const EstParams &e, const PlanLayout &pl, uint64_t n, double *out,
                          unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  switch (pl.block_log2) {
    case 16: return launch_est<16>(e, pl, n, out, outS, outV, s);
    case 15: return launch_est<15>(e, pl, n, out, outS, outV, s);
    case 14: return launch_est<14>(e, pl, n, out, outS, outV, s);
    case 13: return launch_est<13>(e, pl, n, out, outS, outV, s);
    case 12: return launch_est<12>(e, pl, n, out, outS, outV, s);
    case 11: return launch_est<11>(e, pl, n, out, outS, outV, s);
    case 10: return launch_est<10>(e, pl, n, out, outS, outV, s);
    case 9: return launch_est<9>(e, pl, n, out, outS, outV, s);
    case 8: return launch_est<8>(e, pl, n, out, outS, outV, s);
    case 7: return launch_est<7>(e, pl, n, out, outS, outV, s);
    case 6: return launch_est<6>(e, pl, n, out, outS, outV, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vbdr_launch
