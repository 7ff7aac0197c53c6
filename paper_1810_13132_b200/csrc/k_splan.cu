// k_splan.cu -- sorted-plan estimation for a fixed host list (sm_100a),
// compiled with -fmad=false like k_estimate.cu (same fp64 finish).
//
// Alg.5 for every host is a sparse sum over g registers
// regmax[pidx(h, i)] with pidx = getPhyIdx(h, i) (Alg.3).
// The gather kernel (k_estimate.cu) pays one L2 sector request per (h, i):
// the registers are random.  Here a PLAN, built once per host list, lists
// every (h, i) SORTED BY pidx, so consecutive entries read neighbouring
// registers: a warp's 32 gathers touch one or two 128-byte lines instead of
// 32, and most hit L1.
//
//   * The persistent grid (one CTA per SM) is P host groups x C register
//     ranges.  Host h belongs to group h mod P at accumulator slot h / P;
//     CTA (p, c) handles exactly the (h, i) of group p whose pidx falls in
//     range c = [c z/C, (c+1) z/C).  Each CTA keeps (S', V) of all its group's
//     hosts in shared memory (8 B per host), so the register array is read
//     P times in total (not once per SM), and every plan entry once.
//   * Entries are u32: (pidx - segment base) << SB | slot, bucketed by
//     128-register line within a CTA (counting sort at build), in segments of
//     2^(32 - SB) registers, each segment padded to whole rounds of 32 entries
//     (padding adds to one of 32 trash slots).
//   * The 32 warps of a CTA split its rounds evenly; per round a lane loads
//     its entry (streamed once), reads the register byte, and adds 2^(L - M)
//     (M >= 1) into S'[slot] or 1 into V[slot] with one shared-memory atomic
//     (LogLog / PCSA: M into S', zeros into V).
//   * With C > 1 ranges a group's partial sums are combined by the group's
//     last CTA to finish (partials through global memory, a per-group arrival
//     counter), which also runs the fp64 finish of k_estimate.
// Integer sums: bit-identical to vbdr_estimate.
#include "vbdr_dev.cuh"

using namespace vbdr_dev;
using vbdr_launch::EstParams;
using vbdr_launch::PlanLayout;

namespace {

constexpr int kT = vbdr_launch::kSpThreads;  // 1024
constexpr int kW = kT / 32;
constexpr uint32_t kLineLog2 = vbdr_launch::kSpLineLog2;  // buckets of 128 registers

// ---------------------------------------------------------------- build
struct SpBuild {
  const uint32_t *hosts;
  uint64_t n;
  uint32_t g, A0, mask;
  uint32_t P, C, range_log2, seg_log2, nseg, SB, hpg;
  uint32_t *offs;     // [ctas * (range >> 7)] bucket counts -> offsets in segment -> cursors
  uint32_t *segtot;   // [ctas * nseg] entries per segment
  uint32_t *segbase;  // [ctas * nseg + 1] first entry of each segment (padded)
  uint32_t *entries;
};

// (h, i) -> CTA, local segment, global bucket, entry value
__device__ __forceinline__ void sp_locate(const SpBuild &a, uint64_t h, uint32_t i, uint32_t &cta,
                                          uint32_t &seg, uint64_t &bucket, uint32_t &val) {
  const uint32_t s1 = fmix32(i ^ a.A0);                            // Alg.3
  const uint32_t pidx = fmix32(__ldg(a.hosts + h) ^ s1) & a.mask;  // Alg.3
  const uint32_t p = (uint32_t)(h % a.P), slot = (uint32_t)(h / a.P);
  const uint32_t c = pidx >> a.range_log2;
  const uint32_t off = pidx & ((1u << a.range_log2) - 1u);  // offset in the CTA's range
  cta = p * a.C + c;
  seg = off >> a.seg_log2;
  bucket = ((uint64_t)cta << (a.range_log2 - kLineLog2)) + (off >> kLineLog2);
  val = ((off & ((1u << a.seg_log2) - 1u)) << a.SB) | slot;
}

__global__ void k_sp_count(SpBuild a) {
  const uint64_t total = a.n * a.g;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    uint32_t cta, seg, val;
    uint64_t bucket;
    sp_locate(a, x / a.g, (uint32_t)(x % a.g), cta, seg, bucket, val);
    atomicAdd(a.offs + bucket, 1u);
  }
}

// One block per (CTA, segment): exclusive scan of the segment's bucket counts
// in place (-> offset of each bucket within the segment) and the total.
__global__ void __launch_bounds__(1024) k_sp_seg_scan(SpBuild a) {
  __shared__ uint32_t warp_sum[32];
  __shared__ uint32_t carry;
  const uint64_t key = blockIdx.x;  // cta * nseg + seg
  const uint32_t nb = 1u << (a.seg_log2 - kLineLog2);
  uint32_t *cnt = a.offs + key * nb;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nb; base += 1024) {
    const uint32_t b = base + threadIdx.x;
    const uint32_t c = b < nb ? cnt[b] : 0u;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t v = warp_sum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (uint32_t)o) v += y;
      }
      warp_sum[lane] = v;
    }
    __syncthreads();
    const uint32_t incl = x + (w > 0 ? warp_sum[w - 1] : 0u);
    if (b < nb) cnt[b] = carry + incl - c;
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.segtot[key] = carry;
}

// Single block: segment bases, every segment padded to whole rounds of 32.
__global__ void __launch_bounds__(1024) k_sp_seg_base(SpBuild a, uint64_t nkeys,
                                                      unsigned long long *total_out) {
  __shared__ unsigned long long warp_sum[32];
  __shared__ unsigned long long carry;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t base = 0; base < nkeys; base += 1024) {
    const uint64_t k = base + threadIdx.x;
    const unsigned long long c = k < nkeys ? (a.segtot[k] + 31ull) & ~31ull : 0ull;
    unsigned long long x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
      unsigned long long v = warp_sum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= (uint32_t)o) v += y;
      }
      warp_sum[lane] = v;
    }
    __syncthreads();
    const unsigned long long incl = x + (w > 0 ? warp_sum[w - 1] : 0ull);
    if (k < nkeys) a.segbase[k] = (uint32_t)(carry + incl - c);  // < 2^32: checked by the host
    __syncthreads();
    if (threadIdx.x == 1023) carry += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.segbase[nkeys] = (uint32_t)carry;
    *total_out = carry;
  }
}

__global__ void k_sp_fill(SpBuild a) {
  const uint64_t total = a.n * a.g;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    uint32_t cta, seg, val;
    uint64_t bucket;
    sp_locate(a, x / a.g, (uint32_t)(x % a.g), cta, seg, bucket, val);
    const uint32_t pos = atomicAdd(a.offs + bucket, 1u);
    a.entries[(uint64_t)a.segbase[(uint64_t)cta * a.nseg + seg] + pos] = val;
  }
}

// One block per (CTA, segment): the padding to a whole round reads the
// segment's first register into trash slot hpg + lane.
__global__ void __launch_bounds__(32) k_sp_pad(SpBuild a) {
  const uint64_t key = blockIdx.x;
  const uint32_t t = a.segtot[key];
  const uint32_t padded = (t + 31u) & ~31u;
  const uint32_t i = t + threadIdx.x;
  if (i < padded) a.entries[(uint64_t)a.segbase[key] + i] = a.hpg + (i & 31u);
}

// --------------------------------------------------------------- estimate
__device__ __forceinline__ double hll_finish(double agg, double D, double lc, uint64_t V,
                                             double s, const double *lct = nullptr) {
  double E = __ddiv_rn(agg, D);
  // linear counting from the plan's table of s ln(s / V)'s logs (k_plan_lct,
  // the same values) when there is one
  if (E <= lc && V > 0) E = __dmul_rn(s, lct ? __ldg(lct + V) : log(__ddiv_rn(s, (double)V)));
  return E;
}

template <bool SUMS>
__device__ __forceinline__ void sp_finish(const EstParams &e, uint64_t h, uint64_t Sp, uint32_t V,
                                          bool hll, double etot_z, double *out,
                                          unsigned long long *outS, uint32_t *outV,
                                          const double *lct) {
  // HLL: S = S' + V 2^L (each zero register adds 2^(L - 0))
  const unsigned long long S = Sp + (hll ? (unsigned long long)V << e.L : 0ull);
  if constexpr (SUMS) {
    outS[h] = S;
    outV[h] = V;
  } else {
    const double g = (double)e.g;
    double Es;
    if (hll) {
      Es = hll_finish(e.agg, __dmul_rn((double)S, e.inv2L), e.lc_g, V, g, lct);
    } else {
      Es = __dmul_rn(e.coef_g, exp2(__ddiv_rn((double)S, g)));
    }
    // g is a power of two: Es / g is exact as Es * (1 / g)
    const double est = __dmul_rn(e.C, __dsub_rn(__dmul_rn(Es, __drcp_rn(g)), etot_z));
    out[h] = est > 0.0 ? est : 0.0;
  }
}

template <bool SUMS, bool HLL>
__global__ void __launch_bounds__(kT, 1)
k_estimate_sp(EstParams e, PlanLayout pl, uint64_t n, double *__restrict__ out,
              unsigned long long *__restrict__ outS, uint32_t *__restrict__ outV) {
  pdl_wait();
  extern __shared__ __align__(16) uint32_t sp_smem[];
  const uint32_t nslot = pl.sp_hpg + 32u;  // + the 32 trash slots of the padding
  uint32_t *Sacc = sp_smem;                // S' (M >= 1 terms), per slot
  uint32_t *Vacc = Sacc + nslot;           // zero count, per slot
  uint32_t *rs = Vacc + nslot;             // this CTA's segment starts, in rounds
  __shared__ double s_etot_z;
  __shared__ uint32_t s_last;
  const uint32_t cta = blockIdx.x, nseg = pl.sp_nseg;
  const uint32_t p = cta / pl.sp_C, c = cta - p * pl.sp_C;
  for (uint32_t i = threadIdx.x; i < 2 * nslot; i += kT) Sacc[i] = 0u;
  const uint32_t e0 = pl.sp_segbase[(uint64_t)cta * nseg];
  for (uint32_t s = threadIdx.x; s <= nseg; s += kT)
    rs[s] = (pl.sp_segbase[(uint64_t)cta * nseg + s] - e0) >> 5;
  if (!SUMS && threadIdx.x == 0) {
    const unsigned long long St = e.acc[0], Vt = e.acc[1];
    double Et;
    if (HLL) {
      Et = hll_finish(e.azz, __dmul_rn((double)St, e.inv2L), e.lc_z, Vt, e.z);
    } else {
      Et = __dmul_rn(e.coef_z, exp2(__ddiv_rn((double)St, e.z)));
    }
    s_etot_z = __ddiv_rn(Et, e.z);
  }
  __syncthreads();

  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  const uint32_t R = rs[nseg];
  const uint32_t r0 = (uint32_t)(((uint64_t)R * w) / kW), r1 = (uint32_t)(((uint64_t)R * (w + 1)) / kW);
  const uint32_t *ent = pl.entries + e0 + lane;
  const uint8_t *reg = e.regmax + ((uint64_t)c << pl.sp_range_log2);
  const uint32_t SB = pl.sp_SB, smask = (1u << SB) - 1u, segl = pl.sp_seg_log2;
  const uint32_t K = 1u << e.L;  // HLL: 2^(L - M) = K >> M
  const uint32_t sacc = (uint32_t)__cvta_generic_to_shared(Sacc);
  const uint32_t vacc = (uint32_t)__cvta_generic_to_shared(Vacc);
  // the warp's current segment: its end (in rounds) and its register base,
  // kept in registers; crossing into the next segment is a rare warp-uniform
  // branch (segments hold whole rounds)
  uint32_t s = 0;
  while (s + 1 < nseg && rs[s + 1] <= r0) ++s;
  uint32_t seg_end = rs[s + 1];
  const uint8_t *rb = reg + ((uint64_t)s << segl);
  auto seg_at = [&](uint32_t rr) {
    if (rr >= seg_end) {
      do {
        ++s;
        seg_end = rs[s + 1];
      } while (rr >= seg_end);
      rb = reg + ((uint64_t)s << segl);
    }
  };
  // one entry: 2^(L - M) (HLL; M for LogLog / PCSA) into S'[slot] if M >= 1,
  // else 1 into V[slot] -- one shared-memory atomic, address and value selected
  auto add = [&](uint32_t v, uint32_t M) {
    const uint32_t slot = v & smask;
    const bool zero = M == 0u;
    const uint32_t addr = (zero ? vacc : sacc) + 4u * slot;
    const uint32_t val = zero ? 1u : (HLL ? K >> M : M);
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(val) : "memory");
  };
  constexpr int U = vbdr_launch::kSpUnroll;
  uint32_t r = r0;
  const uint32_t *ep = ent + 32ull * r0;  // this lane's entry of round r
  for (; r + U <= r1; r += U, ep += 32 * U) {
#if VBDR_SP_PREFETCH
    // pull the warp's entries VBDR_SP_PREFETCH rounds ahead into L2 (one
    // bulk prefetch per 16 rounds = 2 KB), so the loads below wait on L2
    if (lane == 0 && ((r - r0) & 15u) < (uint32_t)U) {
      const uint32_t a = r + VBDR_SP_PREFETCH;
      if (a < r1) {
        const uint32_t nb = (min(a + 16u, r1) - a) * 128u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ep + 32u * VBDR_SP_PREFETCH),
                     "r"(nb) : "memory");
      }
    }
#endif
    uint32_t v[U], M[U];
    const uint8_t *pa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(ep + 32 * u);  // streamed once
    if (r + U <= seg_end) {  // the whole batch in the current segment (usual)
#pragma unroll
      for (int u = 0; u < U; ++u) pa[u] = rb + (v[u] >> SB);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        seg_at(r + u);
        pa[u] = rb + (v[u] >> SB);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) M[u] = __ldg(pa[u]);  // neighbouring registers: L1 hits
#pragma unroll
    for (int u = 0; u < U; ++u) add(v[u], M[u]);
  }
  for (; r < r1; ++r, ep += 32) {
    const uint32_t v = __ldcs(ep);
    seg_at(r);
    add(v, __ldg(rb + (v >> SB)));
  }
  __syncthreads();
  pdl_trigger();

  const uint32_t P = pl.sp_C == 0 ? 1u : (uint32_t)(pl.ctas / pl.sp_C);
  const uint32_t hpg = pl.sp_hpg;
  if (pl.sp_C == 1) {
    for (uint32_t slot = threadIdx.x; slot < hpg; slot += kT) {
      const uint64_t h = (uint64_t)slot * P + p;
      if (h < n) sp_finish<SUMS>(e, h, Sacc[slot], Vacc[slot], HLL, s_etot_z, out, outS, outV, pl.lct);
    }
    return;
  }
  // C ranges per group: publish the partials, the group's last CTA finishes
  unsigned long long *part = pl.sp_part + (uint64_t)cta * hpg;
  for (uint32_t slot = threadIdx.x; slot < hpg; slot += kT)
    __stcg(part + slot, (unsigned long long)Sacc[slot] | ((unsigned long long)Vacc[slot] << 32));
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(pl.sp_gcount + p, 1u);
    s_last = prev == pl.sp_C - 1u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const unsigned long long *gp = pl.sp_part + (uint64_t)p * pl.sp_C * hpg;
  for (uint32_t slot = threadIdx.x; slot < hpg; slot += kT) {
    const uint64_t h = (uint64_t)slot * P + p;
    if (h >= n) continue;
    unsigned long long Sp = 0;
    uint32_t V = 0;
    for (uint32_t q = 0; q < pl.sp_C; ++q) {
      const unsigned long long x = q == c ? ((unsigned long long)Sacc[slot] |
                                             ((unsigned long long)Vacc[slot] << 32))
                                          : __ldcg(gp + (uint64_t)q * hpg + slot);
      Sp += x & 0xFFFFFFFFull;
      V += (uint32_t)(x >> 32);
    }
    sp_finish<SUMS>(e, h, Sp, V, HLL, s_etot_z, out, outS, outV, pl.lct);
  }
  if (threadIdx.x == 0) pl.sp_gcount[p] = 0u;  // ready for the next launch on this plan
}

}  // namespace

namespace vbdr_launch {

size_t sp_smem_bytes(uint32_t hpg, uint32_t nseg) {
  return (size_t)8 * (hpg + 32u) + (size_t)4 * (nseg + 1u);
}

cudaError_t sp_build(const PlanLayout &pl, const uint32_t *hosts, uint64_t n, uint32_t g,
                     uint32_t A0, uint32_t mask, unsigned long long *d_total, cudaStream_t s) {
  SpBuild a{};
  a.hosts = hosts;
  a.n = n;
  a.g = g;
  a.A0 = A0;
  a.mask = mask;
  a.P = pl.ctas / pl.sp_C;
  a.C = pl.sp_C;
  a.range_log2 = pl.sp_range_log2;
  a.seg_log2 = pl.sp_seg_log2;
  a.nseg = pl.sp_nseg;
  a.SB = pl.sp_SB;
  a.hpg = pl.sp_hpg;
  a.offs = pl.counts;
  a.segtot = pl.range_size;
  a.segbase = pl.sp_segbase;
  a.entries = pl.entries;
  const uint64_t nbuckets = (uint64_t)pl.ctas << (pl.sp_range_log2 - kLineLog2);
  const uint64_t nkeys = (uint64_t)pl.ctas * pl.sp_nseg;
  cudaError_t e = cudaMemsetAsync(a.offs, 0, 4 * nbuckets, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pl.sp_gcount, 0, 4ull * a.P, s);
  if (e != cudaSuccess) return e;
  const uint64_t total = n * g;
  const uint64_t want = (total + 255) / 256;
  const uint32_t grid = (uint32_t)(want < 148ull * 32 ? (want ? want : 1) : 148ull * 32);
  k_sp_count<<<grid, 256, 0, s>>>(a);
  k_sp_seg_scan<<<(uint32_t)nkeys, 1024, 0, s>>>(a);
  k_sp_seg_base<<<1, 1024, 0, s>>>(a, nkeys, d_total);
  return cudaGetLastError();
}

cudaError_t sp_fill(const PlanLayout &pl, const uint32_t *hosts, uint64_t n, uint32_t g,
                    uint32_t A0, uint32_t mask, cudaStream_t s) {
  SpBuild a{};
  a.hosts = hosts;
  a.n = n;
  a.g = g;
  a.A0 = A0;
  a.mask = mask;
  a.P = pl.ctas / pl.sp_C;
  a.C = pl.sp_C;
  a.range_log2 = pl.sp_range_log2;
  a.seg_log2 = pl.sp_seg_log2;
  a.nseg = pl.sp_nseg;
  a.SB = pl.sp_SB;
  a.hpg = pl.sp_hpg;
  a.offs = pl.counts;
  a.segtot = pl.range_size;
  a.segbase = pl.sp_segbase;
  a.entries = pl.entries;
  const uint64_t nkeys = (uint64_t)pl.ctas * pl.sp_nseg;
  const uint64_t total = n * g;
  const uint64_t want = (total + 255) / 256;
  const uint32_t grid = (uint32_t)(want < 148ull * 32 ? (want ? want : 1) : 148ull * 32);
  k_sp_fill<<<grid, 256, 0, s>>>(a);
  k_sp_pad<<<(uint32_t)nkeys, 32, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t estimate_sp(const EstParams &e, const PlanLayout &pl, uint64_t n, double *out,
                        unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  const size_t smem = sp_smem_bytes(pl.sp_hpg, pl.sp_nseg);
  const bool hll = e.est == 0u;
  auto kern = outS ? (hll ? k_estimate_sp<true, true> : k_estimate_sp<true, false>)
                   : (hll ? k_estimate_sp<false, true> : k_estimate_sp<false, false>);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  return launch(kern, dim3(pl.ctas), dim3(kT), smem, s, e, pl, n, out, outS, outV);
}

}  // namespace vbdr_launch
