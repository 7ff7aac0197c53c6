// k_estimate.cu -- per-host estimation kernel (sm_100a), compiled with
// -fmad=false; the fp64 finish uses only explicitly rounded intrinsics so its
// operation order is the oracle's (R#17).
//
// Per host aip (Alg.5, as a gather):
//   S = sum_i 2^(L - M[getPhyIdx(aip, i, A0)]) (exact u64), V = #{M = 0}
//   E_s = alpha_g g^2 / (S 2^-L); linear counting g ln(g/V) if E_s <= 2.5 g
//   and V > 0 (R#16); est = max(0, C (E_s/g - E_tot/z)) (vHLL, PAPER.md:214,
//   R#15), E_tot from the pool sums the slide produced.
//
// G lanes cooperate on one host (a "group"); lane `sub` of the group owns the
// virtual indices i = sub + G q.  s1[i] = H(i, 2^32, A0) (Alg.3) is
// the same for every host, so the block tabulates it once in shared memory.
// The gathers are random 1-byte loads from regmax: L2-resident up to 2^26
// BDRs, where the kernel is bound by the SM's L1-to-L2 request rate (one
// sector per gather); U independent gathers per lane keep
// enough requests in flight.
//
// Larger pools (regmax > 64 MiB, e.g. bigwin's 256 MiB) would make every
// gather a DRAM sector access.  There the kernel runs in passes, each over an
// L2-sized physical range [p 2^R, (p+1) 2^R): a pass gathers only the indices
// in its range and adds the packed partial sums S | V << 40 (S <= g 2^L = 2^32)
// into the 8-byte output slot of the host; the last pass turns the slot into
// the estimate.  Integer partials make the result independent of the split.
#include "vbdr_dev.cuh"

using namespace vbdr_dev;
using vbdr_launch::EstParams;

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kS1SmemMax = 8192;  // g up to this uses the shared table

__device__ __forceinline__ double hll_finish(double agg, double D, double lc, uint64_t V,
                                             double s) {
  double E = __ddiv_rn(agg, D);
  if (E <= lc && V > 0) E = __dmul_rn(s, log(__ddiv_rn(s, (double)V)));
  return E;
}

template <int G, int U, bool SUMS, bool SMEM, bool MULTI>
__global__ void __launch_bounds__(kThreads)
k_estimate(EstParams e, const uint32_t *__restrict__ hosts, uint64_t n, double *__restrict__ out,
           unsigned long long *__restrict__ outS, uint32_t *__restrict__ outV, uint32_t pass,
           bool last) {
  pdl_wait();
  extern __shared__ uint32_t s1tab[];
  __shared__ double s_etot_z;  // E_tot / z
  if constexpr (SMEM) {
    for (uint32_t i = threadIdx.x; i < e.g; i += kThreads) s1tab[i] = fmix32(i ^ e.A0);
  }
  if (!SUMS && (!MULTI || last) && threadIdx.x == 0) {
    const unsigned long long St = e.acc[0], Vt = e.acc[1];
    double Et;
    if (e.est == 0u) {
      const double D = __dmul_rn((double)St, e.inv2L);  // exact: St <= 2^53
      Et = hll_finish(e.azz, D, e.lc_z, Vt, e.z);
    } else {  // LogLog / PCSA: coef * 2^(sum / z)
      Et = __dmul_rn(e.coef_z, exp2(__ddiv_rn((double)St, e.z)));
    }
    s_etot_z = __ddiv_rn(Et, e.z);
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t sub = lane & (G - 1u);
  const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t warp_first = (tid & ~uint64_t(31)) / G;  // first group of this warp
  const uint64_t group = tid / G;
  const uint64_t ngroups = ((uint64_t)gridDim.x * kThreads) / G;
  const uint32_t per_lane = e.g / G;

  for (uint64_t r = 0; warp_first + r < n; r += ngroups) {  // warp-uniform
    const uint64_t h = group + r;
    const bool valid = h < n;
    const uint32_t aip = valid ? (MULTI ? __ldcs(hosts + h) : __ldg(hosts + h)) : 0u;
    unsigned long long S = 0ull;
    uint32_t V = 0u;
    for (uint32_t q = 0; q < per_lane; q += U) {
      uint32_t M[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t i = sub + (uint32_t)G * (q + (uint32_t)u);
        const uint32_t s1 = SMEM ? s1tab[i] : fmix32(i ^ e.A0);
        const uint32_t pidx = fmix32(aip ^ s1) & e.mask;
        if constexpr (MULTI)
          M[u] = (pidx >> e.pass_log2) == pass ? (uint32_t)__ldg(e.regmax + pidx) : 0xFFu;
        else
          M[u] = __ldg(e.regmax + pidx);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (MULTI && M[u] == 0xFFu) continue;  // outside this pass's range
        S += e.est == 0u ? 1ull << (e.L - M[u]) : (unsigned long long)M[u];
        V += M[u] == 0u;
      }
    }
#pragma unroll
    for (uint32_t off = G / 2; off >= 1; off >>= 1) {
      S += __shfl_xor_sync(0xffffffffu, S, off);
      V += __shfl_xor_sync(0xffffffffu, V, off);
    }
    if (valid && sub == 0u) {
      if constexpr (MULTI) {
        unsigned long long *slot =
            SUMS ? outS + h : reinterpret_cast<unsigned long long *>(out) + h;
        unsigned long long packed = S | ((unsigned long long)V << 40);
        if (pass > 0) packed += __ldcs(slot);
        if (!last) {
          __stcs(slot, packed);
          continue;
        }
        S = packed & ((1ull << 40) - 1ull);
        V = (uint32_t)(packed >> 40);
      }
      if constexpr (SUMS) {
        outS[h] = S;
        outV[h] = V;
      } else {
        const double g = (double)e.g;
        double Es;
        if (e.est == 0u) {
          const double D = __dmul_rn((double)S, e.inv2L);  // exact: S <= 2^32
          Es = hll_finish(e.agg, D, e.lc_g, V, g);
        } else {  // LogLog / PCSA: coef * 2^(sum / g) (sum = Alg.5's getSumLBP1 for LogLog)
          Es = __dmul_rn(e.coef_g, exp2(__ddiv_rn((double)S, g)));
        }
        const double est = __dmul_rn(e.C, __dsub_rn(__ddiv_rn(Es, g), s_etot_z));
        out[h] = est > 0.0 ? est : 0.0;
      }
    }
  }
  pdl_trigger();
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int G, int U, bool SMEM>
cudaError_t run(const EstParams &e, const uint32_t *hosts, uint64_t n, double *out,
                unsigned long long *outS, uint32_t *outV, cudaStream_t s, uint32_t *nl) {
  const size_t smem = SMEM ? (size_t)e.g * 4 : 0;
  const uint32_t log2z = 31u - (uint32_t)__builtin_clz((uint32_t)(e.mask)) + 1u;  // mask = z - 1
  const uint32_t passes = (e.pass_log2 >= log2z) ? 1u : (1u << (log2z - e.pass_log2));
  *nl = passes;
  if (passes > 1) {
    auto kern = outS ? k_estimate<G, U, true, SMEM, true> : k_estimate<G, U, false, SMEM, true>;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess ||
        per_sm <= 0)
      per_sm = 1;
    const uint64_t resident = (uint64_t)per_sm * sm_count();
    const uint64_t need = (n * G + kThreads - 1) / kThreads;
    const uint64_t grid = need < resident ? need : resident;
    for (uint32_t p = 0; p < passes; ++p) {
      const cudaError_t err = launch_ex(pdl_mode() == 1, kern, dim3((uint32_t)(grid ? grid : 1)), dim3(kThreads), smem,
                                     s, e, hosts, n, out, outS, outV, p, p + 1 == passes);
      if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
  }
  auto kern = outS ? k_estimate<G, U, true, SMEM, false> : k_estimate<G, U, false, SMEM, false>;
  // occupancy is cached while the s1 table is too small to limit it (g <= 1024)
  static int per_sm_cache[2] = {0, 0};
  int local = 0;
  int &per_sm = smem <= 4096 ? per_sm_cache[outS ? 1 : 0] : local;
  if (per_sm == 0 &&
      (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess ||
       per_sm <= 0))
    per_sm = 1;
  const uint64_t resident = (uint64_t)per_sm * sm_count();
  const uint64_t need = (n * G + kThreads - 1) / kThreads;
  const uint64_t grid = need < resident ? need : resident;
  return launch_ex(pdl_mode() == 1, kern, dim3((uint32_t)(grid ? grid : 1)), dim3(kThreads), smem, s, e, hosts, n, out,
                outS, outV, 0u, true);
}

template <int G>
cudaError_t run_g(const EstParams &e, const uint32_t *hosts, uint64_t n, double *out,
                  unsigned long long *outS, uint32_t *outV, cudaStream_t s, uint32_t *nl) {
  const uint32_t per_lane = e.g / G;
  const bool smem = e.g <= kS1SmemMax;
  if (per_lane >= 8)
    return smem ? run<G, 8, true>(e, hosts, n, out, outS, outV, s, nl)
                : run<G, 8, false>(e, hosts, n, out, outS, outV, s, nl);
  if (per_lane == 4) return run<G, 4, true>(e, hosts, n, out, outS, outV, s, nl);
  if (per_lane == 2) return run<G, 2, true>(e, hosts, n, out, outS, outV, s, nl);
  return run<G, 1, true>(e, hosts, n, out, outS, outV, s, nl);
}

// --------------------------------------------------- pass-id plan
// Multi-pass pools spend most of each pass recomputing getPhyIdx for every
// (host, i) only to keep the quarter that falls in the pass's range.  A
// pass-id plan, built once per host list, stores the pass of every (host, i)
// in 2 bits; a pass then hashes and gathers only its own (host, i).  Lane
// `sub` of host h's group (G = g / 64 lanes) owns i = sub + G q, q = 0..63,
// whose pass ids are the 64 fields of one 16-byte word pid[h * G + sub]
// (field q: bits 2 (q mod 16) of u32 q / 16).  Up to 4 passes.
constexpr uint32_t kPpPerLane = 64;

__global__ void __launch_bounds__(kThreads)
k_passplan_build(const uint32_t *__restrict__ hosts, uint64_t n, uint32_t G, uint32_t A0,
                 uint32_t mask, uint32_t pass_log2, uint4 *__restrict__ pid) {
  const uint64_t total = n * G;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t x = (uint64_t)blockIdx.x * kThreads + threadIdx.x; x < total; x += stride) {
    const uint32_t aip = __ldg(hosts + x / G), sub = (uint32_t)(x % G);
    uint32_t wd[4] = {0u, 0u, 0u, 0u};
#pragma unroll 4
    for (uint32_t q = 0; q < kPpPerLane; ++q) {
      const uint32_t i = sub + G * q;
      const uint32_t pidx = fmix32(aip ^ fmix32(i ^ A0)) & mask;  // Alg.3
      wd[q >> 4] |= (pidx >> pass_log2) << (2u * (q & 15u));
    }
    pid[x] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
}

template <int G, bool SUMS>
__global__ void __launch_bounds__(kThreads)
k_estimate_pp(EstParams e, const uint32_t *__restrict__ hosts, uint64_t n,
              const uint4 *__restrict__ pid, double *__restrict__ out,
              unsigned long long *__restrict__ outS, uint32_t *__restrict__ outV, uint32_t pass,
              bool last) {
  pdl_wait();
  extern __shared__ uint32_t s1tab[];
  __shared__ double s_etot_z;
  for (uint32_t i = threadIdx.x; i < e.g; i += kThreads) s1tab[i] = fmix32(i ^ e.A0);
  if (!SUMS && last && threadIdx.x == 0) {
    const unsigned long long St = e.acc[0], Vt = e.acc[1];
    double Et;
    if (e.est == 0u) {
      Et = hll_finish(e.azz, __dmul_rn((double)St, e.inv2L), e.lc_z, Vt, e.z);
    } else {
      Et = __dmul_rn(e.coef_z, exp2(__ddiv_rn((double)St, e.z)));
    }
    s_etot_z = __ddiv_rn(Et, e.z);
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t sub = lane & (G - 1u);
  const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  const uint64_t warp_first = (tid & ~uint64_t(31)) / G;
  const uint64_t group = tid / G;
  const uint64_t ngroups = ((uint64_t)gridDim.x * kThreads) / G;
  const uint32_t pat = pass * 0x55555555u;  // the pass id in every 2-bit field
  for (uint64_t r = 0; warp_first + r < n; r += ngroups) {
    const uint64_t h = group + r;
    const bool valid = h < n;
    unsigned long long S = 0ull;
    uint32_t V = 0u;
    if (valid) {
      const uint32_t aip = __ldcs(hosts + h);
      const uint4 w4 = __ldcs(pid + h * G + sub);
      const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t xw = wv[k] ^ pat;
        uint32_t m = ~(xw | (xw >> 1)) & 0x55555555u;  // fields equal to the pass
        while (m) {  // up to 4 gathers in flight
          uint32_t M[4], cnt = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            M[u] = 0xFFu;
            if (m) {
              const uint32_t q = 16u * k + ((uint32_t)(__ffs(m) - 1) >> 1);
              m &= m - 1u;
              const uint32_t pidx = fmix32(aip ^ s1tab[sub + G * q]) & e.mask;
              M[u] = __ldg(e.regmax + pidx);
              ++cnt;
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (M[u] == 0xFFu) continue;
            S += e.est == 0u ? 1ull << (e.L - M[u]) : (unsigned long long)M[u];
            V += M[u] == 0u;
          }
          (void)cnt;
        }
      }
    }
#pragma unroll
    for (uint32_t off = G / 2; off >= 1; off >>= 1) {
      S += __shfl_xor_sync(0xffffffffu, S, off);
      V += __shfl_xor_sync(0xffffffffu, V, off);
    }
    if (valid && sub == 0u) {
      unsigned long long *slot = SUMS ? outS + h : reinterpret_cast<unsigned long long *>(out) + h;
      unsigned long long packed = S | ((unsigned long long)V << 40);
      if (pass > 0) packed += __ldcs(slot);
      if (!last) {
        __stcs(slot, packed);
        continue;
      }
      S = packed & ((1ull << 40) - 1ull);
      V = (uint32_t)(packed >> 40);
      if constexpr (SUMS) {
        outS[h] = S;
        outV[h] = V;
      } else {
        const double g = (double)e.g;
        double Es;
        if (e.est == 0u) {
          Es = hll_finish(e.agg, __dmul_rn((double)S, e.inv2L), e.lc_g, V, g);
        } else {
          Es = __dmul_rn(e.coef_g, exp2(__ddiv_rn((double)S, g)));
        }
        const double est = __dmul_rn(e.C, __dsub_rn(__ddiv_rn(Es, g), s_etot_z));
        out[h] = est > 0.0 ? est : 0.0;
      }
    }
  }
  pdl_trigger();
}

template <int G>
cudaError_t run_pp(const EstParams &e, const uint32_t *hosts, uint64_t n, const uint4 *pid,
                   uint32_t passes, double *out, unsigned long long *outS, uint32_t *outV,
                   cudaStream_t s) {
  const size_t smem = (size_t)e.g * 4;
  auto kern = outS ? k_estimate_pp<G, true> : k_estimate_pp<G, false>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess ||
      per_sm <= 0)
    per_sm = 1;
  const uint64_t resident = (uint64_t)per_sm * sm_count();
  const uint64_t need = (n * G + kThreads - 1) / kThreads;
  const uint64_t grid = need < resident ? need : resident;
  for (uint32_t p = 0; p < passes; ++p) {
    const cudaError_t err = launch_ex(pdl_mode() == 1, kern, dim3((uint32_t)(grid ? grid : 1)),
                                      dim3(kThreads), smem, s, e, hosts, n, pid, out, outS, outV,
                                      p, p + 1 == passes);
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

// Super-spreader readout: indices of the hosts whose estimate reaches the
// threshold, compacted with one warp-aggregated atomic per warp (order of the
// output is unspecified; the binding sorts it).
__global__ void __launch_bounds__(kThreads)
k_select_above(const double *__restrict__ est, uint64_t n, double threshold,
               uint32_t *__restrict__ idx, unsigned long long *__restrict__ count) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t n_round = (n + 31) & ~uint64_t(31);  // whole warps stay in the loop
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n_round; i += stride) {
    const bool hit = i < n && est[i] >= threshold;
    const uint32_t ballot = __ballot_sync(0xffffffffu, hit);
    if (ballot == 0u) continue;
    const uint32_t lane = threadIdx.x & 31u;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(ballot));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (hit) idx[base + __popc(ballot & ((1u << lane) - 1u))] = (uint32_t)i;
  }
}

}  // namespace

namespace vbdr_launch {

cudaError_t select_above(const double *est, uint64_t n, double threshold, uint32_t *idx,
                         unsigned long long *count, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess || n == 0) return e;
  const uint64_t need = (n + kThreads - 1) / kThreads;
  const uint32_t grid = (uint32_t)(need < (uint64_t)sm_count() * 8 ? need : (uint64_t)sm_count() * 8);
  k_select_above<<<grid, kThreads, 0, s>>>(est, n, threshold, idx, count);
  return cudaGetLastError();
}

// Lanes per host: `lanes` if given (a power of two <= min(g, 32)), else 8 for
// one pass (best on the caida sweep, profiles/r01_sweep_caida.jsonl) and 4 for
// multi-pass pools (bigwin: 20.8 vs 22.4 ms, profiles/r01_pass_sweep.txt),
// capped at g.
uint32_t passplan_lanes(uint32_t g) { return g / kPpPerLane; }

cudaError_t passplan_build(const uint32_t *hosts, uint64_t n, uint32_t g, uint32_t A0,
                           uint32_t mask, uint32_t pass_log2, void *pid, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint32_t G = passplan_lanes(g);
  const uint64_t need = (n * G + kThreads - 1) / kThreads;
  const uint32_t grid = (uint32_t)(need < (uint64_t)sm_count() * 8 ? need : (uint64_t)sm_count() * 8);
  k_passplan_build<<<grid, kThreads, 0, s>>>(hosts, n, G, A0, mask, pass_log2,
                                             static_cast<uint4 *>(pid));
  return cudaGetLastError();
}

cudaError_t estimate_passplan(const EstParams &e, const uint32_t *hosts, uint64_t n,
                              const void *pid, uint32_t passes, double *out,
                              unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint4 *p4 = static_cast<const uint4 *>(pid);
  switch (passplan_lanes(e.g)) {
    case 1: return run_pp<1>(e, hosts, n, p4, passes, out, outS, outV, s);
    case 2: return run_pp<2>(e, hosts, n, p4, passes, out, outS, outV, s);
    case 4: return run_pp<4>(e, hosts, n, p4, passes, out, outS, outV, s);
    case 8: return run_pp<8>(e, hosts, n, p4, passes, out, outS, outV, s);
    case 16: return run_pp<16>(e, hosts, n, p4, passes, out, outS, outV, s);
    case 32: return run_pp<32>(e, hosts, n, p4, passes, out, outS, outV, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t estimate(const EstParams &e, const uint32_t *hosts, uint64_t n, double *out,
                     unsigned long long *outS, uint32_t *outV, cudaStream_t s, uint32_t *nl) {
  *nl = 0;
  if (n == 0) return cudaSuccess;
  const uint32_t log2z = 31u - (uint32_t)__builtin_clz(e.mask) + 1u;
  uint32_t G = e.lanes ? e.lanes : (e.pass_log2 < log2z ? 4u : 8u);
  if (G > e.g) G = e.g;
  if (G > 32) G = 32;
  switch (G) {
    case 1: return run_g<1>(e, hosts, n, out, outS, outV, s, nl);
    case 2: return run_g<2>(e, hosts, n, out, outS, outV, s, nl);
    case 4: return run_g<4>(e, hosts, n, out, outS, outV, s, nl);
    case 8: return run_g<8>(e, hosts, n, out, outS, outV, s, nl);
    case 16: return run_g<16>(e, hosts, n, out, outS, outV, s, nl);
    case 32: return run_g<32>(e, hosts, n, out, outS, outV, s, nl);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vbdr_launch
