// k_estimate.cu -- per-host estimation kernel (sm_100a), compiled with
// -fmad=false; the fp64 finish uses only explicitly rounded intrinsics so its
// operation order is the oracle's (R#17).
//
// Per host aip (Alg.5, as a gather):
//   S = sum_i 2^(L - M[getPhyIdx(aip, i, A0)]) (exact u64), V = #{M = 0}
//   E_s = alpha_g g^2 / (S 2^-L); linear counting g ln(g/V) if E_s <= 2.5 g
//   and V > 0 (R#16); est = max(0, C (E_s/g - E_tot/z)) (vHLL, PAPER.md:214,
//   R#15), E_tot from the pool sums the slide produced.
// G lanes cooperate on one host (G = min(g, 32)); each lane owns the virtual
// indices i = sub + q G and keeps s1 = H(i, 2^32, A0) (Alg.3) in
// registers for the whole kernel.
#include "vbdr_dev.cuh"

using namespace vbdr_dev;
using vbdr_launch::EstParams;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double hll_finish(double agg_over, double D, double lc, uint64_t V,
                                             double s) {
  double E = __ddiv_rn(agg_over, D);
  if (E <= lc && V > 0) E = __dmul_rn(s, log(__ddiv_rn(s, (double)V)));
  return E;
}

// NQ > 0: compile-time indices per lane; NQ == 0: runtime g/32 (g > 256).
template <int G, int NQ, bool SUMS>
__global__ void __launch_bounds__(kThreads)
k_estimate(EstParams e, const uint32_t *__restrict__ hosts, uint64_t n, double *__restrict__ out,
           unsigned long long *__restrict__ outS, uint32_t *__restrict__ outV) {
  __shared__ double s_etot_z;  // E_tot / z
  if (!SUMS && threadIdx.x == 0) {
    const unsigned long long St = e.acc[0], Vt = e.acc[1];
    const double D = __dmul_rn((double)St, e.inv2L);  // exact: St <= 2^53
    const double Et = hll_finish(e.azz, D, e.lc_z, Vt, e.z);
    s_etot_z = __ddiv_rn(Et, e.z);
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t sub = lane & (G - 1u);
  const uint32_t grp = lane / G;
  constexpr uint32_t HPW = 32 / G;  // hosts per warp
  constexpr int NQR = NQ > 0 ? NQ : 1;
  uint32_t s1[NQR];
#pragma unroll
  for (int q = 0; q < NQR; ++q) s1[q] = fmix32((sub + (uint32_t)q * G) ^ e.A0);
  const uint32_t nq_rt = e.g / G;

  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kThreads) >> 5;
  for (uint64_t base = warp * HPW; base < n; base += nwarps * HPW) {
    const uint64_t h = base + grp;
    const bool valid = h < n;
    const uint32_t aip = valid ? __ldg(hosts + h) : 0u;
    unsigned long long S = 0ull;
    uint32_t V = 0u;
    if constexpr (NQ > 0) {
      uint32_t M[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) M[q] = __ldg(e.regmax + (fmix32(aip ^ s1[q]) & e.mask));
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        S += 1ull << (e.L - M[q]);
        V += M[q] == 0u;
      }
    } else {
      for (uint32_t q = 0; q < nq_rt; ++q) {
        const uint32_t s = fmix32((sub + q * G) ^ e.A0);
        const uint32_t M = __ldg(e.regmax + (fmix32(aip ^ s) & e.mask));
        S += 1ull << (e.L - M);
        V += M == 0u;
      }
    }
#pragma unroll
    for (uint32_t off = G / 2; off >= 1; off >>= 1) {
      S += __shfl_xor_sync(0xffffffffu, S, off);
      V += __shfl_xor_sync(0xffffffffu, V, off);
    }
    if (valid && sub == 0u) {
      if constexpr (SUMS) {
        outS[h] = S;
        outV[h] = V;
      } else {
        const double g = (double)e.g;
        const double D = __dmul_rn((double)S, e.inv2L);  // exact: S <= 2^32
        const double Es = hll_finish(e.agg, D, e.lc_g, V, g);
        const double est = __dmul_rn(e.C, __dsub_rn(__ddiv_rn(Es, g), s_etot_z));
        out[h] = est > 0.0 ? est : 0.0;
      }
    }
  }
}

uint32_t grid_for_hosts(uint64_t n, uint32_t hpw) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const uint64_t warps = (n + hpw - 1) / hpw;
  const uint64_t need = (warps * 32 + kThreads - 1) / kThreads;
  const uint64_t cap = (uint64_t)sms * 8;
  const uint64_t g = need < cap ? need : cap;
  return (uint32_t)(g ? g : 1);
}

template <int G, int NQ>
cudaError_t run(const EstParams &e, const uint32_t *hosts, uint64_t n, double *out,
                unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  const uint32_t grid = grid_for_hosts(n, 32 / G);
  if (outS != nullptr)
    k_estimate<G, NQ, true><<<grid, kThreads, 0, s>>>(e, hosts, n, out, outS, outV);
  else
    k_estimate<G, NQ, false><<<grid, kThreads, 0, s>>>(e, hosts, n, out, outS, outV);
  return cudaGetLastError();
}

}  // namespace

namespace vbdr_launch {

cudaError_t estimate(const EstParams &e, const uint32_t *hosts, uint64_t n, double *out,
                     unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (e.g) {
    case 2: return run<2, 1>(e, hosts, n, out, outS, outV, s);
    case 4: return run<4, 1>(e, hosts, n, out, outS, outV, s);
    case 8: return run<8, 1>(e, hosts, n, out, outS, outV, s);
    case 16: return run<16, 1>(e, hosts, n, out, outS, outV, s);
    case 32: return run<32, 1>(e, hosts, n, out, outS, outV, s);
    case 64: return run<32, 2>(e, hosts, n, out, outS, outV, s);
    case 128: return run<32, 4>(e, hosts, n, out, outS, outV, s);
    case 256: return run<32, 8>(e, hosts, n, out, outS, outV, s);
    default: return run<32, 0>(e, hosts, n, out, outS, outV, s);
  }
}

}  // namespace vbdr_launch
