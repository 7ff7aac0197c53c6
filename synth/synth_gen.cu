// synth_gen.cu -- CUDA twin of synth.generate (see synth/__init__.py for the
// trace model).  Bench/test input generator only: holds none of the VBDR
// method's arithmetic and is not part of libvbdr.so.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

__global__ void k_generate(uint2 *__restrict__ out, uint64_t count, uint64_t base, uint64_t start,
                           const double *__restrict__ cdf, const uint32_t *__restrict__ U,
                           uint32_t H, uint32_t churn, uint32_t burst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += stride) {
    uint64_t src = start + q;
    // bursty variant: back to the first position of the packet train
    for (uint32_t k = 1; k < burst && src > 0; ++k) {
      if ((sm64(sm64(base ^ src) ^ 0xD1B54A32D192ED03ull) >> 63) == 0) break;
      --src;
    }
    const uint64_t x = sm64(base ^ src);
    const double u = (double)(x >> 11) * 0x1.0p-53;
    // first index with cdf[h] > u (numpy searchsorted side='right')
    uint32_t lo = 0, hi = H - 1;  // cdf[H-1] = 1.0 > u
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo) >> 1);
      if (cdf[mid] > u) hi = mid; else lo = mid + 1;
    }
    const uint32_t h = lo;
    const uint32_t aip = lowbias32(h ^ 0xA5A5A5A5u);
    const uint64_t y = sm64(x);
    uint32_t v;
    if ((y >> 56) < churn) v = 0x80000000u | (uint32_t)(y & 0x7FFFFFFFull);
    else v = (uint32_t)((y & 0xFFFFFFFFull) % (uint64_t)U[h]);
    const uint32_t bip = lowbias32((h * 0x9E3779B1u + v) ^ 0x3C3C3C3Cu);
    out[q] = make_uint2(aip, bip);
  }
}

}  // namespace

extern "C" int synth_generate(void *d_out, uint64_t count, uint64_t seed, uint64_t t,
                              uint64_t start, const void *d_cdf, const void *d_U, uint32_t H,
                              uint32_t churn, uint32_t burst, void *stream) {
  if (count == 0) return 0;
  if (!d_out || !d_cdf || !d_U || H == 0) return -1;
  // base = sm64(seed ^ (t << 32)), computed on the host exactly as numpy does
  uint64_t z = (seed ^ (t << 32)) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t base = z ^ (z >> 31);
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  k_generate<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      (uint2 *)d_out, count, base, start, (const double *)d_cdf, (const uint32_t *)d_U, H, churn,
      burst);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
