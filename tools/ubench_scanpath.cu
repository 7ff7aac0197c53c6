// ubench_scanpath.cu -- the scan's memory path alone (round 2): a ceiling for
// k_scan measured on the same stream of BDR updates.  Records are the
// (register index, stamp value) pairs a slice's IP pairs hash to (computed by
// tools/scan_ceiling.py from the bench's own synthetic slices), 8 bytes per
// record like the IP pairs; the kernel streams them with the scan's 16-byte
// loads and grid, and does exactly the scan's global traffic per record --
// mode 0: the L2 check load, then atomicMax when the stored value is smaller
// (k_scan mode 2 without hashing); mode 1: atomicMax on every record; mode 2:
// a u8 per register (z bytes) -- check the byte, then atomicCAS on its word;
// mode 3: layout P's SetDR -- check the field, then atomicAnd clearing it.  No
// hashing, no shared-memory cache: what is left is the cost of the memory
// path, so k_scan's rate over this one is its fraction of the path's bound.
// Built as a shared library (extern "C"), called through ctypes.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void rec(uint32_t j, uint32_t val, uint32_t *sr, int mode) {
  if (mode == 2) {  // u8 per register (the paper's nowLBP1): check the byte, CAS the word
    uint32_t *w = sr + (j >> 2);
    const uint32_t sh = (j & 3u) * 8u, rho = val & 31u;
    uint32_t cur = __ldcg(w);
    while (((cur >> sh) & 0xFFu) < rho) {
      const uint32_t prev = atomicCAS(w, cur, (cur & ~(0xFFu << sh)) | (rho << sh));
      if (prev == cur) break;
      cur = prev;
    }
    return;
  }
  if (mode == 3) {  // layout P: val = the field mask of rank rho in word j (SetDR, Alg.9)
    if ((__ldcg(sr + j) & val) == 0u) return;  // already cleared
    atomicAnd(sr + j, ~val);
    return;
  }
  if (mode == 0 && __ldcg(sr + j) >= val) return;
  atomicMax(sr + j, val);
}

__global__ void __launch_bounds__(kThreads) k_path(const uint4 *r2, uint64_t n2, uint32_t *sr,
                                                   int mode) {
  constexpr int UNROLL = 4;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n2; i += UNROLL * stride) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(r2 + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      rec(v[u].x, v[u].y, sr, mode);
      rec(v[u].z, v[u].w, sr, mode);
    }
  }
  for (; i < n2; i += stride) {
    const uint4 v = __ldcs(r2 + i);
    rec(v.x, v.y, sr, mode);
    rec(v.z, v.w, sr, mode);
  }
}

}  // namespace

extern "C" int sp_run(const void *records, uint64_t n, void *sr, int mode, void *stream) {
  static int grid = 0;
  if (grid == 0) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_path, kThreads, 0);
    grid = per_sm * sms;
  }
  const uint64_t n2 = n / 2;  // n even
  k_path<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4 *>(records), n2, static_cast<uint32_t *>(sr), mode);
  return (int)cudaGetLastError();
}
