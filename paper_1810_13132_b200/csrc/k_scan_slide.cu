// k_scan_slide.cu -- pair-scan, slide/expire and init kernels of the VBDR hot
// path for sm_100a.  DESIGN.md section 6 gives each kernel's roofline.
//
// Layout F ("fast", VBDR-serial/gfast semantics):
//   sr[j] = (T << 5) | max rank seen by BDR j in slice T-1 -- the paper's
//   nowLBP1 with the slice tick folded in, so it never
//   needs clearing; the parallel max is an atomicMax (the race of PAPER.md:220
//   removed, R#18).
// Layout P ("packed", VBDR-gsmall semantics): SetDR on the packed DRV during
//   the scan (Alg.9) as an atomicAnd on the containing word.
// Both: DRV = W planes of n_phys u32 words, F = 32/zb DRs per word; rank rho
//   lives in word (rho-1)/F, field (rho-1)%F.
#include "vbdr_dev.cuh"

using namespace vbdr_dev;

namespace {

constexpr int kThreads = 256;

// Slide: 0 = SWAR on every word; 1 = skip warp-uniformly saturated words
// entirely (fewer bytes than the algorithmic 8W per BDR); 2 = skip their ALU
// work but still store them (default: the kernel moves exactly its
// algorithmic bytes; profiles/r01_slide_variants.txt)
#ifndef VBDR_SLIDE_SKIP
#define VBDR_SLIDE_SKIP 2
#endif

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  return __ldcg(p);  // L2 (skip L1: other SMs update it)
}

// ------------------------------------------------------------------ scan
// MODE 5: a per-block direct-mapped cache in shared memory of (word, value
// known to be in global memory).  Skewed traffic hits the same few thousand
// registers again and again (Zipf super-spreaders); a cache hit that already
// dominates skips both the global check and the atomic, saving the SM's
// L1-to-L2 request slots that bound the scan.  An entry
// is inserted only after its atomic was issued (or a load saw the value), so
// it never exceeds what global memory will hold when the kernel ends.
#ifndef VBDR_SCAN_CACHE_SLOTS
#define VBDR_SCAN_CACHE_SLOTS 2048  // 16 KB per block
#endif
#ifndef VBDR_SCAN_THREADS
#define VBDR_SCAN_THREADS 256
#endif
constexpr int kCacheSlots = VBDR_SCAN_CACHE_SLOTS;
constexpr int kScanThreads = VBDR_SCAN_THREADS;

struct ScanCache {
  unsigned long long e[kCacheSlots];  // (key << 32) | value; key = word index + 1 (0 = empty)
};

__device__ __forceinline__ bool cache_hit(const ScanCache *c, uint32_t key, uint32_t val, bool fast) {
  const unsigned long long ent = c->e[key & (kCacheSlots - 1)];
  if ((uint32_t)(ent >> 32) != key) return false;
  const uint32_t v = (uint32_t)ent;
  return fast ? v >= val : (v & val) == val;  // packed: val = field mask known cleared
}

__device__ __forceinline__ void cache_put(ScanCache *c, uint32_t key, uint32_t v) {
  c->e[key & (kCacheSlots - 1)] = ((unsigned long long)key << 32) | v;
}

// One pair: Alg.4 lines 180-184 then the layout's record.
template <bool FAST, int ZB, int MODE>
__device__ __forceinline__ void record(uint32_t aip, uint32_t bip, const DevParams &p,
                                       uint32_t tickbits, ScanCache *cache) {
  uint32_t pidx, rho;
  pair_index(aip, bip, p, pidx, rho);
  if constexpr (FAST) {
    // nowLBP1 <- max(nowLBP1, LBP1(bip'))
    const uint32_t val = tickbits | rho;
    uint32_t *a = p.sr + pidx;
    if constexpr (MODE == 5) {
      const uint32_t key = pidx + 1u;  // n_phys < 2^32 for this mode
      if (cache_hit(cache, key, val, true)) return;
      const uint32_t cur = ld_relaxed(a);
      if (cur >= val) {
        cache_put(cache, key, cur);
        return;
      }
      atomicMax(a, val);
      cache_put(cache, key, val);
      return;
    }
    if constexpr (MODE == 2) {
      if (ld_relaxed(a) >= val) return;  // stored value dominates: max is a no-op
    }
    atomicMax(a, val);
  } else {
    // SetDR(DRV[LBP1(bip')]) = clear one zb-bit field
    using S = Swar<ZB>;
    const uint32_t r = rho - 1u;
    const uint32_t w = r / (uint32_t)S::F;
    const uint32_t f = r - w * (uint32_t)S::F;
    const uint32_t fm = S::FM << (ZB * f);
    uint32_t *a = p.drv + (uint64_t)w * p.n_phys + pidx;
    if constexpr (MODE == 5) {
      // value cached = mask of fields known to be zero in this word
      const uint32_t key = (pidx << 4 | w) + 1u;  // n_phys <= 2^28, W <= 15 for this mode
      if (cache_hit(cache, key, fm, false)) return;
      const uint32_t cur = ld_relaxed(a);
      uint32_t zero = 0u;  // fields of the word already zero
#pragma unroll
      for (int g = 0; g < S::F; ++g)
        if (((cur >> (ZB * g)) & S::FM) == 0u) zero |= S::FM << (ZB * g);
      if ((cur & fm) != 0u) atomicAnd(a, ~fm);
      cache_put(cache, key, zero | fm);
      return;
    }
    if constexpr (MODE == 2) {
      if ((ld_relaxed(a) & fm) == 0u) return;  // already zero
    }
    atomicAnd(a, ~fm);
  }
}

// Grid-stride over pairs, two pairs per 16-byte load, UNROLL loads in flight.
template <bool FAST, int ZB, int MODE>
__global__ void __launch_bounds__(kScanThreads)
k_scan(const uint4 *__restrict__ pairs2, uint64_t n2, const uint32_t *__restrict__ tail,
       DevParams p) {
  pdl_wait();
  constexpr int UNROLL = 4;
  extern __shared__ unsigned long long scan_dyn_smem[];  // MODE 5 only (dynamic size)
  ScanCache *cache = nullptr;
  if constexpr (MODE == 5) {  // only this mode pays for the shared memory
    cache = reinterpret_cast<ScanCache *>(scan_dyn_smem);
    for (int s = threadIdx.x; s < kCacheSlots; s += kScanThreads) cache->e[s] = 0ull;
    __syncthreads();
  }
  const uint32_t tickbits = p.tick << 5;
  const uint64_t stride = (uint64_t)gridDim.x * kScanThreads;
  uint64_t i = (uint64_t)blockIdx.x * kScanThreads + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n2; i += UNROLL * stride) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(pairs2 + i + u * stride);  // streamed once
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      record<FAST, ZB, MODE>(v[u].x, v[u].y, p, tickbits, cache);
      // a pair repeating its predecessor (packet trains) is the same update
      if (v[u].z != v[u].x || v[u].w != v[u].y) record<FAST, ZB, MODE>(v[u].z, v[u].w, p, tickbits, cache);
    }
  }
  for (; i < n2; i += stride) {
    const uint4 v = __ldcs(pairs2 + i);
    record<FAST, ZB, MODE>(v.x, v.y, p, tickbits, cache);
    if (v.z != v.x || v.w != v.y) record<FAST, ZB, MODE>(v.z, v.w, p, tickbits, cache);
  }
  if (tail != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    record<FAST, ZB, MODE>(tail[0], tail[1], p, tickbits, cache);
  pdl_trigger();  // this block's work is issued: let the next kernel launch
}

// ----------------------------------------------------- layout S (stamps)
// Layout S (the north star's literal "last-seen-slice stamps"
// reading, with VBDR-gsmall semantics): a u32 stamp per (BDR j, rank rho) =
// the tick T of the last slice in which rho was recorded into j, in L planes
// of n_phys words (plane rho - 1).  The scan records EVERY pair's rank (as
// Alg.9's per-pair SetDR) as atomicMax(stamp, T); nothing
// ever ages: a DR's age is T - stamp, computed at readout.  32 L bits per BDR
// (caida: 800, against 75 for Table 1's gsmall) -- the comparison point for
// the packed layouts, not a default.
template <int MODE>
__device__ __forceinline__ void record_stamp(uint32_t aip, uint32_t bip, const DevParams &p,
                                             ScanCache *cache) {
  uint32_t pidx, rho;
  pair_index(aip, bip, p, pidx, rho);  // Alg.4
  const uint64_t word = (uint64_t)(rho - 1u) * p.n_phys + pidx;
  uint32_t *a = p.drv + word;
  const uint32_t val = p.tick;
  if constexpr (MODE == 5) {  // L * n_phys < 2^32 for this mode
    const uint32_t key = (uint32_t)word + 1u;
    if (cache_hit(cache, key, val, true)) return;
    const uint32_t cur = ld_relaxed(a);
    if (cur >= val) {
      cache_put(cache, key, cur);
      return;
    }
    atomicMax(a, val);
    cache_put(cache, key, val);
    return;
  }
  if (ld_relaxed(a) >= val) return;  // already stamped in this slice
  atomicMax(a, val);
}

template <int MODE>
__global__ void __launch_bounds__(kScanThreads)
k_scan_stamps(const uint4 *__restrict__ pairs2, uint64_t n2, const uint32_t *__restrict__ tail,
              DevParams p) {
  pdl_wait();
  constexpr int UNROLL = 4;
  extern __shared__ unsigned long long scan_dyn_smem[];
  ScanCache *cache = nullptr;
  if constexpr (MODE == 5) {
    cache = reinterpret_cast<ScanCache *>(scan_dyn_smem);
    for (int s = threadIdx.x; s < kCacheSlots; s += kScanThreads) cache->e[s] = 0ull;
    __syncthreads();
  }
  const uint64_t stride = (uint64_t)gridDim.x * kScanThreads;
  uint64_t i = (uint64_t)blockIdx.x * kScanThreads + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n2; i += UNROLL * stride) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(pairs2 + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      record_stamp<MODE>(v[u].x, v[u].y, p, cache);
      if (v[u].z != v[u].x || v[u].w != v[u].y) record_stamp<MODE>(v[u].z, v[u].w, p, cache);
    }
  }
  for (; i < n2; i += stride) {
    const uint4 v = __ldcs(pairs2 + i);
    record_stamp<MODE>(v.x, v.y, p, cache);
    if (v.z != v.x || v.w != v.y) record_stamp<MODE>(v.z, v.w, p, cache);
  }
  if (tail != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    record_stamp<MODE>(tail[0], tail[1], p, cache);
  pdl_trigger();
}

// Close tick T for layout S: per BDR, the active ranks are those with a stamp
// and T - stamp < k (IsActiveDR, on the derived age); M = the
// highest (Alg.2), PCSA's R = the active run from rank 1.  Streams 4 L bytes
// per BDR, writes nothing back but the register.
template <bool PCSA>
__global__ void __launch_bounds__(kThreads) k_slide_stamps(DevParams p, uint32_t slot) {
  pdl_wait();
  const uint64_t n4 = p.n_phys >> 2;
  const uint4 *st4 = reinterpret_cast<const uint4 *>(p.drv);
  uint32_t *reg4 = reinterpret_cast<uint32_t *>(p.regmax);
  unsigned long long s_acc = 0;
  uint32_t v_acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t q = (uint64_t)blockIdx.x * kThreads + threadIdx.x; q < n4; q += stride) {
    uint32_t act[4] = {0u, 0u, 0u, 0u};  // bit rho - 1: rank rho active
#pragma unroll 8
    for (uint32_t r = 0; r < p.L; ++r) {
      const uint4 s = __ldcs(st4 + (uint64_t)r * n4 + q);
      const uint32_t sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
      for (int c = 0; c < 4; ++c)
        act[c] |= (uint32_t)(sv[c] != 0u && p.tick - sv[c] < p.k) << r;
    }
    uint32_t best[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if constexpr (PCSA)
        best[c] = min((uint32_t)__ffs(~act[c]) - 1u, p.L);  // consecutive active from rank 1
      else
        best[c] = act[c] ? 32u - (uint32_t)__clz(act[c]) : 0u;
    }
    reg4[q] = best[0] | (best[1] << 8) | (best[2] << 16) | (best[3] << 24);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      s_acc += p.est == 0u ? 1ull << (p.L - best[c]) : (unsigned long long)best[c];
      v_acc += best[c] == 0u;
    }
  }
  pdl_trigger();
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    s_acc += __shfl_xor_sync(0xffffffffu, s_acc, off);
    v_acc += __shfl_xor_sync(0xffffffffu, v_acc, off);
  }
  __shared__ unsigned long long ss[kThreads / 32];
  __shared__ uint32_t sv[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    ss[warp] = s_acc;
    sv[warp] = v_acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long st = 0, vt = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      st += ss[w];
      vt += sv[w];
    }
    atomicAdd(p.acc + 2 * slot, st);
    atomicAdd(p.acc + 2 * slot + 1, vt);
    if (blockIdx.x == 0) {
      p.acc[2 * ((slot + 1u) & 3u)] = 0ull;
      p.acc[2 * ((slot + 1u) & 3u) + 1] = 0ull;
    }
  }
}

// ------------------------------------------------------------------ slide
// One thread = 4 consecutive BDRs (16-byte loads of every plane).
//   FAST:   age all DRs (Alg.1), SetDR(DRV[nowLBP1]) if sr is from
//           this tick (Alg.1, R#9), M = GetLBP1BDR (Alg.2).
//   PACKED: M = GetLBP1BDR of the ages at this boundary (Alg.2), then age all
//           DRs for the next slice (Alg.8 hoisted from the next slice open).
// Writes regmax[j] = M and accumulates S_tot = sum 2^(L-M), V_tot = #{M=0}.
// Where this slice's max rank per BDR comes from (FAST layout only):
//   SRC_STAMPS: the local stamps sr (one GPU, or after an allreduce of sr);
//   SRC_DELTA:  a merged u8 array, delta4[q - q0] packing BDRs 4q..4q+3;
//   SRC_PEERS:  the ranks' own u8 deltas read in place (NVLink peer memory on
//               a multi-GPU box) and merged here with a per-byte max -- the
//               merge is fused into the slide, no collective runs.  With
//               peer register/accumulator pointers the kernel also writes its
//               register shard and adds its pool sums into every rank.
// Only BDR quads [q0, q1) are processed (the rank's shard).
//   SRC_NVLS:   every rank's copy of the state in one multicast (NVLS) object
//               (vbdr_slide_multicast): the merge is done by
//               the NVSwitch as the kernel loads -- multimem.ld_reduce MAX of
//               the stamps (layout fast) or AND of the packed DRV words
//               (layout packed: every rank cleared fields of its own copy,
//               Alg.9 SetDR, and AND merges clears) -- and the kernel's results
//               go to every rank with multimem.st (registers; packed: the new
//               DRV words) and multimem.red (pool sums).  No collective runs.
//   SRC_ONE:    SRC_NVLS for a group of one without a multicast object (the
//               "multicast" address is the handle's own state): the same
//               kernel with the multimem operations replaced by the ordinary
//               load / store / atomic they reduce to over a single member.
enum { SRC_STAMPS = 0, SRC_DELTA = 1, SRC_PEERS = 2, SRC_NVLS = 3, SRC_ONE = 4 };

template <bool MC>
__device__ __forceinline__ uint32_t mc_ld_max(const uint32_t *a) {
  if constexpr (!MC) return __ldcg(a);
  uint32_t v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
template <bool MC>
__device__ __forceinline__ unsigned long long mc_ld_and64(const uint32_t *a) {
  if constexpr (!MC) return __ldcg(reinterpret_cast<const unsigned long long *>(a));
  unsigned long long v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.and.b64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
template <bool MC>
__device__ __forceinline__ void mc_st64(uint32_t *a, unsigned long long v) {
  if constexpr (!MC) {
    __stcg(reinterpret_cast<unsigned long long *>(a), v);
    return;
  }
  asm volatile("multimem.st.relaxed.sys.global.b64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
template <bool MC>
__device__ __forceinline__ void mc_st32(void *a, uint32_t v) {
  if constexpr (!MC) {
    __stcg(reinterpret_cast<uint32_t *>(a), v);
    return;
  }
  asm volatile("multimem.st.relaxed.sys.global.b32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
template <bool MC>
__device__ __forceinline__ void mc_red_add64(unsigned long long *a, unsigned long long v) {
  if constexpr (!MC) {
    atomicAdd(a, v);
    return;
  }
  asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

// PCSA (layout packed only): the register value written is R = the number of
// consecutive active ranks from rank 1 (the sliding FM bitmap's lowest zero,
// N4 variant) instead of M (Alg.2).
template <bool FAST, int ZB, int SRC, bool PCSA = false>
__global__ void __launch_bounds__(kThreads)
k_slide(DevParams p, uint32_t addk, uint32_t slot, const uint32_t *__restrict__ delta4,
        uint64_t q0, uint64_t q1, vbdr_launch::Peers peers) {
  pdl_wait();
  using S = Swar<ZB>;
  constexpr int WM = WMax<ZB>::value;
  constexpr bool NV = SRC == SRC_NVLS || SRC == SRC_ONE;  // the multicast slide
  constexpr bool MC = SRC == SRC_NVLS;                    // ... through real multimem ops
  const uint4 *sr4 = reinterpret_cast<const uint4 *>(p.sr);
  // the DRV holds BDR quads [dq0, dq0 + dn4) (all of them unless register-sharded)
  const uint64_t dn4 = p.drv_n >> 2, dq0 = p.drv_j0 >> 2;
  uint4 *drv4 = reinterpret_cast<uint4 *>(p.drv);
  uint32_t *reg4 = reinterpret_cast<uint32_t *>(p.regmax);
  unsigned long long s_acc = 0;
  uint32_t v_acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t q = q0 + (uint64_t)blockIdx.x * kThreads + threadIdx.x; q < q1; q += stride) {
    uint32_t hit[4] = {0u, 0u, 0u, 0u};  // this slice's max rank of each BDR, or 0
    if constexpr (FAST && SRC == SRC_DELTA) {
      const uint32_t d = __ldcs(delta4 + (q - q0));
#pragma unroll
      for (int c = 0; c < 4; ++c) hit[c] = (d >> (8 * c)) & 0xFFu;
    } else if constexpr (FAST && SRC == SRC_PEERS) {
      uint32_t d = 0u;
      for (uint32_t r = 0; r < peers.n; ++r)
        d = __vmaxu4(d, __ldcs(reinterpret_cast<const uint32_t *>(peers.delta[r]) + q));
#pragma unroll
      for (int c = 0; c < 4; ++c) hit[c] = (d >> (8 * c)) & 0xFFu;
    } else if constexpr (FAST && NV) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // max over every rank's stamp (NVSwitch reduction)
        const uint32_t sv = mc_ld_max<MC>(peers.sr_mc + 4 * q + c);
        hit[c] = ((sv >> 5) == p.tick) ? (sv & 31u) : 0u;
      }
    } else if constexpr (FAST) {
      const uint4 s = __ldcs(sr4 + q);
      const uint32_t sv[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) hit[c] = ((sv[c] >> 5) == p.tick) ? (sv[c] & 31u) : 0u;
    }
    uint4 x[WM];
#pragma unroll
    for (int w = 0; w < WM; ++w) {
      if (w >= (int)p.W) continue;
      if constexpr (!FAST && NV) {  // AND over every rank's copy of the words
        const uint32_t *a = peers.drv_mc + (uint64_t)w * p.drv_n + 4 * q;
        const unsigned long long lo = mc_ld_and64<MC>(a), hi = mc_ld_and64<MC>(a + 2);
        x[w] = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
      } else {
        x[w] = drv4[(uint64_t)w * dn4 + (q - dq0)];
      }
    }
    // where the slid words go: local, or (packed, NVLS) every rank's copy
    auto store_words = [&](int w, const uint4 &v) {
      if constexpr (!FAST && NV) {
        uint32_t *a = peers.drv_mc + (uint64_t)w * p.drv_n + 4 * q;
        mc_st64<MC>(a, (unsigned long long)v.x | ((unsigned long long)v.y << 32));
        mc_st64<MC>(a + 2, (unsigned long long)v.z | ((unsigned long long)v.w << 32));
      } else {
        drv4[(uint64_t)w * dn4 + (q - dq0)] = v;
      }
    };
    uint32_t best[4] = {0u, 0u, 0u, 0u};
    uint32_t run[4] = {0u, 0u, 0u, 0u};  // PCSA: active ranks from the bottom of word w up
#pragma unroll
    for (int w = WM - 1; w >= 0; --w) {
      if (w >= (int)p.W) continue;
      uint32_t xv[4] = {x[w].x, x[w].y, x[w].z, x[w].w};
      uint32_t clr[4] = {0u, 0u, 0u, 0u};  // FAST: the field Alg.1's SetDR clears in this word
      bool sat = true;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if constexpr (FAST) {
          const uint32_t r = hit[c] - 1u;
          const uint32_t ws = r / (uint32_t)S::F;
          clr[c] = (hit[c] != 0u && ws == (uint32_t)w) ? S::FM << (ZB * (r - ws * (uint32_t)S::F))
                                                       : 0u;
        }
        sat = sat && xv[c] == S::INIT && clr[c] == 0u;
      }
#if VBDR_SLIDE_SKIP
      // Words whose fields are all saturated (the InitDR pattern) stay so
      // under SlideDR and hold no active rank; when that is true for the whole
      // warp (typical for the high-rank words) skip the SWAR work.
      if (__all_sync(__activemask(), sat)) {
#if VBDR_SLIDE_SKIP == 2
        store_words(w, x[w]);  // unchanged, stored anyway
#endif
        if constexpr (PCSA) {
#pragma unroll
          for (int c = 0; c < 4; ++c) run[c] = 0u;  // no active field in this word
        }
        continue;  // VBDR_SLIDE_SKIP 1: unchanged words are not rewritten
      }
#endif
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t a;
        if constexpr (FAST) {
          xv[c] = S::age(xv[c]) & ~clr[c];  // Alg.1: SlideDR every DR, then SetDR(DRV[nowLBP1])
          a = S::active(xv[c], addk);       // Alg.2 on the new ages
        } else {
          a = S::active(xv[c], addk);  // Alg.2 on this boundary's ages
          xv[c] = S::age(xv[c]);       // Alg.8 for the next slice
        }
        if (best[c] == 0u && a != 0u) best[c] = (uint32_t)w * S::F + S::top_field(a) + 1u;
        if constexpr (PCSA) {
          const uint32_t inact = ~a & S::LSB;  // unused high fields are S: inactive
          run[c] = inact ? (uint32_t)(__ffs(inact) - 1) / (uint32_t)ZB : (uint32_t)S::F + run[c];
        }
      }
      store_words(w, make_uint4(xv[0], xv[1], xv[2], xv[3]));
    }
    if constexpr (PCSA) {
#pragma unroll
      for (int c = 0; c < 4; ++c) best[c] = min(run[c], p.L);
    }
    const uint32_t r4 = best[0] | (best[1] << 8) | (best[2] << 16) | (best[3] << 24);
    if constexpr (NV) {
      mc_st32<MC>(peers.regmax_mc + 4 * q, r4);  // every rank's register buffer
    } else if (SRC == SRC_PEERS && peers.n_regmax > 0) {
      for (uint32_t r = 0; r < peers.n_regmax; ++r) reinterpret_cast<uint32_t *>(peers.regmax[r])[q] = r4;
    } else {
      reg4[q] = r4;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // HLL: harmonic sum 2^(L - M); LogLog / PCSA: plain sum of the values
      s_acc += p.est == 0u ? 1ull << (p.L - best[c]) : (unsigned long long)best[c];
      v_acc += best[c] == 0u;
    }
  }
  pdl_trigger();
  // block reduction, one atomic per block (integers: order-independent)
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    s_acc += __shfl_xor_sync(0xffffffffu, s_acc, off);
    v_acc += __shfl_xor_sync(0xffffffffu, v_acc, off);
  }
  __shared__ unsigned long long ss[kThreads / 32];
  __shared__ uint32_t sv[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    ss[warp] = s_acc;
    sv[warp] = v_acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long st = 0, vt = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      st += ss[w];
      vt += sv[w];
    }
    if constexpr (SRC == SRC_NVLS || SRC == SRC_ONE) {
      mc_red_add64<SRC == SRC_NVLS>(peers.acc_mc + 2 * slot, st);  // into every rank's slot
      mc_red_add64<SRC == SRC_NVLS>(peers.acc_mc + 2 * slot + 1, vt);
    } else if (SRC == SRC_PEERS && peers.n_acc > 0) {
      for (uint32_t r = 0; r < peers.n_acc; ++r) {
        atomicAdd(peers.acc[r] + 2 * slot, st);
        atomicAdd(peers.acc[r] + 2 * slot + 1, vt);
      }
    } else {
      atomicAdd(p.acc + 2 * slot, st);
      atomicAdd(p.acc + 2 * slot + 1, vt);
    }
    if (blockIdx.x == 0) {  // the next tick's slot is the next slide's accumulator
      p.acc[2 * ((slot + 1u) & 3u)] = 0ull;
      p.acc[2 * ((slot + 1u) & 3u) + 1] = 0ull;
    }
  }
}

// ------------------------------------------------------------- delta
// Compact the stamps of the open slice to one byte per BDR: rho if the stamp
// is from tick T, else 0 (the u8 merge payload, 4x less than the stamps).
__global__ void __launch_bounds__(kThreads) k_delta(DevParams p, uint32_t *__restrict__ delta4) {
  const uint64_t n4 = p.n_phys >> 2;
  const uint4 *sr4 = reinterpret_cast<const uint4 *>(p.sr);
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t q = (uint64_t)blockIdx.x * kThreads + threadIdx.x; q < n4; q += stride) {
    const uint4 s = __ldcs(sr4 + q);
    const uint32_t sv[4] = {s.x, s.y, s.z, s.w};
    uint32_t d = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) d |= (((sv[c] >> 5) == p.tick) ? (sv[c] & 31u) : 0u) << (8 * c);
    __stcs(delta4 + q, d);
  }
}

// ------------------------------------------------------- sparse exchange
// SURVEY.md 8(e) iii: for pools far sparser than a slice (bigwin: 0.06 pairs
// per BDR), the ranks exchange only the BDRs their pairs touched: record
// ((j - j0(o)) << 5) | rho for every BDR j with a stamp from the open tick,
// listed per owner rank o (BDR shards of `shard` BDRs), then each owner folds
// the records it receives into its u8 delta shard with a per-byte max.
__global__ void __launch_bounds__(kThreads)
k_sparse_extract(DevParams p, uint64_t shard, uint32_t *__restrict__ records, uint64_t cap,
                 unsigned long long *__restrict__ counts) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t n = p.n_phys;
  const uint64_t n_round = (n + 31) & ~uint64_t(31);
  for (uint64_t j = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j < n_round; j += stride) {
    uint32_t sv = 0u;
    if (j < n) sv = __ldcs(p.sr + j);
    const bool hit = j < n && (sv >> 5) == p.tick;
    const uint32_t owner = hit ? (uint32_t)(j / shard) : 0xFFFFFFFFu;
    // one counter atomic per (warp, owner): lanes of a warp share owners
    const uint32_t peers = __match_any_sync(0xffffffffu, owner);
    const uint32_t leader = __ffs(peers) - 1u;
    unsigned long long base = 0;
    if (hit && lane == leader) base = atomicAdd(counts + owner, (unsigned long long)__popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) {
      const unsigned long long k = base + __popc(peers & ((1u << lane) - 1u));
      if (k < cap)
        records[(uint64_t)owner * cap + k] = (uint32_t)((j - (uint64_t)owner * shard) << 5) | (sv & 31u);
    }
  }
}

// delta[r >> 5] = max(delta[r >> 5], r & 31) for every received record (a
// byte max by compare-and-swap on the containing word; records for the same
// BDR come from at most one record per rank).
__global__ void __launch_bounds__(kThreads)
k_sparse_apply(const uint32_t *__restrict__ records, uint64_t n, uint32_t *__restrict__ delta4) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const uint32_t r = __ldcs(records + i);
    const uint64_t jl = r >> 5;
    const uint32_t rho = r & 31u, sh = 8u * (uint32_t)(jl & 3u);
    uint32_t *w = delta4 + (jl >> 2);
    uint32_t old = *w;
    while (((old >> sh) & 0xFFu) < rho) {
      const uint32_t want = (old & ~(0xFFu << sh)) | (rho << sh);
      const uint32_t got = atomicCAS(w, old, want);
      if (got == old) break;
      old = got;
    }
  }
}

// ------------------------------------------------------------------ init
// InitDR on every DR, stamps and registers 0 (the first
// register buffer; the host clears the second).  Accumulator slot 0 describes
// the empty window (all M = 0) so estimates before the first slide are 0;
// slot 1 is the first slide's accumulator.
template <int ZB>
__global__ void __launch_bounds__(kThreads) k_init(DevParams p, bool fast) {
  using S = Swar<ZB>;
  const uint64_t n4 = p.n_phys >> 2;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint4 *drv4 = reinterpret_cast<uint4 *>(p.drv);
  const uint64_t dn4 = p.drv_n >> 2, dq0 = p.drv_j0 >> 2;
  for (uint64_t q = (uint64_t)blockIdx.x * kThreads + threadIdx.x; q < n4; q += stride) {
    if (q >= dq0 && q < dq0 + dn4)
      for (uint32_t w = 0; w < p.W; ++w)
        drv4[(uint64_t)w * dn4 + (q - dq0)] = make_uint4(S::INIT, S::INIT, S::INIT, S::INIT);
    if (fast) reinterpret_cast<uint4 *>(p.sr)[q] = make_uint4(0u, 0u, 0u, 0u);
    reinterpret_cast<uint32_t *>(p.regmax)[q] = 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.acc[0] = p.est == 0u ? (unsigned long long)p.n_phys << p.L : 0ull;
    p.acc[1] = p.n_phys;
    for (int i = 2; i < 8; ++i) p.acc[i] = 0ull;
  }
}

// ------------------------------------------------------------- export
// Gather the W packed words of sampled BDRs (parity exports of huge pools).
__global__ void __launch_bounds__(kThreads)
k_gather_words(DevParams p, const uint64_t *__restrict__ idx, uint64_t n, uint32_t *out) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
    const uint64_t j = idx[i];
    for (uint32_t w = 0; w < p.W; ++w)
      out[i * p.W + w] = (j >= p.drv_j0 && j < p.drv_j0 + p.drv_n)
                             ? p.drv[(uint64_t)w * p.drv_n + (j - p.drv_j0)]
                             : 0u;  // outside the (shard of the) pool
  }
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

// Persistent grid: as many blocks as can be resident (occupancy of this
// kernel x SM count), never more than the work needs.
template <typename K>
uint32_t grid_for(K kernel, uint64_t work, int threads = kThreads, size_t smem = 0) {
  static int resident = 0;  // one static per kernel instantiation
  if (resident == 0) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess ||
        per_sm <= 0)
      per_sm = 1;
    resident = per_sm * sm_count();
  }
  const uint64_t need = (work + threads - 1) / threads;
  const uint64_t g = need < (uint64_t)resident ? need : (uint64_t)resident;
  return (uint32_t)(g ? g : 1);
}

template <template <int> class Fn, typename... Args>
cudaError_t dispatch_zb(uint32_t zb, Args &&...args) {
  switch (zb) {
    case 1: return Fn<1>::run(args...);
    case 2: return Fn<2>::run(args...);
    case 3: return Fn<3>::run(args...);
    case 4: return Fn<4>::run(args...);
    case 5: return Fn<5>::run(args...);
    case 6: return Fn<6>::run(args...);
    case 7: return Fn<7>::run(args...);
    case 8: return Fn<8>::run(args...);
    case 9: return Fn<9>::run(args...);
    case 10: return Fn<10>::run(args...);
    default: return cudaErrorInvalidValue;
  }
}

template <int ZB>
struct InitFn {
  static cudaError_t run(const DevParams &p, bool fast, cudaStream_t s) {
    k_init<ZB><<<grid_for(k_init<ZB>, p.n_phys >> 2), kThreads, 0, s>>>(p, fast);
    return cudaGetLastError();
  }
};

template <int ZB, int SRC>
cudaError_t launch_nvls_zb(const DevParams &p, bool fast, uint32_t addk, uint32_t slot, uint64_t q0,
                           uint64_t q1, const vbdr_launch::Peers &pe, cudaStream_t s) {
  const uint64_t work = q1 - q0;
  if (fast)
    return launch(k_slide<true, ZB, SRC>, grid_for(k_slide<true, ZB, SRC>, work), kThreads, 0, s,
                  p, addk, slot, (const uint32_t *)nullptr, q0, q1, pe);
  if (p.est == 2)
    return launch(k_slide<false, ZB, SRC, true>, grid_for(k_slide<false, ZB, SRC, true>, work),
                  kThreads, 0, s, p, addk, slot, (const uint32_t *)nullptr, q0, q1, pe);
  return launch(k_slide<false, ZB, SRC>, grid_for(k_slide<false, ZB, SRC>, work), kThreads, 0, s,
                p, addk, slot, (const uint32_t *)nullptr, q0, q1, pe);
}

template <int ZB>
struct SlideFn {
  template <int SRC>
  static cudaError_t launch_nvls(const DevParams &p, bool fast, uint32_t addk, uint32_t slot,
                                 uint64_t q0, uint64_t q1, const vbdr_launch::Peers &pe,
                                 cudaStream_t s) {
    return launch_nvls_zb<ZB, SRC>(p, fast, addk, slot, q0, q1, pe, s);
  }
  static cudaError_t run(const DevParams &p, bool fast, const uint32_t *delta4, uint64_t q0,
                         uint64_t q1, const vbdr_launch::Peers *peers, cudaStream_t s) {
    // (2^zb - k) at every even field's LSB (Swar::active)
    uint32_t addk = 0;
    for (uint32_t f = 0; f < Swar<ZB>::F; f += 2) addk |= ((1u << ZB) - p.k) << (ZB * f);
    const uint32_t slot = p.tick & 3u;  // four slots: the estimate of tick T-1 may still read its own
    const uint64_t work = q1 - q0;
    const vbdr_launch::Peers none{};
    if (peers && peers->nvls == 1) return launch_nvls<SRC_NVLS>(p, fast, addk, slot, q0, q1, *peers, s);
    if (peers && peers->nvls == 2) return launch_nvls<SRC_ONE>(p, fast, addk, slot, q0, q1, *peers, s);
    if (fast && peers)
      return launch(k_slide<true, ZB, SRC_PEERS>, grid_for(k_slide<true, ZB, SRC_PEERS>, work),
                    kThreads, 0, s, p, addk, slot, (const uint32_t *)nullptr, q0, q1, *peers);
    if (fast && delta4)
      return launch(k_slide<true, ZB, SRC_DELTA>, grid_for(k_slide<true, ZB, SRC_DELTA>, work),
                    kThreads, 0, s, p, addk, slot, delta4, q0, q1, none);
    if (fast)
      return launch(k_slide<true, ZB, SRC_STAMPS>, grid_for(k_slide<true, ZB, SRC_STAMPS>, work),
                    kThreads, 0, s, p, addk, slot, (const uint32_t *)nullptr, q0, q1, none);
    if (p.est == 2)
      return launch(k_slide<false, ZB, SRC_STAMPS, true>,
                    grid_for(k_slide<false, ZB, SRC_STAMPS, true>, work), kThreads, 0, s, p, addk,
                    slot, (const uint32_t *)nullptr, q0, q1, none);
    return launch(k_slide<false, ZB, SRC_STAMPS>, grid_for(k_slide<false, ZB, SRC_STAMPS>, work),
                  kThreads, 0, s, p, addk, slot, (const uint32_t *)nullptr, q0, q1, none);
  }
};

template <bool FAST, int ZB>
cudaError_t launch_scan(const DevParams &p, int mode, const uint4 *pairs2, uint64_t n2,
                        const uint32_t *tail, cudaStream_t s) {
  const uint64_t work = n2 ? n2 : 1;
  constexpr int T = kScanThreads;
  constexpr size_t cache_bytes = sizeof(ScanCache);
  switch (mode) {
    case 2:
      return launch(k_scan<FAST, ZB, 2>, grid_for(k_scan<FAST, ZB, 2>, work, T), T, 0, s, pairs2,
                    n2, tail, p);
    case 5:
      return launch(k_scan<FAST, ZB, 5>, grid_for(k_scan<FAST, ZB, 5>, work, T, cache_bytes), T,
                    cache_bytes, s, pairs2, n2, tail, p);
    default:
      return cudaErrorInvalidValue;
  }
}

template <int ZB>
struct ScanPackedFn {
  static cudaError_t run(const DevParams &p, int mode, const uint4 *pairs2, uint64_t n2,
                         const uint32_t *tail, cudaStream_t s) {
    return launch_scan<false, ZB>(p, mode, pairs2, n2, tail, s);
  }
};

}  // namespace

namespace vbdr_launch {

cudaError_t init(const DevParams &p, bool fast, cudaStream_t s) {
  return dispatch_zb<InitFn>(p.zb, p, fast, s);
}

cudaError_t slide(const DevParams &p, bool fast, cudaStream_t s) {
  return dispatch_zb<SlideFn>(p.zb, p, fast, (const uint32_t *)nullptr, (uint64_t)0,
                              p.n_phys >> 2, (const Peers *)nullptr, s);
}

cudaError_t slide_delta(const DevParams &p, const uint8_t *delta, uint64_t j0, uint64_t j1,
                        cudaStream_t s) {
  return dispatch_zb<SlideFn>(p.zb, p, true, reinterpret_cast<const uint32_t *>(delta), j0 >> 2,
                              j1 >> 2, (const Peers *)nullptr, s);
}

cudaError_t slide_peers(const DevParams &p, const Peers &peers, uint64_t j0, uint64_t j1,
                        cudaStream_t s) {
  return dispatch_zb<SlideFn>(p.zb, p, true, (const uint32_t *)nullptr, j0 >> 2, j1 >> 2, &peers,
                              s);
}

cudaError_t slide_multicast(const DevParams &p, const Peers &mc, uint64_t j0, uint64_t j1,
                            bool fast, cudaStream_t s) {
  return dispatch_zb<SlideFn>(p.zb, p, fast, (const uint32_t *)nullptr, j0 >> 2, j1 >> 2, &mc, s);
}

cudaError_t scan_stamps(const DevParams &p, int mode, const uint32_t *pairs, uint64_t n,
                        cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t n2 = n >> 1;
  const uint32_t *tail = (n & 1u) ? pairs + 2 * (n - 1) : nullptr;
  const uint4 *pairs2 = reinterpret_cast<const uint4 *>(pairs);
  const uint64_t work = n2 ? n2 : 1;
  constexpr int T = kScanThreads;
  if (mode == 5)
    return launch(k_scan_stamps<5>, grid_for(k_scan_stamps<5>, work, T, sizeof(ScanCache)), T,
                  sizeof(ScanCache), s, pairs2, n2, tail, p);
  return launch(k_scan_stamps<2>, grid_for(k_scan_stamps<2>, work, T), T, 0, s, pairs2, n2, tail, p);
}

cudaError_t slide_stamps(const DevParams &p, cudaStream_t s) {
  const uint32_t slot = p.tick & 3u;
  const uint64_t work = p.n_phys >> 2;
  if (p.est == 2)
    return launch(k_slide_stamps<true>, grid_for(k_slide_stamps<true>, work), kThreads, 0, s, p, slot);
  return launch(k_slide_stamps<false>, grid_for(k_slide_stamps<false>, work), kThreads, 0, s, p, slot);
}

cudaError_t delta(const DevParams &p, uint8_t *out, cudaStream_t s) {
  k_delta<<<grid_for(k_delta, p.n_phys >> 2), kThreads, 0, s>>>(p, reinterpret_cast<uint32_t *>(out));
  return cudaGetLastError();
}

cudaError_t sparse_extract(const DevParams &p, uint32_t owners, uint32_t *records, uint64_t cap,
                           unsigned long long *counts, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(counts, 0, 8ull * owners, s);
  if (e != cudaSuccess) return e;
  k_sparse_extract<<<grid_for(k_sparse_extract, p.n_phys), kThreads, 0, s>>>(
      p, p.n_phys / owners, records, cap, counts);
  return cudaGetLastError();
}

cudaError_t sparse_apply(const uint32_t *records, uint64_t n, uint8_t *delta, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_sparse_apply<<<grid_for(k_sparse_apply, n), kThreads, 0, s>>>(
      records, n, reinterpret_cast<uint32_t *>(delta));
  return cudaGetLastError();
}

cudaError_t gather_words(const DevParams &p, const uint64_t *idx, uint64_t n, uint32_t *out,
                         cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_gather_words<<<grid_for(k_gather_words, n), kThreads, 0, s>>>(p, idx, n, out);
  return cudaGetLastError();
}

cudaError_t scan(const DevParams &p, bool fast, int mode, const uint32_t *pairs, uint64_t n,
                 cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const uint64_t n2 = n >> 1;
  const uint32_t *tail = (n & 1u) ? pairs + 2 * (n - 1) : nullptr;
  const uint4 *pairs2 = reinterpret_cast<const uint4 *>(pairs);
  if (fast) return launch_scan<true, 1>(p, mode, pairs2, n2, tail, s);
  return dispatch_zb<ScanPackedFn>(p.zb, p, mode, pairs2, n2, tail, s);
}

}  // namespace vbdr_launch
