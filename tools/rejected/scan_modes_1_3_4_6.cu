// RECORD ONLY (not compiled, not part of libvbdr.so): the round-1 scan modes that
// measured slower than the default (profiles/r01_scan_modes.txt) and were
// removed from the product library in round 2.  Mode 1: plain atomic per pair;
// mode 3: warp-aggregated atomic (__match_any_sync + __reduce_max_sync, the
// north star's literal wording; 2.4x slower than mode 5 at caida); mode 4:
// L1-cached load-check; mode 6: binned scan (per-bucket bins, shared-memory
// max, coalesced stamp merge; 1.4x slower).  Extracted verbatim from
// paper_1810_13132_b200/csrc/k_scan_slide.cu at commit 6a87544.

    if constexpr (MODE == 3) {
      // warp-aggregated atomicMax (north star): lanes hitting the same BDR
      // combine their ranks with a max reduction, the lowest of them checks
      // L2 (as mode 2) and issues the one atomic
      const uint32_t live = __activemask();
      const uint32_t peers = __match_any_sync(live, pidx);
      const uint32_t m = __reduce_max_sync(peers, val);
      if ((threadIdx.x & 31u) != (uint32_t)(__ffs(peers) - 1)) return;
      if (ld_relaxed(a) >= m) return;
      atomicMax(a, m);
      return;
    }
    if constexpr (MODE == 2) {
      if (ld_relaxed(a) >= val) return;  // stored value dominates: max is a no-op
    }
    if constexpr (MODE == 4) {
      // L1-cached check: a stale line can only hold a smaller (older) value,
      // so skipping when it dominates is still exact
      if (__ldca(a) >= val) return;
    }
    atomicMax(a, val);
    // ... packed layout:
    if constexpr (MODE == 3) {
      // warp-aggregated SetDR: lanes hitting the same word OR their field
      // masks, the lowest of them checks L2 and issues the one atomicAnd
      const uint32_t live = __activemask();
      const uint32_t peers = __match_any_sync(live, (unsigned long long)(uintptr_t)a);
      const uint32_t m = __reduce_or_sync(peers, fm);
      if ((threadIdx.x & 31u) != (uint32_t)(__ffs(peers) - 1)) return;
      if ((ld_relaxed(a) & m) == 0u) return;
      atomicAnd(a, ~m);
      return;
    }
    if constexpr (MODE == 2) {
      if ((ld_relaxed(a) & fm) == 0u) return;  // already zero
    }
    if constexpr (MODE == 4) {
      // within a slice fields only go to zero: a stale (older) line showing
      // zero is still zero now
      if ((__ldca(a) & fm) == 0u) return;
    }

// ------------------------------------------------------------ binned scan
// MODE 6 (layout F): the random 4-byte atomics of the other modes are bound by
// L2 sector operations (one per pair, plus the check load).  Here a chunk of
// pairs is first PARTITIONED by bucket (2^bkt_log2 consecutive BDRs, 16K) into
// per-bucket record bins -- sequential writes -- and then every bucket's
// records are reduced in shared memory (atomicMax on the rank) and merged
// into the bucket's stamp words with coalesced loads and stores.  Same
// nowLBP1 = max rank per BDR per slice as the atomic modes,
// bit-identical state.  A record that finds its bin full falls back to the
// direct atomicMax (exact, just slower), so no input can overflow.
constexpr int kBinThreads = 1024;
constexpr int kBinPairs = 8;  // pairs per thread per tile (4 x 16-byte loads)
constexpr int kBinTile = kBinThreads * kBinPairs;  // 8192 pairs
constexpr uint32_t kNoBkt = 0xFFFFFFFFu;

// Shared memory of k_bin for n_bkt buckets: per bucket count, tile start and
// bin base (3 x u32), per tile slot the record (u32) and its bucket (u16).
__host__ __device__ inline size_t bin_smem(uint32_t n_bkt) {
  return (size_t)12 * n_bkt + (size_t)6 * kBinTile;
}

// Per tile: (1) ranks within the tile's buckets (shared atomics); (2) bucket
// starts in the tile (block scan) and one global reservation per bucket;
// (3) records placed bucket-sorted in shared memory; (4) written out by
// consecutive threads, so each bucket's run of the tile is one coalesced
// stretch of its bin.
__global__ void __launch_bounds__(kBinThreads)
k_bin(const uint4 *__restrict__ pairs2, uint64_t n2, const uint32_t *__restrict__ tail,
      DevParams p) {
  pdl_wait();
  extern __shared__ uint32_t bin_sm[];
  const uint32_t n_bkt = (uint32_t)(p.n_phys >> p.bkt_log2);
  uint32_t *cnt = bin_sm;                  // [n_bkt]
  uint32_t *start = cnt + n_bkt;           // [n_bkt]
  uint32_t *gbase = start + n_bkt;         // [n_bkt]
  uint32_t *srec = gbase + n_bkt;          // [kBinTile]
  uint16_t *sbkt = reinterpret_cast<uint16_t *>(srec + kBinTile);  // [kBinTile]
  __shared__ uint32_t warp_tot[kBinThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
  for (uint32_t b = tid; b < n_bkt; b += kBinThreads) cnt[b] = 0u;
  __syncthreads();
  const uint32_t tickbits = p.tick << 5;
  const uint32_t omask = (1u << p.bkt_log2) - 1u;
  constexpr uint64_t kTile4 = kBinTile / 2;  // uint4 per tile
  const uint32_t per_thr = (n_bkt + kBinThreads - 1) / kBinThreads;  // buckets per thread
  for (uint64_t t0 = (uint64_t)blockIdx.x * kTile4; t0 < n2; t0 += (uint64_t)gridDim.x * kTile4) {
    uint32_t bkt[kBinPairs], rec[kBinPairs], rank[kBinPairs];
#pragma unroll
    for (int u = 0; u < kBinPairs / 2; ++u) {
      const uint64_t i = t0 + (uint64_t)u * kBinThreads + tid;
      const bool ok = i < n2;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (ok) v = __ldcs(pairs2 + i);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int q = 2 * u + h;
        uint32_t pidx, rho;
        pair_index(h ? v.z : v.x, h ? v.w : v.y, p, pidx, rho);
        bkt[q] = ok ? pidx >> p.bkt_log2 : kNoBkt;
        rec[q] = ((pidx & omask) << 5) | rho;
        rank[q] = ok ? atomicAdd(cnt + bkt[q], 1u) : 0u;
      }
    }
    __syncthreads();
    // exclusive scan of the bucket counts: thread t owns buckets
    // [t * per_thr, (t + 1) * per_thr); reserve each non-empty bucket's run
    uint32_t local = 0;
    for (uint32_t j = 0; j < per_thr; ++j) {
      const uint32_t b = tid * per_thr + j;
      if (b < n_bkt) local += cnt[b];
    }
    uint32_t x = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= (uint32_t)off) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    uint32_t wpre = 0;
    for (uint32_t w = 0; w < wid; ++w) wpre += warp_tot[w];
    uint32_t run = wpre + x - local;
    for (uint32_t j = 0; j < per_thr; ++j) {
      const uint32_t b = tid * per_thr + j;
      if (b < n_bkt) {
        const uint32_t c = cnt[b];
        start[b] = run;
        if (c) gbase[b] = atomicAdd(p.bcursor + b, c);
        run += c;
      }
    }
    __syncthreads();
    uint32_t n_tile = 0;
#pragma unroll
    for (int w = 0; w < kBinThreads / 32; ++w) n_tile += warp_tot[w];
#pragma unroll
    for (int q = 0; q < kBinPairs; ++q) {
      if (bkt[q] == kNoBkt) continue;
      const uint32_t s = start[bkt[q]] + rank[q];
      srec[s] = rec[q];
      sbkt[s] = (uint16_t)bkt[q];
    }
    __syncthreads();
    for (uint32_t i = tid; i < n_tile; i += kBinThreads) {
      const uint32_t b = sbkt[i];
      const uint32_t pos = gbase[b] + (i - start[b]);
      const uint32_t r = srec[i];
      if (pos < p.bcap) {
        p.bins[(uint64_t)b * p.bcap + pos] = r;
      } else {  // bin full: the direct update (mode 1)
        atomicMax(p.sr + (((uint64_t)b << p.bkt_log2) | (r >> 5)), tickbits | (r & 31u));
      }
    }
    for (uint32_t j = 0; j < per_thr; ++j) {
      const uint32_t b = tid * per_thr + j;
      if (b < n_bkt) cnt[b] = 0u;
    }
    __syncthreads();
  }
  if (tail != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t pidx, rho;
    pair_index(tail[0], tail[1], p, pidx, rho);
    atomicMax(p.sr + pidx, tickbits | rho);
  }
  pdl_trigger();
}

// One CTA per bucket: max rank per BDR in shared memory, then merged into the
// bucket's stamp words (only words whose BDR received a pair are touched).
__global__ void __launch_bounds__(kBinThreads)
k_bin_apply(DevParams p) {
  pdl_wait();
  extern __shared__ uint32_t bin_rmax[];  // [2^bkt_log2]
  const uint32_t nb = 1u << p.bkt_log2;
  const uint32_t b = blockIdx.x;
  for (uint32_t j = threadIdx.x; j < nb; j += kBinThreads) bin_rmax[j] = 0u;
  __syncthreads();
  const uint32_t cnt = min(p.bcursor[b], p.bcap);
  const uint32_t *bin = p.bins + (uint64_t)b * p.bcap;
  constexpr int U = 4;
  uint32_t i = threadIdx.x;
  for (; i + (U - 1) * kBinThreads < cnt; i += U * kBinThreads) {
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = __ldcs(bin + i + u * kBinThreads);
#pragma unroll
    for (int u = 0; u < U; ++u) atomicMax(bin_rmax + (r[u] >> 5), r[u] & 31u);
  }
  for (; i < cnt; i += kBinThreads) {
    const uint32_t r = __ldcs(bin + i);
    atomicMax(bin_rmax + (r >> 5), r & 31u);
  }
  __syncthreads();
  const uint32_t tickbits = p.tick << 5;
  uint32_t *sr = p.sr + ((uint64_t)b << p.bkt_log2);
  for (uint32_t j0 = threadIdx.x; j0 < nb; j0 += U * kBinThreads) {
    uint32_t r[U], o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = j0 + u * kBinThreads;
      r[u] = j < nb ? bin_rmax[j] : 0u;
      o[u] = r[u] ? sr[j] : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = tickbits | r[u];
      if (r[u] != 0u && o[u] < v) sr[j0 + u * kBinThreads] = v;  // this CTA owns the words
    }
  }
  if (threadIdx.x == 0) p.bcursor[b] = 0u;  // the bin is empty for the next chunk
  pdl_trigger();
}
