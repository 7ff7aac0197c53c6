// k_plan.cu -- plan-based estimation for a fixed host list (sm_100a),
// compiled with -fmad=false like k_estimate.cu (same fp64 finish).
//
// The gather estimate (k_estimate.cu) is bound by the SM's L1-to-L2 request
// rate: one 32-byte sector request per 1-byte register read.  For pools whose
// register array is small (n_phys <= 2^22, 4 MiB) the same sums can be formed
// from shared memory instead:
//   * a PLAN, built once per host list, assigns every host to an accumulator
//     slot of one warp of one of P persistent CTAs, spreading hosts over
//     CTAs first, then warps, then lanes (host_of below), and lists, for
//     every (CTA, register block) phase and every warp, the warp's (host, i)
//     gathers that fall in that block (Alg.5 / Alg.3 indices, precomputed) as
//     ROUNDS of 32 entries (offset in block | accumulator byte offset << 16),
//     one entry per lane.  Any lane may serve any of its
//     warp's hosts, so all lanes stay busy (a thread-owns-its-hosts layout
//     idles ~35 % of the lanes on the longest run).  The entries of a group
//     are first striped over its rounds by shared-memory bank of their
//     register (k_plan_fill), then re-ordered so each round touches every
//     bank -- register side and accumulator side -- as few times as possible
//     (k_plan_sched);
//   * per slice, each CTA streams the register array through shared memory
//     one 64 KB block at a time (TMA bulk copies issued by a producer warp,
//     two stages, full / empty mbarriers, the next block's entries prefetched
//     into L2), together with its entries for that block, and every lane adds
//     2^(L - M) for M >= 1 (M for LogLog/PCSA) into the entry's u32
//     accumulator with a shared-memory atomic, or 2^L (1) into the host's
//     zero count for M = 0 (S = S' + V 2^L; S' <= g 2^(L-1) = 2^31 for
//     L = 32 - log2 g) -- no L2 gathers.  The last step is the fp64 finish
//     of k_estimate.
// (Splitting the grid into host groups x register ranges, so each CTA
// streams only part of the array, measured slower: the register stream is
// not the bound; tools/rejected/plan_ranges, profiles/r02_plan_ranges.txt.)
// Integer sums make the result bit-identical to the gather kernel.
#include "vbdr_dev.cuh"

using namespace vbdr_dev;
using vbdr_launch::EstParams;
using vbdr_launch::PlanLayout;

namespace {

#ifndef VBDR_PLAN_ILP
#define VBDR_PLAN_ILP 4  // rounds whose loads are issued before their atomics
#endif
#ifndef VBDR_PLAN_PREFETCH
#define VBDR_PLAN_PREFETCH 1  // phases ahead (0 = off; profiles/r01_plan_variants.txt)
#endif
#ifndef VBDR_PLAN_PREFETCH_TAB
#define VBDR_PLAN_PREFETCH_TAB 0
#endif
#ifndef VBDR_PLAN_SORT
#define VBDR_PLAN_SORT 0  // fill order: 0 register bank, 1 accumulator bank, 2 both (experiment)
#endif

#ifdef VBDR_PLAN_TRACE  // diagnostics build only (tools/plan_trace.py): per-CTA globaltimer stamps
// [cta][phase][0..3] = consumer warp 0: wait-full start, wait-full end, release;
// producer: wait-empty end (issue); [cta][64][0..3] = start, loop end (warp 0), finish end
__device__ unsigned long long g_plan_trace[148][65][4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PTRACE(ph, k) g_plan_trace[blockIdx.x % 148][(ph) < 64 ? (ph) : 64][k] = gtime()
#else
#define PTRACE(ph, k) ((void)0)
#endif

constexpr int kT = vbdr_launch::kPlanThreads;   // 512
constexpr int kW = kT / 32;                     // 16 warps
constexpr int kCap = vbdr_launch::kPlanEntCap;  // largest entries per (CTA, phase) buffer
constexpr int kStride = vbdr_launch::kPlanStride;  // round starts per key (kW + 1 used)
// per warp: `slots` host slots per lane + one trash word per lane (accw words)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---------------------------------------------------------------- build
struct BuildArgs {
  const uint32_t *hosts;
  uint64_t n;
  uint32_t g, A0, mask, block_log2;
  uint32_t phases;       // register blocks
  uint32_t P, slots;     // CTAs, accumulator slots per lane
  uint32_t *counts;      // [P * phases * kW * 32]: per (group, bank) counts, then cursors
  uint32_t *starts;      // [P * phases * kStride]: round offsets of the kW warps of a key
  uint32_t *range_base;  // [P * phases + 1], in entries
  uint32_t *entries;
  uint32_t *max_range;   // scalar
  uint32_t hpc;          // hosts per CTA, ceil(n / P)
};

// Host h -> CTA p = h / hpc, q = h % hpc -> lane q % 32, warp (q / 32) % 16,
// slot q / 512; the host's accumulator index in its warp is slot * 32 + lane.
// A warp's 32 lanes hold 32 consecutive hosts of one slot, so the finish of
// a slot writes 256 contiguous bytes.
__host__ __device__ __forceinline__ uint64_t host_of(uint32_t p, uint64_t q, uint32_t hpc) {
  return (uint64_t)p * hpc + q;
}

// (host, i) -> key = (CTA, phase), warp, bank of the register in the block,
// and the entry value (offset in block | accumulator index << 16).
__device__ __forceinline__ void locate_entry(const BuildArgs &a, uint64_t h, uint32_t i,
                                             uint64_t &key, uint32_t &warp, uint32_t &bank,
                                             uint32_t &val) {
  const uint32_t p = (uint32_t)(h / a.hpc);
  const uint64_t q = h % a.hpc;
  const uint32_t lane = (uint32_t)(q & 31u);
  warp = (uint32_t)((q >> 5) % kW);
  const uint32_t slot = (uint32_t)(q / kT);
  const uint32_t s1 = fmix32(i ^ a.A0);                            // Alg.3
  const uint32_t pidx = fmix32(__ldg(a.hosts + h) ^ s1) & a.mask;  // Alg.3
  const uint32_t blk = pidx >> a.block_log2;
  const uint32_t off = pidx & ((1u << a.block_log2) - 1u);
  key = (uint64_t)p * a.phases + blk;
#if VBDR_PLAN_SORT == 1
  bank = lane;  // accumulator bank
#elif VBDR_PLAN_SORT == 2
  bank = ((off >> 2) + lane) & 31u;
#else
  bank = (off >> 2) & 31u;  // register bank in the staged block
#endif
  val = off | ((slot * 32u + lane) << 18);  // accumulator byte offset << 16
}

__global__ void k_plan_count(BuildArgs a) {
  const uint64_t total = a.n * a.g;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    uint64_t key;
    uint32_t warp, bank, val;
    locate_entry(a, x / a.g, (uint32_t)(x % a.g), key, warp, bank, val);
    atomicAdd(a.counts + (key * kW + warp) * 32 + bank, 1u);
  }
}

// One block per key, thread (warp w, lane b) = group w's bank b: exclusive
// scan of the bank counts -> bank starts in the group's sorted order (the
// fill cursors); group sizes n_w -> R_w = ceil(n_w / 32) rounds; exclusive
// scan over the warps -> round offsets; the key's entries = 32 * sum R_w.
__global__ void __launch_bounds__(kT) k_plan_starts(BuildArgs a, uint32_t *range_size) {
  __shared__ uint32_t rounds[kW];
  const uint64_t key = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t *cnt = a.counts + key * kT + threadIdx.x;
  const uint32_t c = *cnt;
  uint32_t x = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= (uint32_t)off) x += y;
  }
  *cnt = x - c;  // cursor: sorted index of this bank's first entry
  if (lane == 31) rounds[w] = (x + 31u) >> 5;
  __syncthreads();
  if (w == 0) {
    const uint32_t r = lane < kW ? rounds[lane] : 0u;
    uint32_t v = r;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= (uint32_t)off) v += y;
    }
    if (lane <= kW) a.starts[key * kStride + lane] = v - r;  // lane kW: the key's total
    if (lane == kW) {
      range_size[key] = 32u * (v - r);
      atomicMax(a.max_range, 32u * (v - r));
    }
  }
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

// Entry with sorted index i of a group of R rounds -> round i % R, lane i / R.
__device__ __forceinline__ uint32_t stripe(uint32_t i, uint32_t R) {
  return (i % R) * 32u + i / R;
}

__global__ void k_plan_fill(BuildArgs a) {
  const uint64_t total = a.n * a.g;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    uint64_t key;
    uint32_t warp, bank, val;
    locate_entry(a, x / a.g, (uint32_t)(x % a.g), key, warp, bank, val);
    const uint32_t i = atomicAdd(a.counts + (key * kW + warp) * 32 + bank, 1u);
    const uint32_t r0 = a.starts[key * kStride + warp], R = a.starts[key * kStride + warp + 1] - r0;
    a.entries[a.range_base[key] + 32u * r0 + stripe(i, R)] = val;
  }
}

// One block per key, warp w pads group w: sorted indices [n_w, 32 R_w) get
// the lane's trash accumulator (offset 0 is a valid register to read).
__global__ void __launch_bounds__(kT) k_plan_pad(BuildArgs a) {
  const uint64_t key = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t n_w = a.counts[(key * kW + w) * 32 + 31];  // cursor of the last bank = n_w
  const uint32_t r0 = a.starts[key * kStride + w], R = a.starts[key * kStride + w + 1] - r0;
  for (uint32_t i = n_w + lane; i < 32u * R; i += 32u) {
    const uint32_t pos = stripe(i, R);
    a.entries[a.range_base[key] + 32u * r0 + pos] = (a.slots * 32u + (pos & 31u)) << 18;
  }
}

// One block per key, warp w re-orders group w's entries round by round so a
// round touches each shared-memory bank of the table (register offset) and of
// the accumulators (host lane) as few times as possible: round r takes
// ceil(remaining / rounds left) entries, first with at most one entry per
// bank on either side, then two, ... (greedy, warp-parallel: per 32-entry
// chunk the lowest lane of each bank wins).  Only the order changes, never
// the entries, so the sums are unchanged; it cuts bank-conflict wavefronts
// in k_estimate_plan.  Keys over the stage capacity are left alone (the
// plan is refused anyway).
// Lane j's entry of a round with `taken` real entries (lanes [0, taken)):
// the padding lanes read the register word of the round's first entry (a
// broadcast) and add into trash accumulators on the banks no real entry of
// the round uses, so padding never adds a bank conflict.
__device__ __forceinline__ uint32_t pad_round(uint32_t mine, uint32_t taken, uint32_t lane,
                                              uint32_t kTrash) {
  const bool real = lane < taken;
  const uint32_t used = __reduce_or_sync(0xffffffffu, real ? 1u << ((mine >> 18) & 31u) : 0u);
  const uint32_t off0 = __shfl_sync(0xffffffffu, mine, 0) & 0xFFFFu;
  if (real) return mine;
  const uint32_t bank = __fns(~used, 0, (int)(lane - taken) + 1);  // (lane - taken)-th free bank
  return (taken ? off0 : 0u) | ((kTrash + (bank & 31u)) << 18);
}

__global__ void __launch_bounds__(kT) k_plan_sched(BuildArgs a, const uint32_t *range_size) {
  __shared__ uint32_t E[kCap];        // the key's entries: per group the remaining list
  __shared__ uint32_t cnt[kW][64];    // per warp: table-bank [0, 32) and acc-bank [32, 64) use
  extern __shared__ uint8_t sched_dyn[];  // per warp: u8 loads [32 rounds][32 banks], two sides
  const uint64_t key = blockIdx.x;
  const uint32_t total = range_size[key];
  if (total > (uint32_t)kCap) return;
  const uint32_t lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
  uint32_t *ent = a.entries + a.range_base[key];
  for (uint32_t i = threadIdx.x; i < total; i += kT) E[i] = ent[i];
  __syncthreads();
  const uint32_t r0 = a.starts[key * kStride + w], R = a.starts[key * kStride + w + 1] - r0;
  uint32_t *L = E + 32u * r0;  // this warp's list
  uint32_t *out = ent + 32u * r0;
  const uint32_t kTrash = a.slots * 32u;  // accumulator indices >= this are padding
  constexpr uint32_t kTaken = 0xFFFFFFFFu;
  // drop the padding: compact the real entries to the front
  uint32_t rem = 0;
  for (uint32_t c = 0; c < 32u * R; c += 32u) {
    const uint32_t v = L[c + lane];
    const bool real = (v >> 18) < kTrash;
    const uint32_t m = __ballot_sync(0xffffffffu, real);
    __syncwarp();
    if (real) L[rem + __popc(m & ((1u << lane) - 1u))] = v;
    rem += __popc(m);
    __syncwarp();
  }
  if (R <= 32u) {
    // Best fit: each entry, in list order, goes to the round whose bank
    // maxima it raises least -- register side plus accumulator side, i.e. the
    // shared-memory wavefronts it adds to k_estimate_plan -- ties to the
    // emptiest round.  Lane r keeps round r's fill and maxima; the rounds'
    // per-bank loads live in shared memory.  (A round's base wavefront is
    // free: the maxima start at 1.)
    uint32_t *LRw = reinterpret_cast<uint32_t *>(sched_dyn + (size_t)w * 2048u);
    for (uint32_t i = lane; i < 512u; i += 32u) LRw[i] = 0u;
    uint8_t *LR = sched_dyn + (size_t)w * 2048u, *LA = LR + 1024u;
    __syncwarp();
    uint32_t fill = 0, mr = 1, ma = 1;
    for (uint32_t e = 0; e < rem; ++e) {
      const uint32_t v = L[e];
      const uint32_t tb = (v >> 2) & 31u, ab = (v >> 18) & 31u;
      uint32_t k = 0xFFFFFFFFu;
      if (lane < R && fill < 32u) {
        const uint32_t lr = LR[lane * 32u + tb] + 1u, la = LA[lane * 32u + ab] + 1u;
        const uint32_t inc = (lr > mr ? lr - mr : 0u) + (la > ma ? la - ma : 0u);
        k = (inc << 16) | (fill << 8) | lane;
      }
      const uint32_t bestr = __reduce_min_sync(0xffffffffu, k) & 0xFFu;
      if (lane == bestr) {
        out[32u * lane + fill] = v;
        const uint32_t lr = ++LR[lane * 32u + tb], la = ++LA[lane * 32u + ab];
        mr = max(mr, lr);
        ma = max(ma, la);
        ++fill;
      }
      __syncwarp();
    }
    for (uint32_t r = 0; r < R; ++r) {
      const uint32_t taken = __shfl_sync(0xffffffffu, fill, r);
      const uint32_t mine = lane < taken ? out[32u * r + lane] : 0u;
      __syncwarp();
      out[32u * r + lane] = pad_round(mine, taken, lane, kTrash);
    }
    return;
  }
  // more than 32 rounds (a few very full groups): round by round, greedy
  for (uint32_t r = 0; r < R; ++r) {
    const uint32_t target = min(32u, (rem + (R - r) - 1u) / (R - r));
    cnt[w][lane] = 0u;
    cnt[w][32 + lane] = 0u;
    __syncwarp();
    uint32_t taken = 0, mine = 0;  // lane j ends up holding the entry of round lane j
    for (uint32_t cap = 1; taken < target; ++cap) {
      for (uint32_t c = 0; c < rem && taken < target; c += 32u) {
        const uint32_t idx = c + lane;
        const uint32_t v = idx < rem ? L[idx] : kTaken;
        const uint32_t tb = (v >> 2) & 31u, ab = (v >> 18) & 31u;
        bool cand = v != kTaken && cnt[w][tb] < cap && cnt[w][32 + ab] < cap;
        const uint32_t cm = __ballot_sync(0xffffffffu, cand);
        // lowest candidate lane per table bank and per accumulator bank
        const uint32_t mt = __match_any_sync(0xffffffffu, cand ? tb : 64u + lane) & cm;
        const uint32_t ma = __match_any_sync(0xffffffffu, cand ? ab : 64u + lane) & cm;
        cand = cand && (mt & ((1u << lane) - 1u)) == 0u && (ma & ((1u << lane) - 1u)) == 0u;
        const uint32_t am = __ballot_sync(0xffffffffu, cand);
        const uint32_t rank = __popc(am & ((1u << lane) - 1u));
        const bool acc = cand && taken + rank < target;
        const uint32_t got = __ballot_sync(0xffffffffu, acc);
        if (acc) {
          cnt[w][tb] += 1u;
          cnt[w][32 + ab] += 1u;
          L[idx] = kTaken;
        }
        // hand each accepted entry to the lane of its round slot
#pragma unroll 1
        for (uint32_t m = got; m; m &= m - 1u) {
          const uint32_t src = __ffs(m) - 1u;
          const uint32_t val = __shfl_sync(0xffffffffu, v, src);
          if (lane == taken) mine = val;
          ++taken;
        }
        __syncwarp();
      }
    }
    out[32u * r + lane] = pad_round(mine, taken, lane, kTrash);
    // drop the taken entries from the list
    uint32_t n2 = 0;
    for (uint32_t c = 0; c < rem; c += 32u) {
      const uint32_t idx = c + lane;
      const uint32_t v = idx < rem ? L[idx] : kTaken;
      const bool keep = v != kTaken;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      __syncwarp();
      if (keep) L[n2 + __popc(m & ((1u << lane) - 1u))] = v;
      n2 += __popc(m);
      __syncwarp();
    }
    rem = n2;
  }
}

// --------------------------------------------------------------- estimate
__device__ __forceinline__ double hll_finish(double agg, double D, double lc, uint64_t V,
                                             double s, const double *lct = nullptr) {
  double E = __ddiv_rn(agg, D);
  // linear counting: s ln(s / V), from the plan's table of the same values
  // (k_plan_lct) when there is one -- bit-identical, without a log per host
  if (E <= lc && V > 0) E = __dmul_rn(s, lct ? __ldg(lct + V) : log(__ddiv_rn(s, (double)V)));
  return E;
}

// lct[V] = ln(g / V) for V = 1..g, computed exactly as hll_finish would
__global__ void k_plan_lct(double *lct, uint32_t g) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= g; v += gridDim.x * blockDim.x)
    lct[v] = v ? log(__ddiv_rn((double)g, (double)v)) : 0.0;
}

template <int BLOCK_LOG2>
struct __align__(128) PlanSmem {
  uint8_t tab[2][1 << BLOCK_LOG2];
  uint32_t ent[2][vbdr_launch::plan_ent_cap(BLOCK_LOG2)];
  uint32_t start[2][kStride];
  uint64_t full[2];          // TMA bytes of buffer b landed
  uint64_t empty[2];         // all kW consumer warps are done with buffer b
  double etot_z;
  uint32_t ok;               // cleared if a staged transfer never landed
  // followed by the accumulators, per warp 2 accw u32 (dynamic):
  // [0, accw) S' = sum over M >= 1 of 2^(L - M) (HLL) or M;
  // [accw, 2 accw) V, the number of M = 0 registers
};

__device__ __forceinline__ bool mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t spin = 0; !done; ++spin) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (spin > (1u << 26)) return false;  // a lost transfer must not hang the GPU
  }
  return true;
}

// The zero count V from the accumulators: HLL adds 2^L per zero register,
// so the word holds V 2^L mod 2^32, which wraps only for V = g when g 2^L =
// 2^32, i.e. every register zero -- exactly when S' = 0 (each M >= 1 adds >= 1).
__device__ __forceinline__ uint32_t plan_zero_count(uint32_t Sp, uint32_t Vz, bool HLL,
                                                    const EstParams &e) {
  return HLL ? (Sp == 0u ? e.g : Vz >> e.L) : Vz;
}

// One host's fp64 finish from its integer sums (k_estimate's operation order).
template <bool SUMS>
__device__ __forceinline__ void plan_finish(const EstParams &e, uint64_t h, uint32_t Sp, uint32_t V,
                                            bool HLL, double etot_z, double *out,
                                            unsigned long long *outS, uint32_t *outV,
                                            const double *lct) {
  const unsigned long long S = Sp + (HLL ? (unsigned long long)V << e.L : 0ull);
  if constexpr (SUMS) {
    outS[h] = S;
    outV[h] = V;
  } else {
    const double g = (double)e.g;
    double Es;
    if (e.est == 0u) {
      Es = hll_finish(e.agg, __dmul_rn((double)S, e.inv2L), e.lc_g, V, g, lct);
    } else {
      Es = __dmul_rn(e.coef_g, exp2(__ddiv_rn((double)S, g)));
    }
    // g is a power of two: Es / g is exact as Es * (1 / g)
    const double est = __dmul_rn(e.C, __dsub_rn(__dmul_rn(Es, __drcp_rn(g)), etot_z));
    out[h] = est > 0.0 ? est : 0.0;
  }
}

template <bool SUMS>
__device__ __forceinline__ void plan_poison(uint64_t h, double *out, unsigned long long *outS,
                                            uint32_t *outV) {
  if constexpr (SUMS) {  // loud: never a stale value from an earlier slice
    outS[h] = ~0ull;
    outV[h] = ~0u;
  } else {
    out[h] = __longlong_as_double(0x7FF8000000000000ll);  // NaN
  }
}

// kW consumer warps + one producer warp (TMA issue only).  Buffers are
// handed over with full / empty mbarriers, so a warp that finishes a block
// early starts on the next one instead of waiting at a CTA barrier.
template <int BLOCK_LOG2, bool SUMS, bool HLL>
__global__ void __launch_bounds__(kT + 32, 1)
k_estimate_plan(EstParams e, PlanLayout pl, uint64_t n, double *__restrict__ out,
                unsigned long long *__restrict__ outS, uint32_t *__restrict__ outV,
                unsigned long long *__restrict__ err) {
  constexpr uint32_t BLOCK = 1u << BLOCK_LOG2;
  constexpr int ILP = VBDR_PLAN_ILP;
  pdl_wait();
  extern __shared__ __align__(128) uint8_t raw[];
  PlanSmem<BLOCK_LOG2> &sm = *reinterpret_cast<PlanSmem<BLOCK_LOG2> *>(raw);
  const uint32_t accw = pl.st_slots * 32u + 32u;
  uint32_t *acc_all = reinterpret_cast<uint32_t *>(raw + sizeof(PlanSmem<BLOCK_LOG2>));
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t p = blockIdx.x;
  if (w < kW) {
    for (uint32_t i = lane; i < 2u * accw; i += 32u) acc_all[w * 2u * accw + i] = 0u;
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&sm.full[b])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(&sm.empty[b])), "r"(kW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    sm.ok = 1u;
  }
  __syncthreads();
  const uint32_t phases = pl.phases;
  const uint8_t *regs = e.regmax;
  if (tid == 0) PTRACE(64, 0);
  if (w == kW) {  // producer
    if (lane == 0) {
      for (uint32_t ph = 0; ph < phases; ++ph) {
        const int b = ph & 1;
        if (ph == (phases > 2u ? 2u : 0u) && !SUMS) {
          // the pool's own estimate E_tot / z for the noise subtraction, off the
          // first stages' critical path: the consumers read it in their finish,
          // after waiting on a stage this lane armed later (release / acquire)
          const unsigned long long St = e.acc[0], Vt = e.acc[1];
          double Et;
          if (e.est == 0u) {
            Et = hll_finish(e.azz, __dmul_rn((double)St, e.inv2L), e.lc_z, Vt, e.z);
          } else {
            Et = __dmul_rn(e.coef_z, exp2(__ddiv_rn((double)St, e.z)));
          }
          sm.etot_z = __ddiv_rn(Et, e.z);
        }
        // buffer b last held phase ph - 2: wait for its (ph/2 - 1)-th release
        if (ph >= 2 && !mbar_wait(&sm.empty[b], ((ph >> 1) + 1u) & 1u)) {
          atomicAdd(err, 1ull);
          break;
        }
        PTRACE(ph, 3);
        const uint64_t key = (uint64_t)p * phases + ph;
        const uint32_t e0 = pl.range_base[key], e1 = pl.range_base[key + 1];
        const uint32_t ebytes = (e1 - e0) * 4u;  // ranges are multiples of 32 entries
        const uint32_t sbytes = kStride * 4u;
        const uint32_t fb = smem_u32(&sm.full[b]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fb),
                     "r"(BLOCK + ebytes + sbytes)
                     : "memory");
        auto bulk = [&](void *dst, const void *src, uint32_t bytes) {
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
              "[%3];" ::"r"(smem_u32(dst)),
              "l"(src), "r"(bytes), "r"(fb)
              : "memory");
        };
        bulk(sm.tab[b], regs + (uint64_t)ph * BLOCK, BLOCK);
        if (ebytes) bulk(sm.ent[b], pl.entries + e0, ebytes);
        bulk(sm.start[b], pl.starts + key * kStride, sbytes);
#if VBDR_PLAN_PREFETCH
        // warm L2 with a later phase's entries (streamed from DRAM once): the
        // stage refill then waits on L2, not DRAM, latency
        const uint32_t pf = ph + VBDR_PLAN_PREFETCH;
        if (pf < phases) {
          const uint64_t k2 = (uint64_t)p * phases + pf;
          const uint32_t f0 = pl.range_base[k2], f1 = pl.range_base[k2 + 1];
          if (f1 > f0)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pl.entries + f0),
                         "r"((f1 - f0) * 4u)
                         : "memory");
#if VBDR_PLAN_PREFETCH_TAB
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(regs + (uint64_t)pf * BLOCK),
                       "r"(BLOCK)
                       : "memory");
#endif
        }
#endif
      }
    }
  } else {
    uint32_t *acc = acc_all + w * 2u * accw;
    const uint32_t acc_base = smem_u32(acc);
    const uint32_t vofs = 4u * accw;  // V array, same bank as the host's S'
    const uint32_t K = 1u << e.L;     // 2^(L - M) = K >> M
    for (uint32_t ph = 0; ph < phases; ++ph) {
      const int b = ph & 1;
      if (w == 0 && lane == 0) PTRACE(ph, 0);
      if (!mbar_wait(&sm.full[b], (ph >> 1) & 1u)) {
        if (lane == 0) {
          atomicAdd(err, 1ull);
          sm.ok = 0u;  // a staged transfer that never landed poisons the CTA's hosts (NaN)
        }
        break;
      }
      if (w == 0 && lane == 0) PTRACE(ph, 1);
      const uint8_t *tab = sm.tab[b];
      const uint32_t r0 = sm.start[b][w], r1 = sm.start[b][w + 1];
      const uint32_t *ent = sm.ent[b] + lane;
      // one entry per lane per round; ILP rounds' loads are issued before their
      // atomics.  One atomic per lane: M >= 1 adds its term to S', M = 0 adds
      // 1 to V
      auto add = [&](uint32_t v, uint32_t M) {
        // HLL: 2^(L - M) = K >> M for every M, the zero count included (it
        // holds V 2^L mod 2^32; plan_zero_count recovers V) -- one shift, no
        // select; LogLog / PCSA: M into S', 1 into the zero count
        const uint32_t cv = HLL ? K >> M : (M == 0u ? 1u : M);
        const uint32_t addr = acc_base + (v >> 16) + (M == 0u ? vofs : 0u);
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(cv) : "memory");
      };
      uint32_t r = r0;
      for (; r + ILP <= r1; r += ILP) {
        uint32_t v[ILP], M[ILP];
#pragma unroll
        for (int j = 0; j < ILP; ++j) v[j] = ent[(r + j) * 32u];
#pragma unroll
        for (int j = 0; j < ILP; ++j) M[j] = tab[v[j] & (BLOCK - 1u)];
#pragma unroll
        for (int j = 0; j < ILP; ++j) add(v[j], M[j]);
      }
      for (; r < r1; ++r) {
        const uint32_t v = ent[r * 32u];
        add(v, tab[v & (BLOCK - 1u)]);
      }
      __syncwarp();
      if (w == 0 && lane == 0) PTRACE(ph, 2);
      if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(smem_u32(&sm.empty[b])) : "memory");
    }
    if (w == 0 && lane == 0) PTRACE(64, 1);
    pdl_trigger();
    // this warp's hosts are final once its last block is done (only this
    // warp adds into them): finish them now, beside the other warps' last
    // rounds -- slot s holds hosts q = s 512 + w 32 + lane of this CTA
    const double etot_z = SUMS ? 0.0 : sm.etot_z;
    for (uint32_t ss = 0; ss < pl.st_slots; ++ss) {
      const uint32_t q = ss * (uint32_t)kT + (uint32_t)w * 32u + (uint32_t)lane;
      const uint64_t h = host_of(p, q, pl.st_hpc);
      if (q >= pl.st_hpc || h >= n) break;
      if (!sm.ok) {  // (a CTA that timed out still writes its hosts: NaN)
        plan_poison<SUMS>(h, out, outS, outV);
        continue;
      }
      plan_finish<SUMS>(e, h, acc[ss * 32u + lane],
                        plan_zero_count(acc[ss * 32u + lane], acc[accw + ss * 32u + lane], HLL, e),
                        HLL, etot_z, out,
                        outS, outV, pl.lct);
    }
#ifdef VBDR_PLAN_TRACE
    if (w == 0 && lane == 0) PTRACE(64, 2);
#endif
  }
}

template <int BL>
cudaError_t launch_est(const EstParams &e, const PlanLayout &pl, uint64_t n, double *out,
                       unsigned long long *outS, uint32_t *outV, cudaStream_t s) {
  const size_t smem = vbdr_launch::plan_smem_bytes(pl.block_log2, pl.st_slots);
  auto kern = outS ? (e.est == 0u ? k_estimate_plan<BL, true, true> : k_estimate_plan<BL, true, false>)
                   : (e.est == 0u ? k_estimate_plan<BL, false, true> : k_estimate_plan<BL, false, false>);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  return launch(kern, dim3(pl.ctas), dim3(kT + 32), smem, s, e, pl, n, out, outS, outV, pl.error);
}

}  // namespace

namespace vbdr_launch {

size_t plan_smem_bytes(uint32_t block_log2, uint32_t slots) {
  size_t fixed = 0;
  switch (block_log2) {
#define VBDR_PLAN_SMEM_CASE(BL) \
  case BL: fixed = sizeof(PlanSmem<BL>); break;
    VBDR_PLAN_SMEM_CASE(16) VBDR_PLAN_SMEM_CASE(15) VBDR_PLAN_SMEM_CASE(14)
    VBDR_PLAN_SMEM_CASE(13) VBDR_PLAN_SMEM_CASE(12) VBDR_PLAN_SMEM_CASE(11)
    VBDR_PLAN_SMEM_CASE(10) VBDR_PLAN_SMEM_CASE(9) VBDR_PLAN_SMEM_CASE(8)
    VBDR_PLAN_SMEM_CASE(7) VBDR_PLAN_SMEM_CASE(6)
#undef VBDR_PLAN_SMEM_CASE
    default: return 0;
  }
  return fixed + (size_t)kW * 2u * (slots * 32u + 32u) * 4u;
}

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
  a.P = pl.ctas;
  a.slots = pl.st_slots;
  a.hpc = pl.st_hpc;
  a.counts = pl.counts;
  a.starts = pl.starts;
  a.range_base = pl.range_base;
  a.entries = pl.entries;
  a.max_range = pl.max_range;
  const uint64_t nkeys = (uint64_t)pl.ctas * pl.phases;
  cudaError_t e = cudaMemsetAsync(pl.counts, 0, nkeys * kW * 32 * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pl.max_range, 0, 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pl.error, 0, 8, s);
  if (e != cudaSuccess) return e;
  const uint64_t total = n * g;
  const uint32_t grid = (uint32_t)((total + 255) / 256 < 148ull * 16 ? (total + 255) / 256 : 148ull * 16);
  k_plan_count<<<grid ? grid : 1, 256, 0, s>>>(a);
  k_plan_starts<<<(uint32_t)nkeys, kT, 0, s>>>(a, range_size_scratch);
  k_plan_bases<<<1, 1024, 0, s>>>(a, range_size_scratch, nkeys);
  k_plan_fill<<<grid ? grid : 1, 256, 0, s>>>(a);
  k_plan_pad<<<(uint32_t)nkeys, kT, 0, s>>>(a);
  e = cudaFuncSetAttribute(k_plan_sched, cudaFuncAttributeMaxDynamicSharedMemorySize, kW * 2048);
  if (e != cudaSuccess) return e;
  k_plan_sched<<<(uint32_t)nkeys, kT, kW * 2048, s>>>(a, range_size_scratch);
  if (pl.lct) k_plan_lct<<<(g + 256) / 256, 256, 0, s>>>(const_cast<double *>(pl.lct), g);
  return cudaGetLastError();
}

cudaError_t plan_lct(const double *lct, uint32_t g, cudaStream_t s) {
  k_plan_lct<<<(g + 256) / 256, 256, 0, s>>>(const_cast<double *>(lct), g);
  return cudaGetLastError();
}

#ifdef VBDR_PLAN_TRACE
}  // namespace vbdr_launch
extern "C" int vbdr_debug_plan_trace(unsigned long long *host, unsigned long long bytes) {
  return (int)cudaMemcpyFromSymbol(host, g_plan_trace, bytes < sizeof(g_plan_trace) ? bytes : sizeof(g_plan_trace));
}
namespace vbdr_launch {
#endif

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
