// vbdr_dev.cuh -- device-side building blocks of the VBDR hot path (sm_100a).
//
// Shared by the kernels of libvbdr.so only (never by oracle/).  Citations:
// PAPER.md:N = line of the paper text; R#n = DESIGN.md section 3 reading.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vbdr_dev {

// Parameters every kernel receives by value.
struct DevParams {
  uint32_t *sr;              // u32[n_phys] stamp words (layout F)
  uint32_t *drv;             // u32[W][drv_n] packed DRV of BDRs [drv_j0, drv_j0 + drv_n), plane-major
  uint8_t *regmax;           // u8[n_phys] register values M[j]: the buffer the next slide writes
  unsigned long long *acc;   // u64[8]: (S_tot, V_tot) per tick mod 4
  uint64_t n_phys;
  uint64_t drv_j0, drv_n;    // the DRV shard (0, n_phys unless register-sharded)
  uint32_t mask;             // n_phys - 1 (n_phys <= 2^32)
  uint32_t b, L, k, zb, F, W;
  uint32_t A0, A1;
  uint32_t tick;             // T of the open slice
  uint32_t est;              // register estimator: 0 HLL, 1 LogLog, 2 PCSA (packed only)
};

// H(x, 2^32, A) = fmix32(x ^ A) (R#6: MurmurHash3 finaliser).
__device__ __forceinline__ uint32_t fmix32(uint32_t t) {
  t ^= t >> 16;
  t *= 0x85EBCA6Bu;
  t ^= t >> 13;
  t *= 0xC2B2AE35u;
  t ^= t >> 16;
  return t;
}

// Alg.4 lines 180-184 for one pair, in registers:
//   bip' = H(bip, 2^32, A1); vidx = LB(bip', b); w = bip' << b;
//   rho  = LBP1(w) = min(clz(w) + 1, L)          (R#4, R#5)
//   pidx = getPhyIdx(aip, vidx, A0) = H(aip, z, H(vidx, 2^32, A0))  (Alg.3)
__device__ __forceinline__ void pair_index(uint32_t aip, uint32_t bip, const DevParams &p,
                                           uint32_t &pidx, uint32_t &rho) {
  const uint32_t bp = fmix32(bip ^ p.A1);
  const uint32_t vidx = bp >> (32u - p.b);
  const uint32_t w = bp << p.b;
  rho = min((uint32_t)__clz(w) + 1u, p.L);
  const uint32_t s1 = fmix32(vidx ^ p.A0);
  pidx = fmix32(aip ^ s1) & p.mask;
}

// SWAR over one 32-bit word of F = 32/ZB packed DRs (field f = bits
// [ZB f, ZB f + ZB)).  Unused high bits are kept zero.
template <int ZB>
struct Swar {
  static constexpr int F = 32 / ZB;
  static constexpr uint32_t FM = (1u << ZB) - 1u;  // one field, all ones = sentinel S
  static constexpr uint32_t lsb_of(int parity) {   // parity: 0 even, 1 odd, 2 all
    uint32_t m = 0;
    for (int f = 0; f < F; ++f)
      if (parity == 2 || (f & 1) == parity) m |= 1u << (ZB * f);
    return m;
  }
  static constexpr uint32_t LSB = lsb_of(2);
  static constexpr uint32_t LSB_EVEN = lsb_of(0);
  static constexpr uint32_t CARRY = LSB_EVEN << ZB;  // carry-out bit of each even slot
  static constexpr uint32_t EVEN = LSB_EVEN * FM;  // fields 0, 2, 4, ...
  static constexpr uint32_t INIT = LSB * FM;        // InitDR on every field

  // SlideDR on every field (R#1: saturating at S = 2^ZB - 1).
  __device__ static __forceinline__ uint32_t age(uint32_t x) {
    uint32_t t = x;
#pragma unroll
    for (int i = 1; i < ZB; ++i) t &= x >> i;  // bit ZB f = AND of field f's bits
    return x + (LSB & ~t);                     // +1 where the field is not S
  }

  // IsActiveDR (dr < k) on every field: returns bit ZB f set iff
  // field f < k.  addk = (2^ZB - k) at every even field's LSB; a field >= k
  // carries into the (zeroed) neighbour above it.
  __device__ static __forceinline__ uint32_t active(uint32_t x, uint32_t addk) {
    const uint32_t ce = ((x & EVEN) + addk) & CARRY;          // even field f -> bit ZB(f+1)
    const uint32_t co = (((x >> ZB) & EVEN) + addk) & CARRY;  // odd field f  -> bit ZB f
    const uint32_t inactive = (ce >> ZB) | co;  // bit ZB f; a phantom field F is masked off
    return ~inactive & LSB;
  }

  // Highest active field of a non-zero mask from active().
  __device__ static __forceinline__ uint32_t top_field(uint32_t a) {
    return (31u - (uint32_t)__clz(a)) / (uint32_t)ZB;
  }
};

// Max useful words per BDR for a field width (L <= 31 ranks).
template <int ZB>
struct WMax {
  static constexpr int value = (31 + Swar<ZB>::F - 1) / Swar<ZB>::F;
};

// Programmatic dependent launch (PDL): hot-path kernels are launched with
// programmatic stream serialization, so a kernel's launch and block
// scheduling overlap the drain of its predecessor on the stream.  Every such
// kernel calls pdl_wait() before its first global-memory access, which blocks
// until the predecessor grid has completed and its writes are visible -- the
// same ordering as a plain launch, minus the launch gap.
// The device side is always compiled in (griddepcontrol.wait is a no-op in a
// grid launched without the attribute); whether a launch sets the attribute
// is decided at run time (pdl_mode below, env VBDR_PDL: 0 off, 1 every
// launch, unset = every launch except the gather estimate, where early
// dependent CTAs unbalance the persistent grid: profiles/r01_pdl.txt).
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// 0 off, 1 on for every launch, 2 (default) on except the gather estimate
int pdl_mode();

template <typename... KArgs, typename... Args>
cudaError_t launch_ex(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args... args) {
  return launch_ex(pdl_mode() != 0, kern, grid, block, smem, s, args...);
}

}  // namespace vbdr_dev

// Launchers implemented in the .cu files (host side, return cudaError_t).
namespace vbdr_launch {
using vbdr_dev::DevParams;

// Peer pointers for the fused merge + slide (vbdr_slide_peers).
constexpr int kMaxPeers = 16;
struct Peers {
  const uint8_t *delta[kMaxPeers];       // every rank's u8[n_phys] delta
  uint8_t *regmax[kMaxPeers];            // every rank's regmax, or n_regmax = 0
  unsigned long long *acc[kMaxPeers];    // every rank's accumulator base, or n_acc = 0
  uint32_t n, n_regmax, n_acc;
  // NVLS (vbdr_slide_multicast): multicast addresses of the state regions;
  // nvls = 1 selects the multicast slide (then the arrays above are unused);
  // 2 = the same for a group of one, through ordinary addresses
  uint32_t nvls;
  const uint32_t *sr_mc;                 // stamps (layout fast)
  uint32_t *drv_mc;                      // packed DRV planes (layout packed)
  uint8_t *regmax_mc;                    // the register buffer the slide writes
  unsigned long long *acc_mc;            // accumulator base
};
cudaError_t init(const DevParams &p, bool fast, cudaStream_t s);
cudaError_t scan(const DevParams &p, bool fast, int mode, const uint32_t *pairs, uint64_t n,
                 cudaStream_t s);
cudaError_t slide(const DevParams &p, bool fast, cudaStream_t s);
// layout S (per-(BDR, rank) stamps in the drv region, L planes)
cudaError_t scan_stamps(const DevParams &p, int mode, const uint32_t *pairs, uint64_t n,
                        cudaStream_t s);
cudaError_t slide_stamps(const DevParams &p, cudaStream_t s);
cudaError_t slide_delta(const DevParams &p, const uint8_t *delta, uint64_t j0, uint64_t j1,
                        cudaStream_t s);
cudaError_t delta(const DevParams &p, uint8_t *out, cudaStream_t s);
cudaError_t slide_peers(const DevParams &p, const Peers &peers, uint64_t j0, uint64_t j1,
                        cudaStream_t s);
cudaError_t slide_multicast(const DevParams &p, const Peers &mc, uint64_t j0, uint64_t j1,
                            bool fast, cudaStream_t s);
cudaError_t gather_words(const DevParams &p, const uint64_t *idx, uint64_t n, uint32_t *out,
                         cudaStream_t s);

struct EstParams {
  const uint8_t *regmax;
  const unsigned long long *acc;  // (S_tot, V_tot) of the closed tick
  uint32_t mask, A0, L, g;
  uint32_t lanes;     // lanes per host (0 = default)
  uint32_t pass_log2; // physical range per pass = 2^pass_log2 BDRs (>= log2(n_phys): one pass)
  double inv2L;       // 2^-L
  double agg;         // alpha_g * g * g
  double lc_g;        // 2.5 * g
  double azz;         // alpha_z * z * z
  double lc_z;        // 2.5 * z
  double z;           // n_phys as double
  double C;           // z g / (z - g)
  uint32_t est;       // 0 HLL, 1 LogLog, 2 PCSA
  double coef_g;      // LogLog alpha_g g, PCSA g / phi
  double coef_z;      // same for the pool of z registers
};
// Plan-based estimate (k_plan.cu): a host list preprocessed into per-(CTA,
// register block, warp) rounds of 32 entries.  Layout of the caller's plan buffer.
constexpr int kPlanThreads = 512;
constexpr int kPlanEntCap = 8192; // entries per (CTA, block) staged in shared memory, 2^16 blocks
// entry stage capacity (entries per (CTA, block) stage), every block size
constexpr uint32_t plan_ent_cap(uint32_t) { return (uint32_t)kPlanEntCap; }
constexpr int kPlanStride = 20;   // round starts per (CTA, block): 16 warps + total, 16-byte padded
// Sorted plan (k_splan.cu): entries sorted by register line, P host groups x
// C register ranges, one CTA per SM.
constexpr int kSpThreads = 1024;
constexpr uint32_t kSpLineLog2 = 7;  // bucket = one 128-byte line of registers
#ifndef VBDR_SP_UNROLL
#define VBDR_SP_UNROLL 8
#endif
constexpr int kSpUnroll = VBDR_SP_UNROLL;
#ifndef VBDR_SP_PREFETCH
#define VBDR_SP_PREFETCH 64 // rounds ahead to bulk-prefetch into L2 (0 = off)
#endif
struct PlanLayout {
  uint32_t kind;         // 0: shared-memory staged rounds (k_plan.cu); 1: pass ids; 2: sorted (k_splan.cu)
  uint32_t ctas, phases, block_log2;
  uint64_t n_hosts;
  uint32_t *hosts;       // kind 1: a copy of the host list
  void *pid;             // kind 1: pass ids
  uint32_t passes;       // kind 1
  uint32_t *range_base;  // [ctas * phases + 1], entries
  uint32_t *starts;      // [ctas * phases * kPlanStride], rounds
  uint32_t *counts;      // [ctas * phases * kPlanThreads] (build scratch: per (warp, bank))
  uint32_t *range_size;  // [ctas * phases] (build scratch)
  uint32_t *entries;
  uint32_t *max_range;   // build: largest (CTA, block) entry count
  unsigned long long *error;  // estimate: set if a staged transfer never landed
  const double *lct;     // kinds 0, 2: ln(g / V) for V = 0..g (linear counting), or null
  uint32_t st_slots;     // kind 0: accumulator slots per lane (hosts per thread)
  uint32_t st_hpc;       // kind 0: hosts per CTA (host h -> CTA h / st_hpc)
  // kind 2 (sorted plan); counts = bucket cursors, range_size = segment totals
  uint32_t sp_C;           // register ranges per host group
  uint32_t sp_hpg;         // accumulator slots per group (hosts / P, rounded up)
  uint32_t sp_nseg;        // segments per CTA range
  uint32_t sp_SB;          // slot bits of an entry
  uint32_t sp_seg_log2;    // registers per segment = 2^sp_seg_log2
  uint32_t sp_range_log2;  // registers per CTA range = z / C
  uint32_t *sp_segbase;    // [ctas * nseg + 1] first entry of each segment
  unsigned long long *sp_part;  // [ctas * hpg] partial (S', V) (C > 1)
  uint32_t *sp_gcount;     // [P] arrivals per group (C > 1)
};
size_t plan_smem_bytes(uint32_t block_log2, uint32_t slots);  // 0: unsupported block
cudaError_t plan_lct(const double *lct, uint32_t g, cudaStream_t s);  // fill a plan's log table
cudaError_t plan_build(const PlanLayout &pl, const uint32_t *hosts, uint64_t n, uint32_t g,
                       uint32_t A0, uint32_t mask, uint32_t *range_size_scratch, cudaStream_t s);
cudaError_t estimate_plan(const EstParams &e, const PlanLayout &pl, uint64_t n, double *out,
                          unsigned long long *outS, uint32_t *outV, cudaStream_t s);

size_t sp_smem_bytes(uint32_t hpg, uint32_t nseg);
// count + segment scan + segment bases (total entries incl. padding -> *d_total), then fill
cudaError_t sp_build(const PlanLayout &pl, const uint32_t *hosts, uint64_t n, uint32_t g,
                     uint32_t A0, uint32_t mask, unsigned long long *d_total, cudaStream_t s);
cudaError_t sp_fill(const PlanLayout &pl, const uint32_t *hosts, uint64_t n, uint32_t g,
                    uint32_t A0, uint32_t mask, cudaStream_t s);
cudaError_t estimate_sp(const EstParams &e, const PlanLayout &pl, uint64_t n, double *out,
                        unsigned long long *outS, uint32_t *outV, cudaStream_t s);

// Pass-id plan for multi-pass gather estimates (k_estimate.cu): 2 bits per
// (host, i), 16 bytes per (host, lane), g / 64 lanes per host.
uint32_t passplan_lanes(uint32_t g);
cudaError_t passplan_build(const uint32_t *hosts, uint64_t n, uint32_t g, uint32_t A0,
                           uint32_t mask, uint32_t pass_log2, void *pid, cudaStream_t s);
cudaError_t estimate_passplan(const EstParams &e, const uint32_t *hosts, uint64_t n,
                              const void *pid, uint32_t passes, double *out,
                              unsigned long long *outS, uint32_t *outV, cudaStream_t s);

// Sparse exchange (k_scan_slide.cu): touched BDRs as per-owner records, and
// their per-byte max into an owner's delta shard.
cudaError_t sparse_extract(const DevParams &p, uint32_t owners, uint32_t *records, uint64_t cap,
                           unsigned long long *counts, cudaStream_t s);
cudaError_t sparse_apply(const uint32_t *records, uint64_t n, uint8_t *delta, cudaStream_t s);

cudaError_t select_above(const double *est, uint64_t n, double threshold, uint32_t *idx,
                         unsigned long long *count, cudaStream_t s);

// *nl receives the number of kernels launched (passes).
cudaError_t estimate(const EstParams &e, const uint32_t *hosts, uint64_t n, double *out,
                     unsigned long long *outS, uint32_t *outV, cudaStream_t s, uint32_t *nl);
}  // namespace vbdr_launch
