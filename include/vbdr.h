/*
 * vbdr.h -- C ABI of the B200-native VBDR hot path (libvbdr.so).
 *
 * VBDR: Jie Xu, "Cardinalities estimation under sliding time window by sharing
 * HyperLogLog Counter", arXiv 1810.13132.  Citations "PAPER.md:N" are lines of
 * the paper text; "R#n" rows of the reading ledger in DESIGN.md section 3.
 *
 * One slice of the method is
 *     vbdr_scan_slice (any number of times)  -> [merge, N > 1] -> vbdr_slide
 *     -> vbdr_estimate (any number of times)
 *
 * Conventions (all entry points):
 *  - Pointers prefixed d_ are device pointers, h_ host pointers.  The CALLER
 *    owns all device memory (the state buffer, pair batches, host lists,
 *    outputs) and keeps it alive until the stream work that uses it is done;
 *    the library stores only pointers and the configuration.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls are stream-ordered and asynchronous unless marked SYNC.
 *  - Argument errors are reported synchronously (VBDR_EINVAL / VBDR_ERANGE /
 *    VBDR_ESTATE) before anything is launched; a CUDA error (including an
 *    asynchronous fault from earlier work) is returned as VBDR_ECUDA.  The
 *    text of the last error of a handle is vbdr_last_error(h).
 *  - One handle per device and host thread; a handle is not thread-safe.
 *  - IP addresses are host-order u32 (a.b.c.d -> a<<24|b<<16|c<<8|d, R#21).
 */
#ifndef VBDR_H
#define VBDR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vbdr vbdr_t; /* opaque handle */

typedef enum {
    VBDR_OK = 0,
    VBDR_EINVAL = -1, /* bad argument or configuration                       */
    VBDR_ERANGE = -2, /* size out of the supported range                     */
    VBDR_ESTATE = -3, /* call not valid in the handle's current state        */
    VBDR_ENOMEM = -4, /* state buffer too small / host allocation failed     */
    VBDR_ECUDA = -5   /* CUDA runtime error (text in vbdr_last_error)        */
} vbdr_status;

typedef enum {
    /* Stamp word sr[j] = (T << 5) | max rank of the open slice (the paper's
     * nowLBP1, made race-free with atomicMax)
     * plus the packed DRV.  VBDR-serial / VBDR-gfast semantics (Alg.1/4 and
     * Alg.6/7): one rank recorded per register-slice. */
    VBDR_LAYOUT_FAST = 0,
    /* Packed DRV only, every rank recorded with atomicAnd (Alg.9)
     * and aged at the slide (Alg.8 hoisted).  VBDR-gsmall
     * semantics, the memory-efficient variant (Table 1). */
    VBDR_LAYOUT_PACKED = 1,
    /* Layout S: a u32 last-seen stamp per (BDR, rank) -- the literal "stamps"
     * reading of the north star, with VBDR-gsmall semantics: the scan records
     * every pair's rank (as Alg.9's SetDR) with
     * atomicMax(stamp[rho-1][pidx], T); nothing is aged, a DR's age is
     * T - stamp at readout (IsActiveDR).  32 L bits per BDR: a
     * comparison point for the two packed layouts.  Single
     * GPU or the "stamps" merge (allreduce MAX of all stamps); scan_mode 2 or
     * 5 (5 only while L * n_phys < 2^32).  Ages export as T - stamp (0xFFFF
     * never recorded; canonical: min(age, k)). */
    VBDR_LAYOUT_STAMPS = 2
} vbdr_layout;

typedef struct {
    /* m: virtual BDRs per host -- the paper's g = 2^b.  Power of
     * two, 2 <= m, 2*m <= n_phys (R#15), n_phys * 2^L <= 2^53 (exact sums;
     * with the default L = 32 - log2(m): n_phys / m <= 2^21). */
    uint32_t m;
    /* k: window length in slices, W(t,k).  1 <= k. */
    uint32_t k;
    /* n_phys: physical BDRs in the shared pool BDRP -- the paper's z
     * (PAPER.md:152, 164).  Power of two, 4 <= n_phys <= 2^32. */
    uint64_t n_phys;
    /* seed_a0 / seed_a1: the paper's A0 (physical index, Alg.3)
     * and A1 (opposite host, Alg.4).  Defaults (R#7):
     * 0x5EED0001 / 0x5EED0002 when both are 0. */
    uint32_t seed_a0;
    uint32_t seed_a1;
    /* zbits: DR width z.  0 = ceil(log2(k+1)), plus one for
     * VBDR_LAYOUT_PACKED when k = 2^zbits - 1 (R#2).  Explicit values must
     * satisfy 2^zbits - 1 >= k (packed: 2^zbits - 2 >= k); 1 <= zbits <= 10. */
    uint32_t zbits;
    /* rank_cap: L, the number of ranks per BDR (R#3).  0 = 32 - log2(m);
     * otherwise 1 <= rank_cap <= 32 - log2(m). */
    uint32_t rank_cap;
    /* layout: vbdr_layout. */
    uint32_t layout;
    /* scan_mode: 0 = default (5 for layout fast, 2 for packed); 2 = L2
     * load-check, skip the atomic when the stored value already dominates;
     * 5 = a per-block shared-memory cache of recently updated words in front
     * of the mode-2 check.  Other values: VBDR_EINVAL.  Both modes give
     * bit-identical state (stored values only move one way within a slice). */
    uint32_t scan_mode;
    /* est_lanes: lanes cooperating on one host in vbdr_estimate (1, 2, 4, 8,
     * 16 or 32; 0 = auto).  Tuning only; results are identical. */
    uint32_t est_lanes;
    /* est_pass_log2: vbdr_estimate gathers from physical ranges of
     * 2^est_pass_log2 registers, one kernel pass per range, so each pass's
     * slice of the register array stays L2-resident (0 = auto: 26, i.e. one
     * pass up to 2^26 BDRs).  Tuning only; results are identical. */
    uint32_t est_pass_log2;
    /* estimator: the register estimator the BDR pool feeds (PAPER.md:214, 319:
     * "BDRP could also be used in PCSA, LogLog"): 0 = HyperLogLog (default,
     * R#15); 1 = LogLog, alpha_g g 2^(sum M / g), on Alg.5's getSumLBP1;
     * 2 = PCSA, (g / 0.77351) 2^(sum R / g) with R = the number of active
     * ranks counted up from rank 1 (the sliding Flajolet-Martin bitmap) --
     * layout packed only, since only gsmall records every rank.  All three use
     * the shared-pool noise subtraction of R#15.  With PCSA the register array
     * (vbdr_export_regmax) holds R; the pool sums are sum R (LogLog: sum M)
     * and the zero count. */
    uint32_t estimator;
    /* drv_shards / drv_shard: register-sharded state (layout
     * fast only).  With drv_shards = N > 1 the handle stores the packed DRV
     * of BDRs [r S, (r + 1) S) only (r = drv_shard, S = n_phys / N, a
     * multiple of 4), so DRV memory is /N; stamps and registers stay
     * full-size (every rank scans anywhere and estimates from all registers).
     * Such a handle closes slices only with vbdr_slide_delta /
     * vbdr_slide_peers over its own shard (vbdr_slide and vbdr_export_ages
     * return VBDR_ESTATE; vbdr_export_ages_at reads zeros outside the shard).
     * 0 or 1 = unsharded. */
    uint32_t drv_shards;
    uint32_t drv_shard;
} vbdr_config;

/* Derived sizes and the layout of the state buffer (byte offsets from the
 * d_state pointer passed to vbdr_create). */
typedef struct {
    uint32_t b;            /* log2(m)                                         */
    uint32_t L;            /* ranks per BDR                                   */
    uint32_t zbits;        /* DR width in bits                                */
    uint32_t fields;       /* F = floor(32 / zbits) DRs per 32-bit word       */
    uint32_t words;        /* W = ceil(L / F) words per BDR                   */
    uint32_t tick;         /* T = t + 1 of the open slice t                   */
    uint64_t n_phys;
    uint64_t slices_closed;/* number of vbdr_slide calls so far               */
    uint64_t off_acc;      /* u64[8]: (S_tot, V_tot) for tick mod 4 = 0..3    */
    uint64_t off_sr;       /* u32[n_phys] stamp words (LAYOUT_FAST only)      */
    uint64_t off_drv;      /* u32[W][n_phys] packed DRV, plane-major          */
    uint64_t off_regmax;   /* u8[n_phys] register values M[j] (Alg.2) of the
                            * closed tick (two buffers alternate by tick parity) */
    uint64_t state_bytes;  /* total bytes the state buffer needs              */
    uint64_t launches;     /* kernels launched by this handle so far          */
    uint64_t off_regmax_next; /* the register buffer the next slide writes     */
} vbdr_info_t;

/* SYNC.  Bytes of device memory the caller must provide for this config. */
vbdr_status vbdr_state_bytes(const vbdr_config *cfg, uint64_t *bytes);

/* SYNC, host only.  NULL if cfg is valid, else why not (thread-local text,
 * valid until the next call on this thread). */
const char *vbdr_config_check(const vbdr_config *cfg);

/* Validate cfg, bind the caller's state buffer (d_state, >= state_bytes,
 * 256-byte aligned) and initialise it on `stream`: every DR to InitDR = 2^z-1
 * (PAPER.md:94), stamps and registers to 0.  Slice t = 0 is open.
 * *out receives the handle (host memory owned by the library). */
vbdr_status vbdr_create(const vbdr_config *cfg, void *d_state, uint64_t bytes,
                        void *stream, vbdr_t **out);

/* Frees the handle and its streams/events; does not free d_state. */
vbdr_status vbdr_destroy(vbdr_t *h);

/* Scan n_pairs IP pairs of the open slice (Alg.4 lines 179-185 / Alg.9,
 * PAPER.md:179-185, 288-292).  d_pairs is u32[2*n_pairs], interleaved
 * (aip, bip), 16-byte aligned.  n_pairs = 0 is legal.  May be called any
 * number of times per slice; the resulting state does not depend on the order
 * or split of the pairs. */
vbdr_status vbdr_scan_slice(vbdr_t *h, const uint32_t *d_pairs, uint64_t n_pairs,
                            void *stream);

/* Close the open slice t: age every DR, expire ranks older
 * than k, record this slice's ranks (Alg.1 / Alg.8), materialise the register
 * values M[j] = GetLBP1BDR (Alg.2) and the pool sums
 * S_tot = sum_j 2^(L - M[j]) and V_tot = #{M[j] = 0}.  Opens slice t+1.
 * Multi-GPU: the caller merges the stamp arrays of all ranks (elementwise
 * max over sr, see vbdr_info) BEFORE this call. */
vbdr_status vbdr_slide(vbdr_t *h, void *stream);

/* ---- multi-GPU merge (layout fast) ----------------------------------- */

/* Compact the open slice's stamps to one byte per BDR (d_delta, u8[n_phys],
 * 16-byte aligned): the slice's max rank rho at BDR j, or 0 -- the paper's
 * nowLBP1.  The elementwise MAX of the ranks' deltas
 * (NCCL allreduce / reduce-scatter on uint8) is the whole slice's nowLBP1,
 * because max is commutative and idempotent.  VBDR_ESTATE on layout packed. */
vbdr_status vbdr_stamp_delta(vbdr_t *h, uint8_t *d_delta, void *stream);

/* vbdr_slide driven by a MERGED delta instead of the local stamps, over the
 * BDR range [j0, j1) only (multiples of 4; d_delta[j - j0] is BDR j's rank).
 * With [0, n_phys) every rank slides its full replica; with a shard per rank
 * the ranks then all-gather regmax (vbdr_info off_regmax) and all-reduce (SUM)
 * the pool sums of the closed tick (the two u64 at off_acc + 16 * (T mod 4),
 * T = the closed tick) before estimating.  DRs outside [j0, j1) are not aged
 * and must not be used afterwards.  Closes the slice like vbdr_slide. */
vbdr_status vbdr_slide_delta(vbdr_t *h, const uint8_t *d_delta, uint64_t j0, uint64_t j1,
                             void *stream);

/* Sparse exchange for pools far sparser than a slice (SURVEY 8(e) iii): list
 * the BDRs this rank's pairs touched in the open slice, per OWNER rank o of
 * n_owners equal BDR shards [o S, (o + 1) S), S = n_phys / n_owners (a
 * multiple of 4, <= 2^27), as u32 records ((j - o S) << 5) | rho into
 * d_records[o * cap .. o * cap + count_o), and count_o into d_counts[o]
 * (u64[n_owners]; counts are exact even when they exceed cap, in which case
 * only the first cap records of that owner are written -- call again with a
 * larger cap).  Record order within an owner is unspecified.  The caller
 * exchanges the lists (e.g. all-to-all) and every owner folds the records it
 * received into its delta shard with vbdr_sparse_apply, then closes the slice
 * with vbdr_slide_delta over its shard.  VBDR_ESTATE on layout packed. */
vbdr_status vbdr_sparse_extract(vbdr_t *h, uint32_t n_owners, uint32_t *d_records, uint64_t cap,
                                uint64_t *d_counts, void *stream);

/* d_delta_shard[j] = max(d_delta_shard[j], rho) for every record (j << 5) |
 * rho of d_records (u32[n_records], any order, any number of ranks); the
 * caller zeroes the shard first.  A per-byte max, so the result is the
 * merged nowLBP1 of the shard whatever the record order. */
vbdr_status vbdr_sparse_apply(vbdr_t *h, const uint32_t *d_records, uint64_t n_records,
                              uint8_t *d_delta_shard, void *stream);

/* Fused merge + slide over peer memory (the B200 path: no collective kernel).
 * h_peer_delta is a HOST array of n_peers (1..16) device pointers, one per
 * rank, each to that rank's u8[n_phys] delta from vbdr_stamp_delta -- local or
 * mapped over NVLink (CUDA IPC / symmetric memory).  The kernel merges the
 * deltas of BDRs [j0, j1) with a per-byte max while sliding them.  If
 * h_peer_regmax is given -- n_peers pointers to the register buffer every
 * rank's NEXT slide writes, i.e. base + vbdr_info off_regmax_next read BEFORE
 * this call (the two register buffers alternate with the tick; off_regmax is
 * the closed tick's buffer and is wrong here) -- the register shard is written
 * into every rank's buffer instead of only the local one; VBDR_EINVAL if no
 * entry equals this handle's own next buffer.  If h_peer_acc (n_peers pointers to
 * every rank's accumulator base, vbdr_info off_acc) is given, the shard's pool
 * sums are added atomically into every rank (own rank included in both
 * lists).  The caller orders it between two cross-rank barriers: after every
 * rank's vbdr_stamp_delta, and before any rank's vbdr_estimate.  Closes the
 * slice like vbdr_slide. */
vbdr_status vbdr_slide_peers(vbdr_t *h, const uint8_t *const *h_peer_delta, uint32_t n_peers,
                             uint64_t j0, uint64_t j1, uint8_t *const *h_peer_regmax,
                             uint64_t *const *h_peer_acc, void *stream);

/* Fused NVLS merge + slide, both layouts.  d_mc_state is
 * the MULTICAST address of a multicast object to which every rank bound its
 * state buffer (each laid out by vbdr_create with the same config; e.g. torch
 * symmetric memory's multicast_ptr, or vbdr_mc_alloc for one device).  The
 * kernel closes the slice for BDRs [j0, j1) (multiples of 4; the rank's
 * shard) with the merge done by the NVSwitch as it loads:
 *  - layout fast: multimem.ld_reduce MAX of every rank's stamp words -- the
 *    serial max of Alg.4 is commutative and idempotent, so the
 *    reduced stamp is the whole slice's nowLBP1 -- then Alg.1 and Alg.2 on
 *    the local DRV shard ([j0, j1) must lie in this handle's DRV shard);
 *  - layout packed: multimem.ld_reduce AND of every rank's copy of the DRV
 *    words -- each rank's scan cleared fields of its own copy (Alg.9 SetDR,
 *    PAPER.md:292; clears commute), so the AND holds every
 *    clear of the slice -- then Alg.2 and Alg.8, and the new words are
 *    stored into every rank's copy (multimem.st); needs drv_shards <= 1.
 * The registers of [j0, j1) are stored into every rank's register buffer
 * (multimem.st) and the shard's pool sums added into every rank's
 * accumulator (multimem.red).  The caller orders it between two cross-rank
 * barriers: after every rank's scan of the slice, and before any rank's next
 * scan or estimate.  Closes the slice like vbdr_slide.  d_mc_state may also be
 * this handle's own d_state: a group of one with no multicast object, where
 * the same kernel runs with the multimem operations replaced by the ordinary
 * load, store and atomic they reduce to over a single member (tests; one
 * GPU whose driver cannot create multicast objects). */
vbdr_status vbdr_slide_multicast(vbdr_t *h, void *d_mc_state, uint64_t j0, uint64_t j1,
                                 void *stream);

/* SYNC.  Test / single-GPU support for vbdr_slide_multicast: allocate
 * >= bytes of device memory on the current device bound to a one-device
 * multicast object; *d_uc receives the ordinary (unicast) address to pass to
 * vbdr_create, *d_mc the multicast address of the same memory, *granted the
 * size (rounded up to the multicast granularity).  VBDR_ECUDA if the device or
 * driver has no multicast support.  Free with vbdr_mc_free(d_uc). */
vbdr_status vbdr_mc_alloc(uint64_t bytes, void **d_uc, void **d_mc, uint64_t *granted);
vbdr_status vbdr_mc_free(void *d_uc);
/* Why the calling thread's last vbdr_mc_alloc failed ("" after a success). */
const char *vbdr_mc_last_error(void);

/* Estimate |OP(aip, t, k)| (Definition 1) for n_hosts hosts
 * over the window W(t-k+1..t) of the last closed slice: Alg.5 gather
 * (PAPER.md:197-213), HyperLogLog harmonic mean with linear counting, vHLL
 * noise subtraction (R#15, R#16), fp64.  d_hosts is
 * u32[n_hosts], d_out f64[n_hosts].  Before the first slide every estimate
 * is 0. */
vbdr_status vbdr_estimate(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts,
                          double *d_out, void *stream);

/* Integer stage of vbdr_estimate for parity: per host S = sum_i
 * 2^(L - M[pidx_i]) (u64) and V = #{M[pidx_i] = 0} (u32). */
vbdr_status vbdr_host_sums(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts,
                           uint64_t *d_S, uint32_t *d_V, void *stream);

/* Super-spreader readout (the paper's motivation, PAPER.md:28,
 * 68): write into d_idx (u32[n]) the positions j of the estimates d_est[j]
 * >= threshold and their number into *d_count (u64, device).  The order of the
 * positions is unspecified (sort them by estimate as needed). */
vbdr_status vbdr_select_above(vbdr_t *h, const double *d_est, uint64_t n, double threshold,
                              uint32_t *d_idx, uint64_t *d_count, void *stream);

/* ---- plan-based estimation (a fixed host list) ------------------------ */

/* The gather estimate (vbdr_estimate) reads each register of Alg.5
 * with its own L2 sector request: the (host, i) indices of
 * Alg.3 are random.  A PLAN preprocesses a host list once
 * (the monitored hosts) so that every later estimate reads the same registers
 * in a cheaper order.  All kinds produce the same integer sums and the same
 * fp64 finish: results are bit-identical to vbdr_estimate.  Kinds:
 *  - VBDR_PLAN_SORTED (k_splan.cu): every (host, i) listed once, sorted by
 *    register line, per CTA of a grid of P host groups x C register ranges;
 *    each CTA keeps its group's (S', V) in shared memory (8 B per host), so
 *    needs ceil(n_hosts / P) * 8 B <= the SM's shared memory (with C = 1:
 *    about 4.2 M hosts on 148 SMs), g * 2^(L-1) (HLL) or g * 255 below 2^32,
 *    n_phys >= 128.  Plan: 4 B per (host, i) plus the bucket table
 *    (n_phys * P / 128 * 4 B).  One estimate per plan at a time (stream-ordered).
 *  - VBDR_PLAN_STAGED (k_plan.cu): the register array streamed through shared
 *    memory in blocks of up to 64 KB by TMA, (host, i) entries grouped by
 *    block and warp in bank-scheduled rounds (4 B per (host, i)); n_phys in
 *    [64, 2^22]; the hosts' accumulators (8 B per host per CTA) share the
 *    SM's shared memory with the stages, so larger host lists get smaller
 *    blocks (caida's 500 k hosts: 64 KB; 1.2 M: 16 KB).
 *  - VBDR_PLAN_PASSID (k_estimate.cu): for pools whose gather estimate runs
 *    in 2..4 passes (est_pass_log2), 64 <= g <= 2048: the pass of every
 *    (host, i) in 2 bits, so each pass hashes and gathers only its registers.
 * VBDR_PLAN_AUTO takes STAGED when it fits and n_hosts * m >= n_phys (the
 * gathers outnumber the registers every SM streams), else the first that
 * fits in the order SORTED, STAGED, PASSID; otherwise VBDR_ERANGE. */
typedef enum {
    VBDR_PLAN_AUTO = 0,
    VBDR_PLAN_STAGED = 1,
    VBDR_PLAN_PASSID = 2,
    VBDR_PLAN_SORTED = 3
} vbdr_plan_kind;

/* SYNC, host only.  Bytes of the caller's plan buffer for n_hosts hosts
 * (VBDR_PLAN_AUTO); VBDR_ERANGE if no kind fits. */
vbdr_status vbdr_plan_bytes(const vbdr_t *h, uint64_t n_hosts, uint64_t *bytes);

/* vbdr_plan_bytes for one kind (vbdr_plan_kind). */
vbdr_status vbdr_plan_bytes_kind(const vbdr_t *h, uint64_t n_hosts, uint32_t kind,
                                 uint64_t *bytes);

/* SYNC.  Build the plan for d_hosts (u32[n_hosts], kept by the plan only as
 * indices: later estimates report host j at position j) into d_plan
 * (256-byte aligned, >= vbdr_plan_bytes), kind VBDR_PLAN_AUTO.  VBDR_ERANGE
 * if no kind fits (then use vbdr_estimate).  The plan belongs to this handle
 * and stays valid until vbdr_plan_release or the handle is destroyed. */
vbdr_status vbdr_plan_build(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts, void *d_plan,
                            uint64_t bytes, void *stream);

/* vbdr_plan_build of one kind (vbdr_plan_kind; bytes from vbdr_plan_bytes_kind). */
vbdr_status vbdr_plan_build_kind(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts,
                                 uint32_t kind, void *d_plan, uint64_t bytes, void *stream);

/* vbdr_estimate for the plan's hosts (d_out f64[n_hosts]). */
vbdr_status vbdr_estimate_plan(vbdr_t *h, const void *d_plan, double *d_out, void *stream);

/* vbdr_estimate_plan into the device stage d_out_stage, then copied to the
 * HOST buffer h_out (pinned for overlap; valid after `stream` syncs). */
vbdr_status vbdr_estimate_plan_host(vbdr_t *h, const void *d_plan, double *d_out_stage,
                                    double *h_out, void *stream);

/* vbdr_host_sums for the plan's hosts. */
vbdr_status vbdr_host_sums_plan(vbdr_t *h, const void *d_plan, uint64_t *d_S, uint32_t *d_V,
                                void *stream);

/* SYNC.  VBDR_ECUDA if a plan estimate on this plan ever timed out waiting for
 * a staged transfer (VBDR_PLAN_STAGED only; never expected: the kernel stops
 * instead of hanging and writes NaN estimates, or all-ones sums, for the hosts
 * it could not finish -- never a stale value). */
vbdr_status vbdr_plan_check(vbdr_t *h, const void *d_plan, void *stream);

/* Forget a plan (the caller frees its buffer). */
vbdr_status vbdr_plan_release(vbdr_t *h, const void *d_plan);

/* ---- host-buffer entry points (end-to-end path) ---------------------- */

/* vbdr_scan_slice on HOST pairs: copies h_pairs (pinned for overlap) through
 * the caller's device staging buffer d_stage (u32[2*stage_pairs], split in
 * two halves) chunk by chunk on an internal copy stream, overlapping each
 * chunk's host-to-device copy with the scan of the previous chunk -- and,
 * across calls, with the slide/estimate queued in between (a copy into a half
 * waits only for the last scan that read it).  Scans are ordered on `stream`;
 * h_pairs must stay valid until `stream` reaches this point.  Use the same
 * staging buffer for consecutive calls. */
vbdr_status vbdr_scan_slice_host(vbdr_t *h, const uint32_t *h_pairs, uint64_t n_pairs,
                                 uint32_t *d_stage, uint64_t stage_pairs, void *stream);

/* vbdr_estimate on HOST buffers: copies h_hosts into d_hosts_stage on the
 * internal copy stream (behind earlier pair copies, never behind compute), runs
 * the estimate into d_out_stage on `stream` and copies the results into h_out.
 * Stream-ordered; h_out is valid after `stream` is synchronised. */
vbdr_status vbdr_estimate_host(vbdr_t *h, const uint32_t *h_hosts, uint64_t n_hosts,
                               uint32_t *d_hosts_stage, double *d_out_stage,
                               double *h_out, void *stream);

/* ---- introspection and SYNC exports (tests, snapshots) ---------------- */

vbdr_status vbdr_info(const vbdr_t *h, vbdr_info_t *info);

/* SYNC (synchronises `stream`).  DR ages as u16[n_phys * L], row j, column
 * rho-1.  mode 0: the stored values (LAYOUT_FAST: the paper's DR values at
 * the last boundary, R#1; LAYOUT_PACKED: values already aged for the open
 * slice).  mode 1: canonical C_k[j][rho] = min(age, k) at the last boundary
 * (DESIGN.md section 4). */
vbdr_status vbdr_export_ages(vbdr_t *h, uint16_t *h_ages, int mode, void *stream);

/* SYNC.  vbdr_export_ages for the sampled BDRs d_idx (u64[n_idx], device),
 * through the caller's device scratch d_scratch (u32[n_idx * words]); h_ages
 * is u16[n_idx * L].  For pools too large to export whole. */
vbdr_status vbdr_export_ages_at(vbdr_t *h, const uint64_t *d_idx, uint64_t n_idx,
                                uint32_t *d_scratch, uint16_t *h_ages, int mode, void *stream);

/* SYNC.  Register values M[j] (u8[n_phys]) of the last boundary. */
vbdr_status vbdr_export_regmax(vbdr_t *h, uint8_t *h_regmax, void *stream);

/* SYNC.  Pool sums of the last boundary. */
vbdr_status vbdr_export_pool_sums(vbdr_t *h, uint64_t *h_S_tot, uint64_t *h_V_tot,
                                  void *stream);

/* TEST ONLY.  Start a fresh pool (no slide yet) at slice tick `tick` (odd,
 * < 2^26) so tests reach the stamp-tick wrap-around (every 2^26 slices) in a
 * few slices.  Semantically a no-op: stamps are 0 and only compare to ticks. */
vbdr_status vbdr_debug_set_tick(vbdr_t *h, uint32_t tick);

const char *vbdr_last_error(const vbdr_t *h);
const char *vbdr_status_string(vbdr_status s);

#ifdef __cplusplus
}
#endif
#endif /* VBDR_H */
