/*
 * vbdr_oracle.c -- plain, slow, single-threaded CPU oracle for VBDR
 * (Jie Xu, "Cardinalities estimation under sliding time window by sharing
 * HyperLogLog Counter", arXiv 1810.13132).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1810_13132_b200/) never links, imports or calls it,
 * and this file shares no header, helper, table or constant generator with
 * the CUDA path.
 *
 * Citations "PAPER.md:N" are lines of the paper text; "SPEC.md:N" lines of
 * the companion CPU specification; "R#n" rows of the reading ledger in
 * DESIGN.md section 3 (where the paper is silent, garbled or inconsistent).
 *
 * Representation: one uint16_t per distance recorder (DR), no packing, no
 * SIMD.  Every pool keeps its DRV as drv[j*L + (r-1)] for physical BDR j and
 * rank r in 1..L (R#3).  Floating point is fp64, round-to-nearest, compiled
 * with -ffp-contract=off (R#17).
 *
 * Pins (tests/, -m "not gpu"):
 *   H / fmix32 ........ MurmurHash3_x86_32 published vectors (tests/golden)
 *   LB, LBP1 .......... SPEC.md:56-58, 177-179 vectors; brute-force bit scan
 *   DR ops ............ SPEC.md:63-86 (definitional)
 *   Alg.1/2/8 traces .. SPEC.md:102-104, 111-113, 120-122
 *   pool readout ...... brute-force windowed max (sliding correctness,
 *                       SPEC.md:125), variant equivalence,
 *                       expiry, order invariance
 *   getPhyIdx+gather .. textbook HyperLogLog of one host, no sharing
 *   HLL / vHLL ........ closed forms (all-equal registers, linear counting)
 *   Table 1 ........... SPEC.md:280-282 integers
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* L1: hashing and indexing (section 4.1)            */
/* ------------------------------------------------------------------ */

/* H(x, N, A): "a random hash function with seed A that maps an integer x
 * to an integer smaller than N".  The paper does not name
 * the function; R#6 fixes the MurmurHash3 32-bit finaliser applied to x XOR
 * A, reduced mod N (N = 2^32 is the identity). */
uint32_t orc_fmix32(uint32_t x)
{
    uint32_t t = x;
    t ^= t >> 16;
    t *= 0x85EBCA6Bu;
    t ^= t >> 13;
    t *= 0xC2B2AE35u;
    t ^= t >> 16;
    return t;
}

uint64_t orc_H(uint32_t x, uint64_t N, uint32_t A)
{
    uint64_t t = (uint64_t)orc_fmix32(x ^ A);
    return t % N; /* N = 2^32 leaves t unchanged */
}

/* LB(x, i): "return the left i bits of the binary form of integer x"
 * (PAPER.md:170). */
uint32_t orc_LB(uint32_t x, uint32_t i)
{
    if (i == 0) return 0;
    return x >> (32 - i);
}

/* LBP1(v): "the most left 1 bit position as defined in HyperLogLog"
 * (PAPER.md:90), 1-based from the MSB (R#5), saturating at w when the top w
 * bits are all zero (R#4).  Written as the plain bit scan. */
uint32_t orc_LBP1(uint32_t v, uint32_t w)
{
    for (uint32_t pos = 1; pos <= w; ++pos) {
        uint32_t bit = 32 - pos; /* position 1 is bit 31 */
        if ((v >> bit) & 1u) return pos;
    }
    return w;
}

/* Alg.3 getPhyIdx:
 *   s1 <- H(i, 2^32, A0);  j <- H(aip, z, s1). */
uint64_t orc_getPhyIdx(uint32_t aip, uint32_t i, uint32_t A0, uint64_t z)
{
    uint32_t s1 = (uint32_t)orc_H(i, 1ull << 32, A0);
    return orc_H(aip, z, s1);
}

/* Per-pair front end of Alg.4:
 *   bip' <- H(bip, 2^32, A1); vidx <- LB(bip', b); bip' <- bip' << b;
 *   pidx <- getPhyIdx(aip, vidx, A0); rank <- LBP1(bip').
 * Rank width L (R#3: L = 32 - b by default, any 1 <= L <= 32 - b). */
void orc_pair_index(uint32_t aip, uint32_t bip, uint32_t b, uint32_t L,
                    uint32_t A0, uint32_t A1, uint64_t z,
                    uint64_t *pidx, uint32_t *rank)
{
    uint32_t bp = (uint32_t)orc_H(bip, 1ull << 32, A1);
    uint32_t vidx = orc_LB(bp, b);
    bp = bp << b;
    *pidx = orc_getPhyIdx(aip, vidx, A0, z);
    *rank = orc_LBP1(bp, L);
}

/* ------------------------------------------------------------------ */
/* L2: distance recorder operations (section 3)         */
/* ------------------------------------------------------------------ */

/* InitDR: "set the value of dr to 2^z - 1". */
void orc_InitDR(uint16_t *dr, uint32_t zb) { *dr = (uint16_t)((1u << zb) - 1u); }

/* SetDR: "set the value of dr to 0". */
void orc_SetDR(uint16_t *dr) { *dr = 0; }

/* SlideDR: "if dr <= 2^k-1, dr++" -- garbled; R#1 reads it
 * as a saturating increment at the recorder's own maximum 2^zb - 1. */
void orc_SlideDR(uint16_t *dr, uint32_t zb)
{
    uint32_t sentinel = (1u << zb) - 1u;
    if (*dr < sentinel) *dr = (uint16_t)(*dr + 1);
}

/* IsActiveDR: "if dr < k, dr is active". */
int orc_IsActiveDR(uint16_t dr, uint32_t k) { return dr < k; }

/* ------------------------------------------------------------------ */
/* Single-BDR algorithms (DRV = L recorders, drv[r-1] is rank r)        */
/* ------------------------------------------------------------------ */

/* Alg.1 EndSliceUpdateBDR: SlideDR every DR, then
 * SetDR(DRV[nowLBP1]).  nowLBP1 = 0 means nothing was seen (R#9). */
void orc_bdr_end_slice_serial(uint16_t *drv, uint32_t L, uint32_t zb, uint32_t now)
{
    for (uint32_t r = 1; r <= L; ++r) orc_SlideDR(&drv[r - 1], zb);
    if (now > 0) orc_SetDR(&drv[now - 1]);
}

/* Alg.6 EndSliceUpdateBDRGpu with R#10: SlideDR every DR,
 * then lbp1 <- the biggest rank whose bsLBP1 bit is 1 ("finding the biggest
 * 1 bit position"), SetDR(DRV[lbp1]) if any.  Bit r-1 of bs
 * stands for rank r. */
void orc_bdr_end_slice_gfast(uint16_t *drv, uint32_t L, uint32_t zb, uint32_t bs)
{
    for (uint32_t r = 1; r <= L; ++r) orc_SlideDR(&drv[r - 1], zb);
    uint32_t lbp1 = 0;
    for (uint32_t i = 1; i <= L; ++i)
        if ((bs >> (i - 1)) & 1u) lbp1 = i;
    if (lbp1 > 0) orc_SetDR(&drv[lbp1 - 1]);
}

/* Alg.8 BeginSliceUpdateDRV: SlideDR every DR. */
void orc_bdr_begin_slice_gsmall(uint16_t *drv, uint32_t L, uint32_t zb)
{
    for (uint32_t r = 1; r <= L; ++r) orc_SlideDR(&drv[r - 1], zb);
}

/* Alg.2 GetLBP1BDR with R#12: lbp1 runs from L down to 1;
 * the first active DR gives the answer; "Return 0" when none is active. */
uint32_t orc_bdr_GetLBP1(const uint16_t *drv, uint32_t L, uint32_t k)
{
    for (uint32_t lbp1 = L; lbp1 >= 1; --lbp1)
        if (orc_IsActiveDR(drv[lbp1 - 1], k)) return lbp1;
    return 0;
}

/* ------------------------------------------------------------------ */
/* L3: the BDR pool BDRP and the three paper variants    */
/* ------------------------------------------------------------------ */

enum { ORC_SERIAL = 0, ORC_GFAST = 1, ORC_GSMALL = 2 };

typedef struct {
    int variant;
    uint32_t b, L, k, zb, A0, A1;
    uint64_t z;      /* number of physical BDRs (the paper's pool size z) */
    uint16_t *drv;    /* z * L distance recorders                          */
    uint8_t *now;    /* serial: nowLBP1 per BDR              */
    uint32_t *bs;    /* gfast: bsLBP1 per BDR               */
    uint64_t slices; /* number of closed slices                            */
} orc_pool;

orc_pool *orc_pool_new(int variant, uint32_t b, uint32_t L, uint32_t k,
                       uint32_t zb, uint64_t z, uint32_t A0, uint32_t A1)
{
    if (variant < 0 || variant > 2 || b < 1 || b > 31 || L < 1 || L > 32 - b ||
        L > 32 || k < 1 || zb < 1 || zb > 16 || ((1u << zb) - 1u) < k || z < 1)
        return NULL;
    orc_pool *p = (orc_pool *)calloc(1, sizeof(orc_pool));
    if (!p) return NULL;
    p->variant = variant; p->b = b; p->L = L; p->k = k; p->zb = zb;
    p->A0 = A0; p->A1 = A1; p->z = z;
    p->drv = (uint16_t *)malloc((size_t)(z * L) * sizeof(uint16_t));
    p->now = (uint8_t *)calloc((size_t)z, 1);
    p->bs = (uint32_t *)calloc((size_t)z, sizeof(uint32_t));
    if (!p->drv || !p->now || !p->bs) {
        free(p->drv); free(p->now); free(p->bs); free(p);
        return NULL;
    }
    for (uint64_t i = 0; i < z * L; ++i) orc_InitDR(&p->drv[i], zb);
    return p;
}

void orc_pool_free(orc_pool *p)
{
    if (!p) return;
    free(p->drv); free(p->now); free(p->bs); free(p);
}

/* Slice open.  gsmall: Alg.8 on every BDR "at the beginning of a time slice
 * before scanning the IP pairs".  gfast: "Every bit of bsLBP1
 * is reset to 0 at the beginning of every time slice" (R#11).
 * serial: nothing (nowLBP1 is reset after its use in the close, R#9). */
void orc_begin_slice(orc_pool *p)
{
    if (p->variant == ORC_GSMALL) {
        for (uint64_t j = 0; j < p->z; ++j)
            orc_bdr_begin_slice_gsmall(&p->drv[j * p->L], p->L, p->zb);
    } else if (p->variant == ORC_GFAST) {
        for (uint64_t j = 0; j < p->z; ++j) p->bs[j] = 0;
    }
}

/* Scan of IPpair(t) (interleaved aip, bip).  serial: Alg.4
 * nowLBP1 <- max(nowLBP1, LBP1); gfast: Alg.7
 * bsLBP1[LBP1] = 1; gsmall: Alg.9
 * SetDR(DRV[LBP1]). */
void orc_scan(orc_pool *p, const uint32_t *pairs, uint64_t n)
{
    for (uint64_t q = 0; q < n; ++q) {
        uint64_t pidx;
        uint32_t r;
        orc_pair_index(pairs[2 * q], pairs[2 * q + 1], p->b, p->L, p->A0,
                       p->A1, p->z, &pidx, &r);
        if (p->variant == ORC_SERIAL) {
            if (r > p->now[pidx]) p->now[pidx] = (uint8_t)r;
        } else if (p->variant == ORC_GFAST) {
            p->bs[pidx] |= 1u << (r - 1);
        } else {
            orc_SetDR(&p->drv[pidx * p->L + (r - 1)]);
        }
    }
}

/* Slice close.  serial: Alg.4 lines 187-189 run Alg.1 on every BDR, then
 * nowLBP1 <- 0.  gfast: Alg.6 on every BDR.  gsmall: nothing (its ageing is
 * Alg.8 at the next slice open). */
void orc_end_slice(orc_pool *p)
{
    if (p->variant == ORC_SERIAL) {
        for (uint64_t j = 0; j < p->z; ++j) {
            orc_bdr_end_slice_serial(&p->drv[j * p->L], p->L, p->zb, p->now[j]);
            p->now[j] = 0;
        }
    } else if (p->variant == ORC_GFAST) {
        for (uint64_t j = 0; j < p->z; ++j)
            orc_bdr_end_slice_gfast(&p->drv[j * p->L], p->L, p->zb, p->bs[j]);
    }
    p->slices += 1;
}

/* GetLBP1BDR (Alg.2) of every physical BDR: M[j]. */
void orc_readout(const orc_pool *p, uint8_t *M)
{
    for (uint64_t j = 0; j < p->z; ++j)
        M[j] = (uint8_t)orc_bdr_GetLBP1(&p->drv[j * p->L], p->L, p->k);
}

void orc_export_drv(const orc_pool *p, uint16_t *out)
{
    memcpy(out, p->drv, (size_t)(p->z * p->L) * sizeof(uint16_t));
}

void orc_import_drv(orc_pool *p, const uint16_t *in)
{
    memcpy(p->drv, in, (size_t)(p->z * p->L) * sizeof(uint16_t));
}

void orc_export_now(const orc_pool *p, uint8_t *out)
{
    memcpy(out, p->now, (size_t)p->z);
}

/* Alg.5 getSumLBP1: sum over i of GetLBP1BDR of
 * BDRP[getPhyIdx(aip, i, A0)], from a readout M. */
uint64_t orc_getSumLBP1(const orc_pool *p, const uint8_t *M, uint32_t aip)
{
    uint64_t s = 0;
    uint32_t g = 1u << p->b;
    for (uint32_t i = 0; i < g; ++i) s += M[orc_getPhyIdx(aip, i, p->A0, p->z)];
    return s;
}

/* gather of the virtual vector VBV(aip): the g register
 * values the estimator consumes. */
void orc_gather(const orc_pool *p, const uint8_t *M, uint32_t aip, uint8_t *regs)
{
    uint32_t g = 1u << p->b;
    for (uint32_t i = 0; i < g; ++i) regs[i] = M[orc_getPhyIdx(aip, i, p->A0, p->z)];
}

/* ------------------------------------------------------------------ */
/* L4: estimator (delegated by PAPER.md:214 to vHLL eq.(5); R#15/16)    */
/* ------------------------------------------------------------------ */

/* HyperLogLog constant alpha_s. */
double orc_alpha(uint64_t s)
{
    if (s == 16) return 0.673;
    if (s == 32) return 0.697;
    if (s == 64) return 0.709;
    return 0.7213 / (1.0 + 1.079 / (double)s);
}

/* Harmonic-mean sum Z = sum_j 2^-M[j] and the zero count V, plain loop. */
void orc_hll_sums(const uint8_t *M, uint64_t s, double *Z, uint64_t *V)
{
    double z = 0.0;
    uint64_t v = 0;
    for (uint64_t j = 0; j < s; ++j) {
        z += ldexp(1.0, -(int)M[j]);
        if (M[j] == 0) v += 1;
    }
    *Z = z;
    *V = v;
}

/* HyperLogLog raw estimate with small-range correction (the
 * formula as fixed by SPEC.md:260): E = alpha_s s^2 / Z; if E <= 2.5 s and
 * V > 0 then E = s ln(s / V).  No large-range correction (R#16). */
double orc_hll_from_sums(uint64_t s, double Z, uint64_t V)
{
    double E = orc_alpha(s) * (double)s * (double)s / Z;
    if (E <= 2.5 * (double)s && V > 0)
        E = (double)s * log((double)s / (double)V);
    return E;
}

double orc_hll_raw(const uint8_t *M, uint64_t s)
{
    double Z;
    uint64_t V;
    orc_hll_sums(M, s, &Z, &V);
    return orc_hll_from_sums(s, Z, V);
}

/* vHLL noise subtraction (PAPER.md:214 -> "equation (5)"):
 * est = max(0, (z g / (z - g)) (E_s / g - E_tot / z)). */
double orc_vhll(uint64_t z, uint32_t g, double E_s, double E_tot)
{
    double C = ((double)z * (double)g) / (double)(z - g);
    double est = C * (E_s / (double)g - E_tot / (double)z);
    return est > 0.0 ? est : 0.0;
}

/* Per-host estimates for a list of hosts from readout M. */
void orc_estimate(const orc_pool *p, const uint8_t *M, const uint32_t *hosts,
                  uint64_t n, double *out)
{
    uint32_t g = 1u << p->b;
    double E_tot = orc_hll_raw(M, p->z);
    uint8_t *regs = (uint8_t *)malloc(g);
    for (uint64_t h = 0; h < n; ++h) {
        orc_gather(p, M, hosts[h], regs);
        double E_s = orc_hll_raw(regs, g);
        out[h] = orc_vhll(p->z, g, E_s, E_tot);
    }
    free(regs);
}

/* Estimates straight from a register array M (no pool needed: for pools too
 * large to hold the oracle's one-DR-per-uint16 state, M comes from
 * orc_rebuild).  Same steps as orc_estimate. */
void orc_estimate_M(uint32_t b, uint32_t A0, uint64_t z, const uint8_t *M,
                    const uint32_t *hosts, uint64_t n, double *out)
{
    uint32_t g = 1u << b;
    double E_tot = orc_hll_raw(M, z);
    uint8_t *regs = (uint8_t *)malloc(g);
    for (uint64_t h = 0; h < n; ++h) {
        for (uint32_t i = 0; i < g; ++i) regs[i] = M[orc_getPhyIdx(hosts[h], i, A0, z)];
        double E_s = orc_hll_raw(regs, g);
        out[h] = orc_vhll(z, g, E_s, E_tot);
    }
    free(regs);
}

void orc_host_sums_M(uint32_t b, uint32_t A0, uint64_t z, const uint8_t *M,
                     const uint32_t *hosts, uint64_t n, double *Z, uint64_t *V)
{
    uint32_t g = 1u << b;
    uint8_t *regs = (uint8_t *)malloc(g);
    for (uint64_t h = 0; h < n; ++h) {
        for (uint32_t i = 0; i < g; ++i) regs[i] = M[orc_getPhyIdx(hosts[h], i, A0, z)];
        orc_hll_sums(regs, g, &Z[h], &V[h]);
    }
    free(regs);
}

/* Per-host harmonic sums (Z_s, V_s) for parity of the integer stage. */
void orc_host_sums(const orc_pool *p, const uint8_t *M, const uint32_t *hosts,
                   uint64_t n, double *Z, uint64_t *V)
{
    uint32_t g = 1u << p->b;
    uint8_t *regs = (uint8_t *)malloc(g);
    for (uint64_t h = 0; h < n; ++h) {
        orc_gather(p, M, hosts[h], regs);
        orc_hll_sums(regs, g, &Z[h], &V[h]);
    }
    free(regs);
}

/* ------------------------------------------------------------------ */
/* Method variants: the BDR pool under other        */
/* register estimators                                                  */
/* ------------------------------------------------------------------ */

/* PCSA register of one BDR under a sliding window.  PCSA (Flajolet-Martin,
 * PAPER.md:58) keeps a bitmap per register and reads R = the position of its
 * lowest zero bit.  "BDRP could also be used in PCSA ... by replacing its
 * nowLBP1 with the value recorded in other algorithms": the
 * sliding bitmap is {r : DRV[r] active} -- which needs every rank recorded,
 * i.e. the gsmall DRV (Alg.9).  R = (lowest inactive rank) - 1, or L when all
 * L ranks are active. */
uint32_t orc_bdr_pcsa_R(const uint16_t *drv, uint32_t L, uint32_t k)
{
    for (uint32_t r = 1; r <= L; ++r)
        if (!orc_IsActiveDR(drv[r - 1], k)) return r - 1;
    return L;
}

void orc_readout_pcsa(const orc_pool *p, uint8_t *R)
{
    for (uint64_t j = 0; j < p->z; ++j)
        R[j] = (uint8_t)orc_bdr_pcsa_R(&p->drv[j * p->L], p->L, p->k);
}

/* LogLog bias constant (Durand & Flajolet 2003):
 *   alpha_m = (Gamma(-1/m) (1 - 2^(1/m)) / ln 2)^(-m).
 * Both factors are negative; written in logs,
 *   alpha_m = exp(-m [ln|Gamma(-1/m)| + ln(2^(1/m) - 1) - ln ln 2]),
 * with 2^(1/m) - 1 = expm1(ln2 / m) so large m does not cancel digits. */
double orc_loglog_alpha(uint64_t m)
{
    double x = 1.0 / (double)m;
    double lb = lgamma(-x) + log(expm1(x * log(2.0))) - log(log(2.0));
    return exp(-(double)m * lb);
}

/* LogLog raw estimate from the register values: alpha_s s 2^(sum M / s) --
 * the geometric-mean estimator that consumes exactly Alg.5's sum of LBP1
 * (PAPER.md:195-213, 60). */
double orc_loglog_raw(const uint8_t *M, uint64_t s)
{
    uint64_t sum = 0;
    for (uint64_t j = 0; j < s; ++j) sum += M[j];
    return orc_loglog_alpha(s) * (double)s * pow(2.0, (double)sum / (double)s);
}

/* PCSA raw estimate: (s / phi) 2^(sum R / s), phi = 0.77351 (Flajolet-Martin). */
double orc_pcsa_raw(const uint8_t *R, uint64_t s)
{
    uint64_t sum = 0;
    for (uint64_t j = 0; j < s; ++j) sum += R[j];
    return ((double)s / 0.77351) * pow(2.0, (double)sum / (double)s);
}

/* Per-host estimates with a chosen register estimator (0 HLL, 1 LogLog,
 * 2 PCSA) on register values V (M for HLL/LogLog, R for PCSA), combined with
 * the same shared-pool noise subtraction as orc_vhll (R#15). */
void orc_estimate_variant(uint32_t b, uint32_t A0, uint64_t z, const uint8_t *V,
                          const uint32_t *hosts, uint64_t n, int estimator, double *out)
{
    uint32_t g = 1u << b;
    double E_tot = estimator == 0 ? orc_hll_raw(V, z)
                 : estimator == 1 ? orc_loglog_raw(V, z) : orc_pcsa_raw(V, z);
    uint8_t *regs = (uint8_t *)malloc(g);
    for (uint64_t h = 0; h < n; ++h) {
        for (uint32_t i = 0; i < g; ++i) regs[i] = V[orc_getPhyIdx(hosts[h], i, A0, z)];
        double E_s = estimator == 0 ? orc_hll_raw(regs, g)
                   : estimator == 1 ? orc_loglog_raw(regs, g) : orc_pcsa_raw(regs, g);
        out[h] = orc_vhll(z, g, E_s, E_tot);
    }
    free(regs);
}

/* ------------------------------------------------------------------ */
/* LFPM (list of future possible maxima), the prior-art sliding counter  */
/* of LFPM-HLL the BDR replaces (section 2.3) */
/* ------------------------------------------------------------------ */

/* One LFPM: cells (slice, rank) with slices strictly increasing and ranks
 * strictly decreasing from head to tail.  Insert removes dominated cells
 * (rank <= new rank) from the tail, then appends; a query keeps
 * cells with slice > t - k and returns the head's rank, or 0. */
typedef struct {
    uint32_t n, cap;
    uint64_t *slice;
    uint32_t *rank;
} orc_lfpm;

orc_lfpm *orc_lfpm_new(void)
{
    orc_lfpm *l = (orc_lfpm *)calloc(1, sizeof(orc_lfpm));
    return l;
}

void orc_lfpm_free(orc_lfpm *l)
{
    if (!l) return;
    free(l->slice); free(l->rank); free(l);
}

void orc_lfpm_insert(orc_lfpm *l, uint64_t slice, uint32_t rank)
{
    while (l->n > 0 && l->rank[l->n - 1] <= rank) l->n -= 1;
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 8;
        l->slice = (uint64_t *)realloc(l->slice, l->cap * sizeof(uint64_t));
        l->rank = (uint32_t *)realloc(l->rank, l->cap * sizeof(uint32_t));
    }
    l->slice[l->n] = slice;
    l->rank[l->n] = rank;
    l->n += 1;
}

uint32_t orc_lfpm_query(orc_lfpm *l, uint64_t t, uint32_t k)
{
    uint32_t drop = 0;
    while (drop < l->n && l->slice[drop] + k <= t) drop += 1;  /* slice <= t - k: expired */
    if (drop) {
        memmove(l->slice, l->slice + drop, (l->n - drop) * sizeof(uint64_t));
        memmove(l->rank, l->rank + drop, (l->n - drop) * sizeof(uint32_t));
        l->n -= drop;
    }
    return l->n ? l->rank[0] : 0;
}

uint32_t orc_lfpm_len(const orc_lfpm *l) { return l->n; }

/* ------------------------------------------------------------------ */
/* Independent references                                               */
/* ------------------------------------------------------------------ */

/* Rebuild from scratch: M*[j] = max rank over every pair of the window's
 * slices mapping to j -- the windowed maximum the BDR maintains
 * (SPEC.md:117, 125).  pairs holds all pairs of
 * slices t-k+1..t concatenated. */
void orc_rebuild(uint32_t b, uint32_t L, uint32_t A0, uint32_t A1, uint64_t z,
                 const uint32_t *pairs, uint64_t n, uint8_t *Mstar)
{
    memset(Mstar, 0, (size_t)z);
    for (uint64_t q = 0; q < n; ++q) {
        uint64_t pidx;
        uint32_t r;
        orc_pair_index(pairs[2 * q], pairs[2 * q + 1], b, L, A0, A1, z, &pidx, &r);
        if (r > Mstar[pidx]) Mstar[pidx] = (uint8_t)r;
    }
}

/* Table 1: bits per BDR, with log2(n/g) -> L and
 * log2(k+1) -> zb = ceil(log2(k+1)).  The serial row's
 * log2(log2(n/g)) is the nowLBP1 width ceil(log2 L). */
uint64_t orc_memory_bits(int variant, uint32_t b, uint32_t k)
{
    uint32_t L = 32 - b;
    uint32_t zb = 0;
    while ((1ull << zb) < (uint64_t)k + 1) ++zb;
    uint32_t lgL = 0;
    while ((1u << lgL) < L) ++lgL;
    if (variant == ORC_SERIAL) return (uint64_t)lgL + (uint64_t)L * zb;
    if (variant == ORC_GFAST) return (uint64_t)L + (uint64_t)L * zb;
    return (uint64_t)L * zb;
}
