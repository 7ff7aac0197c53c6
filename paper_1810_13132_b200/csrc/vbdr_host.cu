// vbdr_host.cu -- the C ABI of libvbdr.so (declared in include/vbdr.h):
// configuration validation, state-layout planning, launches, host-buffer
// pipelines, estimate plans and parity exports.  No compute happens on the
// host: every step of the path runs in the kernels of k_scan_slide.cu,
// k_estimate.cu and k_plan.cu.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/vbdr.h"
#include "vbdr_dev.cuh"
#include <cstdlib>

using vbdr_dev::DevParams;

struct vbdr {
  vbdr_config cfg{};
  vbdr_info_t info{};
  DevParams p{};
  bool fast = true;     // layout F
  bool stamps = false;  // layout S (per-(BDR, rank) stamps)
  double alpha_g = 0, alpha_z = 0;
  std::string err;
  // host-buffer pipeline resources (created on first use)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_scanned[2] = {nullptr, nullptr};
  std::map<const void *, vbdr_launch::PlanLayout> plans;  // built plans by device address
  cudaEvent_t ev_hosts_in = nullptr;    // host ids copied (copy stream)
  cudaEvent_t ev_hosts_free = nullptr;  // last estimate that read the host stage
  // two register buffers: the slide of tick T writes buffer T & 1, so the
  // estimate of tick T - 1 may run concurrently with the next slide
  uint8_t *regmax_base = nullptr;
  uint64_t regmax_stride = 0;
};

namespace vbdr_dev {
int pdl_mode() {
  static const int mode = [] {
    const char *v = std::getenv("VBDR_PDL");
    if (!v || !*v) return 2;
    return v[0] == '0' ? 0 : (v[0] == '1' ? 1 : 2);
  }();
  return mode;
}
}  // namespace vbdr_dev

namespace {

constexpr uint32_t kTickLimit = 1u << 26;  // sr = (T << 5) | rho < 2^31: also a valid int32 for MAX merges

uint64_t align256(uint64_t x) { return (x + 255u) & ~uint64_t(255); }

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

uint32_t log2u(uint64_t x) {
  uint32_t r = 0;
  while ((1ull << r) < x) ++r;
  return r;
}

// LogLog bias constant (Durand & Flajolet): alpha_m = (Gamma(-1/m)(1 - 2^(1/m))
// / ln 2)^(-m), evaluated in logs with expm1 (no cancellation at large m).
double loglog_alpha(uint64_t m) {
  const double x = 1.0 / (double)m;
  const double lb = std::lgamma(-x) + std::log(std::expm1(x * std::log(2.0))) - std::log(std::log(2.0));
  return std::exp(-(double)m * lb);
}

// Register-estimator constant coef_s (LogLog alpha_s s, PCSA s / phi).
double est_coef(uint32_t est, uint64_t s) {
  if (est == 1) return loglog_alpha(s) * (double)s;
  if (est == 2) return (double)s / 0.77351;
  return 0.0;
}

// HyperLogLog alpha_s (R#16), same double operations as the oracle.
double alpha_of(uint64_t s) {
  if (s == 16) return 0.673;
  if (s == 32) return 0.697;
  if (s == 64) return 0.709;
  return 0.7213 / (1.0 + 1.079 / (double)s);
}

struct StateLayout {
  uint32_t b, L, zb, F, W;
  uint64_t off_acc, off_sr, off_drv, off_regmax, regmax_stride, bytes;
};

// scan_mode 0 = default: 5 for layout F, 2 for layout P
// (profiles/r01_scan_modes.txt; the slower modes 1, 3, 4 and 6 of round 1
// are recorded in tools/rejected/, not built).
uint32_t effective_scan_mode(const vbdr_config &n) {
  const bool fast = n.layout != VBDR_LAYOUT_PACKED;  // layout S as fast: the block cache
  return n.scan_mode ? n.scan_mode : (fast ? 5u : 2u);
}

// Validate a config and lay out the state buffer.  Returns an error text or
// empty on success.
std::string layout_state(const vbdr_config *c, vbdr_config *norm, StateLayout *pl) {
  if (!c) return "null config";
  vbdr_config n = *c;
  if (n.seed_a0 == 0 && n.seed_a1 == 0) {  // R#7 defaults
    n.seed_a0 = 0x5EED0001u;
    n.seed_a1 = 0x5EED0002u;
  }
  if (n.layout > 2) return "layout must be 0 (fast), 1 (packed) or 2 (stamps)";
  if (n.scan_mode != 0 && n.scan_mode != 2 && n.scan_mode != 5)
    return "scan_mode must be 0 (default), 2 (L2 check) or 5 (block cache + L2 check)";
  if (n.est_lanes > 32 || (n.est_lanes & (n.est_lanes - 1)))
    return "est_lanes must be 0 or a power of two <= 32";
  if (n.est_pass_log2 > 32) return "est_pass_log2 must be 0..32";
  if (n.estimator > 2) return "estimator must be 0 (HLL), 1 (LogLog) or 2 (PCSA)";
  if (n.drv_shards > 1) {
    if (n.layout != VBDR_LAYOUT_FAST) return "drv_shards needs layout fast";
    if (n.drv_shard >= n.drv_shards) return "drv_shard must be < drv_shards";
    if (n.n_phys % n.drv_shards || (n.n_phys / n.drv_shards) % 4)
      return "drv_shards must split n_phys into shards of multiples of 4";
  } else if (n.drv_shard != 0) {
    return "drv_shard needs drv_shards > 1";
  }
  if (n.estimator == 2 && n.layout == VBDR_LAYOUT_FAST)
    return "PCSA needs layout packed or stamps (every rank recorded: the sliding bitmap)";
  if (n.m < 2 || !is_pow2(n.m)) return "m must be a power of two >= 2";
  if (n.k < 1) return "k must be >= 1";
  if (n.n_phys < 4 || !is_pow2(n.n_phys) || n.n_phys > (1ull << 32))
    return "n_phys must be a power of two in [4, 2^32]";
  if (2ull * n.m > n.n_phys) return "2*m must be <= n_phys (vHLL denominator, R#15)";
  const uint32_t b = log2u(n.m);
  if (b > 31) return "m too large";
  const uint32_t L = n.rank_cap ? n.rank_cap : 32u - b;
  if (L < 1 || L > 32u - b) return "rank_cap must be in [1, 32 - log2(m)]";
  // the pool sum S_tot <= n_phys 2^L must convert to fp64 exactly
  if (log2u(n.n_phys) + L > 53) return "n_phys * 2^L must be <= 2^53 (exact fp64 pool sums)";
  uint32_t zb = n.zbits;
  const bool packed = n.layout == VBDR_LAYOUT_PACKED;
  if (zb == 0) {
    zb = log2u((uint64_t)n.k + 1);
    if (zb == 0) zb = 1;
    if (packed && ((1ull << zb) - 2) < n.k) zb += 1;  // R#2: S - 1 >= k for layout P
  }
  if (zb < 1 || zb > 10) return "zbits must be in [1, 10]";
  if (((1ull << zb) - 1) < n.k) return "2^zbits - 1 must be >= k (PAPER.md:92)";
  if (packed && ((1ull << zb) - 2) < n.k)
    return "layout packed needs 2^zbits - 2 >= k (canonical export, R#2)";
  n.zbits = zb;
  n.rank_cap = L;
  const bool stamps = n.layout == VBDR_LAYOUT_STAMPS;
  // layout S: one u32 stamp per (BDR, rank): L "words" of one field each
  const uint32_t F = stamps ? 1u : 32u / zb;
  const uint32_t W = stamps ? L : (L + F - 1) / F;
  uint64_t off = 0;
  pl->off_acc = off;
  off = align256(off + 8 * sizeof(uint64_t));  // (S_tot, V_tot) for tick mod 4
  pl->off_sr = off;
  if (!packed && !stamps) off = align256(off + 4ull * n.n_phys);
  pl->off_drv = off;
  const uint64_t drv_n = n.drv_shards > 1 ? n.n_phys / n.drv_shards : n.n_phys;
  off = align256(off + 4ull * W * drv_n);
  pl->off_regmax = off;  // two register buffers: the slide of tick T writes buffer T & 1
  pl->regmax_stride = align256(n.n_phys);
  off = align256(off + 2 * pl->regmax_stride);
  pl->bytes = off;
  pl->b = b;
  pl->L = L;
  pl->zb = zb;
  pl->F = F;
  pl->W = W;
  *norm = n;
  return {};
}

vbdr_status fail(vbdr *h, vbdr_status s, const std::string &msg) {
  if (h) h->err = msg;
  return s;
}

vbdr_status cuda_fail(vbdr *h, cudaError_t e, const char *where) {
  return fail(h, VBDR_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Sticky or pending asynchronous errors surface on the next call.
vbdr_status check_async(vbdr *h, const char *where) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(h, e, where);
  return VBDR_OK;
}

cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// scan_mode 0 picks the default (effective_scan_mode).
int scan_mode(const vbdr *h);

// kernels one scan call launches
uint64_t scan_launches(const vbdr *, uint64_t) { return 1; }

int scan_mode(const vbdr *h) {
  const uint32_t m = effective_scan_mode(h->cfg);
  if (h->stamps)  // the cache keys by (plane, BDR) word index: L * n_phys < 2^32
    return m == 5 && (uint64_t)h->p.L * h->p.n_phys < (1ull << 32) ? 5 : 2;
  // mode 5 keys its shared-memory cache by word index: fast needs n_phys < 2^32,
  // packed n_phys <= 2^28 (and W <= 15); otherwise use mode 2
  if (m == 5 && (h->fast ? h->p.n_phys >= (1ull << 32) : (h->p.n_phys > (1ull << 28) || h->p.W > 15)))
    return 2;
  return (int)m;
}

uint8_t *regmax_of(const vbdr *h, uint32_t tick) {
  return h->regmax_base + (tick & 1u) * h->regmax_stride;
}

vbdr_launch::EstParams est_params(const vbdr *h) {
  vbdr_launch::EstParams e{};
  const uint32_t closed = h->p.tick - 1u;  // tick of the last boundary (0 = none)
  e.regmax = regmax_of(h, closed);
  e.acc = h->p.acc + 2 * (closed & 3u);
  e.mask = h->p.mask;
  e.A0 = h->p.A0;
  e.L = h->p.L;
  e.g = h->cfg.m;
  e.lanes = h->cfg.est_lanes;
  // passes over L2-sized physical ranges (k_estimate.cu); 2^26 one-byte
  // registers = 64 MiB stays L2-resident on B200 (126 MB L2).  The packed
  // partial sums need g < 2^24.
  e.pass_log2 = h->cfg.est_pass_log2 ? h->cfg.est_pass_log2 : 26u;
  if (h->cfg.m >= (1u << 24)) e.pass_log2 = 32;
  e.inv2L = std::ldexp(1.0, -(int)h->p.L);
  const double g = (double)h->cfg.m, z = (double)h->cfg.n_phys;
  e.agg = h->alpha_g * g * g;  // exact: g is a power of two
  e.lc_g = 2.5 * g;
  e.azz = h->alpha_z * z * z;
  e.lc_z = 2.5 * z;
  e.z = z;
  e.C = ((double)h->cfg.n_phys * (double)h->cfg.m) / (double)(h->cfg.n_phys - h->cfg.m);
  e.est = h->cfg.estimator;
  e.coef_g = est_coef(e.est, h->cfg.m);
  e.coef_z = est_coef(e.est, h->cfg.n_phys);
  return e;
}

// Unpack one BDR's DR ages from its W packed words (word(w) accessor).
// mode 0: stored values; mode 1: canonical C_k = min(age, k) at the last
// boundary (layout P stores ages already advanced by Alg.8: undo it).
template <typename WordAt>
void decode_ages(const vbdr *h, WordAt word, int mode, uint16_t *out) {
  const uint32_t F = h->p.F, zb = h->p.zb, L = h->p.L, k = h->p.k;
  const uint32_t fm = (1u << zb) - 1u, sent = fm;
  for (uint32_t r = 1; r <= L; ++r) {
    const uint32_t w = (r - 1) / F, f = (r - 1) % F;
    uint32_t v = (word(w) >> (zb * f)) & fm;
    if (mode == 1) {
      if (!h->fast) v = (v == sent) ? k : (v ? v - 1u : 0u);
      if (v > k) v = k;
    }
    if (h->stamps) {  // age = closed tick - stamp; never stamped: k (canonical) / 0xFFFF
      const uint32_t st = word(r - 1), closed = h->p.tick - 1u;
      v = st == 0u ? (mode == 1 ? k : 0xFFFFu) : closed - st;
      if (mode == 1 && v > k) v = k;
      if (v > 0xFFFFu) v = 0xFFFFu;
    }
    out[r - 1] = (uint16_t)v;
  }
}

// Plan geometry for this pool: one persistent CTA per SM, blocks of up to
// 2^16 registers (64 KB in shared memory): the largest block whose stages and
// accumulators (hosts / SMs per CTA) fit shared memory and whose expected
// entries per (CTA, block) stay well inside a stage.
struct PlanGeom {
  uint32_t ctas, phases, block_log2, slots, hpc;
  uint64_t nkeys, off_range_base, off_starts, off_counts, off_range_size, off_misc, off_lct,
      off_entries, bytes;
};

bool plan_geom(const vbdr *h, uint64_t n_hosts, PlanGeom *g) {
  const uint64_t z = h->p.n_phys;
  if (z < 64 || z > (1ull << 22)) return false;  // the array streams through shared memory
  int sms = 0, dev = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (sms <= 0) sms = 148;
  if (smem_max <= 0) smem_max = 232448;
  if (n_hosts == 0 || n_hosts > 0xFFFFFFFFull) return false;
  // per-host S' (registers with M >= 1) accumulates in a u32 in shared memory:
  // at most g * 2^(L-1) (HLL) or g * 255
  const uint64_t smax =
      (uint64_t)h->cfg.m * (h->cfg.estimator == 0 ? 1ull << (h->p.L - 1) : 255ull);
  if (smax >> 32) return false;
  const uint64_t hpc = (n_hosts + sms - 1) / sms;
  const uint64_t slots = (hpc + vbdr_launch::kPlanThreads - 1) / vbdr_launch::kPlanThreads;
  // accumulator indices travel in the top 14 bits of an entry (<< 18)
  if (slots * 32 + 32 > (1u << 14)) return false;
  const double per_key_all = (double)n_hosts * h->cfg.m / sms;  // entries per CTA
  bool found = false;
  for (uint32_t bl = z >= (1ull << 16) ? 16u : (uint32_t)log2u(z); bl >= 6 && !found; --bl) {
    const double per_key = per_key_all / (double)(z >> bl);
    if (per_key + 6.0 * sqrt(per_key) + 16.0 * 32.0 > (double)vbdr_launch::plan_ent_cap(bl)) continue;
    const size_t smem = vbdr_launch::plan_smem_bytes(bl, (uint32_t)slots);
    if (smem == 0 || smem > (size_t)smem_max) continue;
    g->block_log2 = bl;
    found = true;
  }
  if (!found) return false;
  g->ctas = (uint32_t)sms;
  g->slots = (uint32_t)slots;
  g->hpc = (uint32_t)hpc;
  g->phases = (uint32_t)(z >> g->block_log2);
  g->nkeys = (uint64_t)g->ctas * g->phases;
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t o = off;
    off = align256(off + bytes);
    return o;
  };
  g->off_range_base = take(4 * (g->nkeys + 1));
  g->off_starts = take(4 * g->nkeys * vbdr_launch::kPlanStride);
  g->off_counts = take(4 * g->nkeys * vbdr_launch::kPlanThreads);
  g->off_range_size = take(4 * g->nkeys);
  g->off_misc = take(64);
  g->off_lct = take(8ull * (h->cfg.m + 1));  // linear-counting log table
  // every (CTA, block, warp) group is padded to whole rounds of 32 entries
  const uint64_t groups = g->nkeys * (vbdr_launch::kPlanThreads / 32);
  g->off_entries = take(4 * (n_hosts * h->cfg.m + 31 * groups));
  g->bytes = off;
  return true;
}

vbdr_launch::PlanLayout plan_layout(const PlanGeom &g, void *d_plan, uint64_t n_hosts) {
  uint8_t *b = static_cast<uint8_t *>(d_plan);
  vbdr_launch::PlanLayout pl{};
  pl.ctas = g.ctas;
  pl.phases = g.phases;
  pl.block_log2 = g.block_log2;
  pl.n_hosts = n_hosts;
  pl.range_base = reinterpret_cast<uint32_t *>(b + g.off_range_base);
  pl.starts = reinterpret_cast<uint32_t *>(b + g.off_starts);
  pl.counts = reinterpret_cast<uint32_t *>(b + g.off_counts);
  pl.range_size = reinterpret_cast<uint32_t *>(b + g.off_range_size);
  pl.max_range = reinterpret_cast<uint32_t *>(b + g.off_misc);
  pl.error = reinterpret_cast<unsigned long long *>(b + g.off_misc + 8);
  pl.st_slots = g.slots;
  pl.lct = reinterpret_cast<const double *>(b + g.off_lct);
  pl.st_hpc = g.hpc;
  pl.entries = reinterpret_cast<uint32_t *>(b + g.off_entries);
  return pl;
}

vbdr_status ensure_pipeline(vbdr *h, cudaStream_t cs) {
  if (h->copy_stream) return VBDR_OK;
  cudaError_t e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&h->ev_copied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_scanned[i], cudaEventDisableTiming);
    // "slot i is free" starts out as: everything queued on the caller's stream so far
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_scanned[i], cs);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_hosts_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_hosts_free, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_hosts_free, cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "pipeline resources");
  return VBDR_OK;
}

// Advance the host-side slice clock after a slide (shared by the slide paths).
vbdr_status after_slide(vbdr_t *h, void *stream) {
  h->info.launches += 1;
  h->info.slices_closed += 1;
  h->p.tick += 1;
  if (h->p.tick >= kTickLimit) {
    // Every stamp is stale after a slide; restart the tick at 4 (kTickLimit
    // mod 4, so the register buffers and accumulator slots keep rotating).
    if (h->fast || h->stamps) {
      const cudaError_t m = h->fast ? cudaMemsetAsync(h->p.sr, 0, 4ull * h->p.n_phys, S(stream))
                                    : cudaMemsetAsync(h->p.drv, 0, 4ull * h->p.W * h->p.n_phys,
                                                      S(stream));
      if (m != cudaSuccess) return cuda_fail(h, m, "tick wrap");
    }
    h->p.tick = 4;
  }
  h->p.regmax = regmax_of(h, h->p.tick);
  return VBDR_OK;
}

}  // namespace

extern "C" {

const char *vbdr_status_string(vbdr_status s) {
  switch (s) {
    case VBDR_OK: return "ok";
    case VBDR_EINVAL: return "invalid argument";
    case VBDR_ERANGE: return "out of range";
    case VBDR_ESTATE: return "invalid state";
    case VBDR_ENOMEM: return "out of memory";
    case VBDR_ECUDA: return "cuda error";
  }
  return "unknown";
}

const char *vbdr_last_error(const vbdr_t *h) { return h ? h->err.c_str() : "null handle"; }

vbdr_status vbdr_state_bytes(const vbdr_config *cfg, uint64_t *bytes) {
  if (!bytes) return VBDR_EINVAL;
  vbdr_config n;
  StateLayout pl;
  if (!layout_state(cfg, &n, &pl).empty()) return VBDR_EINVAL;
  *bytes = pl.bytes;
  return VBDR_OK;
}

const char *vbdr_config_check(const vbdr_config *cfg) {
  static thread_local std::string msg;
  vbdr_config n;
  StateLayout pl;
  msg = layout_state(cfg, &n, &pl);
  return msg.empty() ? nullptr : msg.c_str();
}

vbdr_status vbdr_create(const vbdr_config *cfg, void *d_state, uint64_t bytes, void *stream,
                        vbdr_t **out) {
  if (!out) return VBDR_EINVAL;
  *out = nullptr;
  vbdr *h = new (std::nothrow) vbdr();
  if (!h) return VBDR_ENOMEM;
  StateLayout pl;
  std::string e = layout_state(cfg, &h->cfg, &pl);
  if (!e.empty() || !d_state || (reinterpret_cast<uintptr_t>(d_state) & 255u)) {
    delete h;
    return VBDR_EINVAL;
  }
  if (bytes < pl.bytes) {
    delete h;
    return VBDR_ENOMEM;
  }
  cudaGetLastError();  // do not inherit someone else's error
  h->fast = h->cfg.layout == VBDR_LAYOUT_FAST;
  h->stamps = h->cfg.layout == VBDR_LAYOUT_STAMPS;
  uint8_t *base = static_cast<uint8_t *>(d_state);
  DevParams &p = h->p;
  p.acc = reinterpret_cast<unsigned long long *>(base + pl.off_acc);
  p.sr = h->fast ? reinterpret_cast<uint32_t *>(base + pl.off_sr) : nullptr;
  p.drv = reinterpret_cast<uint32_t *>(base + pl.off_drv);
  h->regmax_base = base + pl.off_regmax;
  h->regmax_stride = pl.regmax_stride;
  p.regmax = h->regmax_base;  // k_init clears buffer 0; buffer 1 below
  p.n_phys = h->cfg.n_phys;
  p.drv_n = h->cfg.drv_shards > 1 ? h->cfg.n_phys / h->cfg.drv_shards : h->cfg.n_phys;
  p.drv_j0 = h->cfg.drv_shards > 1 ? p.drv_n * h->cfg.drv_shard : 0;
  p.mask = (uint32_t)(h->cfg.n_phys - 1);
  p.b = pl.b;
  p.L = pl.L;
  p.k = h->cfg.k;
  p.zb = pl.zb;
  p.F = pl.F;
  p.W = pl.W;
  p.A0 = h->cfg.seed_a0;
  p.A1 = h->cfg.seed_a1;
  p.tick = 1;  // slice t = 0 is open, T = t + 1
  p.est = h->cfg.estimator;
  h->alpha_g = alpha_of(h->cfg.m);
  h->alpha_z = alpha_of(h->cfg.n_phys);
  vbdr_info_t &in = h->info;
  in.b = pl.b;
  in.L = pl.L;
  in.zbits = pl.zb;
  in.fields = pl.F;
  in.words = pl.W;
  in.n_phys = h->cfg.n_phys;
  in.off_acc = pl.off_acc;
  in.off_sr = h->fast ? pl.off_sr : ~0ull;
  in.off_drv = pl.off_drv;
  in.off_regmax = pl.off_regmax;
  in.state_bytes = pl.bytes;
  cudaError_t ce;
  if (h->stamps) {  // no DRs to InitDR: every stamp 0 (never recorded)
    DevParams p0 = p;
    p0.W = 0;
    ce = vbdr_launch::init(p0, false, S(stream));
    if (ce == cudaSuccess) ce = cudaMemsetAsync(p.drv, 0, 4ull * p.W * p.n_phys, S(stream));
  } else {
    ce = vbdr_launch::init(p, h->fast, S(stream));
  }
  if (ce == cudaSuccess)
    ce = cudaMemsetAsync(h->regmax_base + h->regmax_stride, 0, h->cfg.n_phys, S(stream));
  if (ce != cudaSuccess) {
    delete h;
    return VBDR_ECUDA;
  }
  p.regmax = regmax_of(h, p.tick);  // the buffer the next slide writes
  in.launches = 1;
  *out = h;
  return VBDR_OK;
}

vbdr_status vbdr_destroy(vbdr_t *h) {
  if (!h) return VBDR_EINVAL;
  if (h->copy_stream) {
    cudaStreamSynchronize(h->copy_stream);
    cudaStreamDestroy(h->copy_stream);
  }
  for (int i = 0; i < 2; ++i) {
    if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    if (h->ev_scanned[i]) cudaEventDestroy(h->ev_scanned[i]);
  }
  if (h->ev_hosts_in) cudaEventDestroy(h->ev_hosts_in);
  if (h->ev_hosts_free) cudaEventDestroy(h->ev_hosts_free);
  delete h;
  return VBDR_OK;
}

vbdr_status vbdr_info(const vbdr_t *h, vbdr_info_t *info) {
  if (!h || !info) return VBDR_EINVAL;
  *info = h->info;
  info->tick = h->p.tick;
  // the register buffer of the closed tick, and the one the next slide writes
  info->off_regmax = h->info.off_regmax + ((h->p.tick - 1u) & 1u) * h->regmax_stride;
  info->off_regmax_next = h->info.off_regmax + (h->p.tick & 1u) * h->regmax_stride;
  return VBDR_OK;
}

vbdr_status vbdr_scan_slice(vbdr_t *h, const uint32_t *d_pairs, uint64_t n_pairs, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (n_pairs == 0) return VBDR_OK;  // an empty batch still leaves the slice open
  if (!d_pairs || (reinterpret_cast<uintptr_t>(d_pairs) & 15u))
    return fail(h, VBDR_EINVAL, "d_pairs must be a 16-byte aligned device pointer");
  if (vbdr_status s = check_async(h, "before scan")) return s;
  const cudaError_t e = h->stamps
                            ? vbdr_launch::scan_stamps(h->p, scan_mode(h), d_pairs, n_pairs, S(stream))
                            : vbdr_launch::scan(h->p, h->fast, scan_mode(h), d_pairs, n_pairs,
                                                S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "scan launch");
  h->info.launches += scan_launches(h, n_pairs);
  return VBDR_OK;
}

// A register-sharded handle only holds the DRV of [drv_j0, drv_j0 + drv_n).
bool drv_covers(const vbdr *h, uint64_t j0, uint64_t j1) {
  return j0 >= h->p.drv_j0 && j1 <= h->p.drv_j0 + h->p.drv_n;
}

vbdr_status vbdr_slide(vbdr_t *h, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (h->p.drv_n != h->p.n_phys)
    return fail(h, VBDR_ESTATE, "a register-sharded handle closes slices with slide_delta");
  if (vbdr_status s = check_async(h, "before slide")) return s;
  const cudaError_t e = h->stamps ? vbdr_launch::slide_stamps(h->p, S(stream))
                                 : vbdr_launch::slide(h->p, h->fast, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "slide launch");
  return after_slide(h, stream);
}

vbdr_status vbdr_debug_set_tick(vbdr_t *h, uint32_t tick) {
  if (!h) return VBDR_EINVAL;
  if (h->info.slices_closed != 0 || h->p.tick != 1)
    return fail(h, VBDR_ESTATE, "the tick can only be set on a fresh pool");
  if (tick < 1 || tick >= kTickLimit || (tick & 3u) != 1u)
    return fail(h, VBDR_EINVAL, "tick must be 1 mod 4 and in [1, 2^26)");
  h->p.tick = tick;  // fresh pool: every stamp is 0 < tick, buffers / slots rotation kept
  h->p.regmax = regmax_of(h, tick);
  return VBDR_OK;
}

vbdr_status vbdr_stamp_delta(vbdr_t *h, uint8_t *d_delta, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (!h->fast) return fail(h, VBDR_ESTATE, "stamp deltas exist only in layout fast");
  if (!d_delta || (reinterpret_cast<uintptr_t>(d_delta) & 15u))
    return fail(h, VBDR_EINVAL, "d_delta must be a 16-byte aligned device pointer");
  if (vbdr_status s = check_async(h, "before stamp_delta")) return s;
  const cudaError_t e = vbdr_launch::delta(h->p, d_delta, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "stamp_delta launch");
  h->info.launches += 1;
  return VBDR_OK;
}

vbdr_status vbdr_sparse_extract(vbdr_t *h, uint32_t n_owners, uint32_t *d_records,
                                uint64_t cap, uint64_t *d_counts, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (!h->fast) return fail(h, VBDR_ESTATE, "sparse records exist only in layout fast");
  if (n_owners < 1 || h->p.n_phys % n_owners || (h->p.n_phys / n_owners) % 4)
    return fail(h, VBDR_EINVAL, "n_owners must divide n_phys into shards of multiples of 4");
  if (h->p.n_phys / n_owners > (1ull << 27))
    return fail(h, VBDR_EINVAL, "shards above 2^27 BDRs do not fit a 32-bit record");
  if (!d_counts || (cap && !d_records))
    return fail(h, VBDR_EINVAL, "null d_counts / d_records");
  if (vbdr_status s = check_async(h, "before sparse_extract")) return s;
  const cudaError_t e = vbdr_launch::sparse_extract(
      h->p, n_owners, d_records, cap, reinterpret_cast<unsigned long long *>(d_counts), S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "sparse_extract launch");
  h->info.launches += 1;
  return VBDR_OK;
}

vbdr_status vbdr_sparse_apply(vbdr_t *h, const uint32_t *d_records, uint64_t n_records,
                              uint8_t *d_delta_shard, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (!h->fast) return fail(h, VBDR_ESTATE, "sparse records exist only in layout fast");
  if ((n_records && !d_records) || !d_delta_shard ||
      (reinterpret_cast<uintptr_t>(d_delta_shard) & 3u))
    return fail(h, VBDR_EINVAL, "need records and a 4-byte aligned delta shard");
  if (vbdr_status s = check_async(h, "before sparse_apply")) return s;
  const cudaError_t e = vbdr_launch::sparse_apply(d_records, n_records, d_delta_shard, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "sparse_apply launch");
  h->info.launches += n_records ? 1 : 0;
  return VBDR_OK;
}

vbdr_status vbdr_slide_delta(vbdr_t *h, const uint8_t *d_delta, uint64_t j0, uint64_t j1,
                             void *stream) {
  if (!h) return VBDR_EINVAL;
  if (!h->fast) return fail(h, VBDR_ESTATE, "slide_delta exists only in layout fast");
  if (!d_delta || (reinterpret_cast<uintptr_t>(d_delta) & 3u) || j0 >= j1 || j1 > h->p.n_phys ||
      (j0 & 3u) || (j1 & 3u))
    return fail(h, VBDR_EINVAL, "need a 4-byte aligned delta and 0 <= j0 < j1 <= n_phys, both multiples of 4");
  if (!drv_covers(h, j0, j1))
    return fail(h, VBDR_EINVAL, "[j0, j1) outside this handle's DRV shard");
  if (vbdr_status s = check_async(h, "before slide_delta")) return s;
  const cudaError_t e = vbdr_launch::slide_delta(h->p, d_delta, j0, j1, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "slide_delta launch");
  return after_slide(h, stream);
}

vbdr_status vbdr_slide_peers(vbdr_t *h, const uint8_t *const *h_peer_delta, uint32_t n_peers,
                             uint64_t j0, uint64_t j1, uint8_t *const *h_peer_regmax,
                             uint64_t *const *h_peer_acc, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (!h->fast) return fail(h, VBDR_ESTATE, "slide_peers exists only in layout fast");
  if (!h_peer_delta || n_peers < 1 || n_peers > (uint32_t)vbdr_launch::kMaxPeers || j0 >= j1 ||
      j1 > h->p.n_phys || (j0 & 3u) || (j1 & 3u))
    return fail(h, VBDR_EINVAL, "need 1..16 peer deltas and 0 <= j0 < j1 <= n_phys, multiples of 4");
  if (!drv_covers(h, j0, j1))
    return fail(h, VBDR_EINVAL, "[j0, j1) outside this handle's DRV shard");
  vbdr_launch::Peers pe{};
  pe.n = n_peers;
  for (uint32_t r = 0; r < n_peers; ++r) {
    if (!h_peer_delta[r] || (reinterpret_cast<uintptr_t>(h_peer_delta[r]) & 15u))
      return fail(h, VBDR_EINVAL, "peer deltas must be 16-byte aligned device pointers");
    pe.delta[r] = h_peer_delta[r];
    if (h_peer_regmax) {
      if (!h_peer_regmax[r]) return fail(h, VBDR_EINVAL, "null peer regmax");
      pe.regmax[r] = h_peer_regmax[r];
    }
    if (h_peer_acc) {
      if (!h_peer_acc[r]) return fail(h, VBDR_EINVAL, "null peer accumulator");
      pe.acc[r] = reinterpret_cast<unsigned long long *>(h_peer_acc[r]);
    }
  }
  pe.n_regmax = h_peer_regmax ? n_peers : 0;
  pe.n_acc = h_peer_acc ? n_peers : 0;
  if (h_peer_regmax) {  // the local entry must be the buffer this slide writes (off_regmax_next)
    bool own = false;
    for (uint32_t r = 0; r < n_peers; ++r) own = own || pe.regmax[r] == h->p.regmax;
    if (!own)
      return fail(h, VBDR_EINVAL,
                  "h_peer_regmax holds no pointer to this handle's next register buffer "
                  "(vbdr_info off_regmax_next)");
  }
  if (vbdr_status s = check_async(h, "before slide_peers")) return s;
  const cudaError_t e = vbdr_launch::slide_peers(h->p, pe, j0, j1, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "slide_peers launch");
  return after_slide(h, stream);
}

vbdr_status vbdr_slide_multicast(vbdr_t *h, void *d_mc_state, uint64_t j0, uint64_t j1,
                                 void *stream) {
  if (!h) return VBDR_EINVAL;
  if (!d_mc_state || (reinterpret_cast<uintptr_t>(d_mc_state) & 255u) || j0 >= j1 ||
      j1 > h->p.n_phys || (j0 & 3u) || (j1 & 3u))
    return fail(h, VBDR_EINVAL,
                "need a 256-byte aligned multicast state address and 0 <= j0 < j1 <= n_phys, "
                "both multiples of 4");
  if (h->stamps) return fail(h, VBDR_ESTATE, "slide_multicast: layouts fast and packed only");
  if (h->fast ? !drv_covers(h, j0, j1) : h->cfg.drv_shards > 1)
    return fail(h, VBDR_EINVAL, h->fast ? "[j0, j1) outside this handle's DRV shard"
                                        : "layout packed keeps a full DRV replica per rank");
  // the multicast object maps every rank's state buffer, laid out like this one
  uint8_t *mc = static_cast<uint8_t *>(d_mc_state);
  const uint8_t *base = reinterpret_cast<const uint8_t *>(h->p.acc) - h->info.off_acc;
  vbdr_launch::Peers pe{};
  // a group of one without a multicast object: the handle's own state
  pe.nvls = mc == base ? 2u : 1u;
  pe.sr_mc = h->fast ? reinterpret_cast<const uint32_t *>(mc + h->info.off_sr) : nullptr;
  pe.drv_mc = h->fast ? nullptr : reinterpret_cast<uint32_t *>(mc + h->info.off_drv);
  pe.regmax_mc = mc + (h->p.regmax - base);  // the buffer this slide writes
  pe.acc_mc = reinterpret_cast<unsigned long long *>(mc + h->info.off_acc);
  if (vbdr_status s = check_async(h, "before slide_multicast")) return s;
  const cudaError_t e = vbdr_launch::slide_multicast(h->p, pe, j0, j1, h->fast, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "slide_multicast launch");
  return after_slide(h, stream);
}

vbdr_status vbdr_select_above(vbdr_t *h, const double *d_est, uint64_t n, double threshold,
                              uint32_t *d_idx, uint64_t *d_count, void *stream) {
  if (!h || (n && (!d_est || !d_idx)) || !d_count) return VBDR_EINVAL;
  if (n > 0xFFFFFFFFull) return fail(h, VBDR_ERANGE, "at most 2^32 - 1 hosts");
  if (vbdr_status s = check_async(h, "before select_above")) return s;
  const cudaError_t e = vbdr_launch::select_above(
      d_est, n, threshold, d_idx, reinterpret_cast<unsigned long long *>(d_count), S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "select_above");
  h->info.launches += n ? 1 : 0;
  return VBDR_OK;
}

// Sorted plan (k_splan.cu): P host groups x C register ranges over the SMs,
// the group's accumulators in shared memory; the largest C (fewest reads of
// the register array) whose accumulators fit.
struct SpGeom {
  uint32_t ctas, C, P, hpg, SB, range_log2, seg_log2, nseg;
  uint64_t nbuckets, nkeys, off_offs, off_segtot, off_segbase, off_part, off_gcount, off_misc,
      off_lct, off_entries, bytes;
};

bool sp_geom(const vbdr *h, uint64_t n_hosts, SpGeom *g) {
  const uint64_t z = h->p.n_phys;
  if (n_hosts == 0 || z < 128) return false;
  const uint64_t smax =
      (uint64_t)h->cfg.m * (h->cfg.estimator == 0 ? 1ull << (h->p.L - 1) : 255ull);
  if (smax >> 32) return false;  // S' per host accumulates in a u32
  int sms = 0, dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (sms <= 0) sms = 148;
  if (optin <= 0) optin = 227 * 1024;
  const uint64_t budget = (uint64_t)optin - 64;  // static shared memory of the kernel
  for (uint32_t C = 4; C >= 1; C >>= 1) {
    if ((uint32_t)sms % C || z / C < 128) continue;
    const uint32_t P = (uint32_t)sms / C;
    const uint64_t hpg = (n_hosts + P - 1) / P;
    uint32_t SB = 1;
    while ((1ull << SB) < hpg + 32) ++SB;
    const uint32_t range_log2 = log2u(z / C);
    uint32_t seg_log2 = 32u - SB < range_log2 ? 32u - SB : range_log2;
    if (seg_log2 < vbdr_launch::kSpLineLog2) continue;
    const uint64_t nseg = 1ull << (range_log2 - seg_log2);
    if (vbdr_launch::sp_smem_bytes((uint32_t)hpg, (uint32_t)nseg) > budget) continue;
    const uint64_t nkeys = (uint64_t)sms * nseg;
    if (n_hosts * h->cfg.m + 31 * nkeys >= (1ull << 32)) return false;  // u32 entry offsets
    g->ctas = (uint32_t)sms;
    g->C = C;
    g->P = P;
    g->hpg = (uint32_t)hpg;
    g->SB = SB;
    g->range_log2 = range_log2;
    g->seg_log2 = seg_log2;
    g->nseg = (uint32_t)nseg;
    g->nkeys = nkeys;
    g->nbuckets = (uint64_t)sms << (range_log2 - vbdr_launch::kSpLineLog2);
    uint64_t off = 0;
    auto take = [&](uint64_t bytes) {
      const uint64_t o = off;
      off = align256(off + bytes);
      return o;
    };
    g->off_offs = take(4 * g->nbuckets);
    g->off_segtot = take(4 * nkeys);
    g->off_segbase = take(4 * (nkeys + 1));
    g->off_part = take(C > 1 ? 8ull * sms * hpg : 8);
    g->off_gcount = take(4ull * P);
    g->off_misc = take(64);
    g->off_lct = take(8ull * (h->cfg.m + 1));
    g->off_entries = take(4 * (n_hosts * h->cfg.m + 31 * nkeys));
    g->bytes = off;
    return true;
  }
  return false;
}

vbdr_launch::PlanLayout sp_layout(const SpGeom &g, void *d_plan, uint64_t n_hosts) {
  uint8_t *b = static_cast<uint8_t *>(d_plan);
  vbdr_launch::PlanLayout pl{};
  pl.kind = 2;
  pl.ctas = g.ctas;
  pl.n_hosts = n_hosts;
  pl.counts = reinterpret_cast<uint32_t *>(b + g.off_offs);
  pl.range_size = reinterpret_cast<uint32_t *>(b + g.off_segtot);
  pl.sp_segbase = reinterpret_cast<uint32_t *>(b + g.off_segbase);
  pl.sp_part = reinterpret_cast<unsigned long long *>(b + g.off_part);
  pl.sp_gcount = reinterpret_cast<uint32_t *>(b + g.off_gcount);
  pl.error = reinterpret_cast<unsigned long long *>(b + g.off_misc);
  pl.lct = reinterpret_cast<const double *>(b + g.off_lct);
  pl.entries = reinterpret_cast<uint32_t *>(b + g.off_entries);
  pl.sp_C = g.C;
  pl.sp_hpg = g.hpg;
  pl.sp_nseg = g.nseg;
  pl.sp_SB = g.SB;
  pl.sp_seg_log2 = g.seg_log2;
  pl.sp_range_log2 = g.range_log2;
  return pl;
}

// Pass-id plan (k_estimate.cu) for pools the staged plan cannot take whose
// gather estimate runs in 2..4 passes: a copy of the host list, then 16 bytes
// per (host, lane), g / 64 lanes per host.
struct PassPlanGeom {
  uint32_t passes, lanes;
  uint64_t off_hosts, off_pid, bytes;
};

bool passplan_geom(const vbdr *h, uint64_t n_hosts, PassPlanGeom *g) {
  const uint64_t z = h->p.n_phys;
  if (z <= (1ull << 22) || n_hosts == 0) return false;
  const uint32_t g_regs = h->cfg.m;
  if (g_regs < 64 || g_regs / 64 > 32) return false;
  const uint32_t log2z = log2u(z), pl2 = est_params(h).pass_log2;
  if (pl2 >= log2z || log2z - pl2 > 2) return false;  // 2..4 passes
  g->passes = 1u << (log2z - pl2);
  g->lanes = vbdr_launch::passplan_lanes(g_regs);
  g->off_hosts = 0;
  g->off_pid = align256(4 * n_hosts);
  g->bytes = align256(g->off_pid + 16ull * n_hosts * g->lanes);
  return true;
}

// Which plan a request gets: internal kind 2 (sorted), 0 (staged) or 1
// (pass ids), or -1.  VBDR_PLAN_AUTO takes the first that fits in that order.
int choose_plan(const vbdr *h, uint64_t n_hosts, uint32_t want, PlanGeom *g, PassPlanGeom *pg,
                SpGeom *sg) {
  // AUTO: the staged plan when its gathers outnumber the registers it streams
  // through every SM (caida: 16 per register, 82 vs ~100 us for the sorted
  // plan; profiles/r02_sorted_plan.txt), else the sorted plan, else pass ids
  if (want == VBDR_PLAN_AUTO && n_hosts * h->cfg.m >= h->p.n_phys && plan_geom(h, n_hosts, g))
    return 0;
  if ((want == VBDR_PLAN_AUTO || want == VBDR_PLAN_SORTED) && sp_geom(h, n_hosts, sg)) return 2;
  if ((want == VBDR_PLAN_AUTO || want == VBDR_PLAN_STAGED) && plan_geom(h, n_hosts, g)) return 0;
  if ((want == VBDR_PLAN_AUTO || want == VBDR_PLAN_PASSID) && passplan_geom(h, n_hosts, pg)) return 1;
  return -1;
}

vbdr_status vbdr_plan_bytes_kind(const vbdr_t *h, uint64_t n_hosts, uint32_t kind, uint64_t *bytes) {
  if (!h || !bytes || kind > VBDR_PLAN_SORTED) return VBDR_EINVAL;
  PlanGeom g;
  PassPlanGeom pg;
  SpGeom sg;
  *bytes = 0;
  switch (choose_plan(h, n_hosts, kind, &g, &pg, &sg)) {
    case 2: *bytes = sg.bytes; break;
    case 0: *bytes = g.bytes; break;
    case 1: *bytes = pg.bytes; break;
    default: return VBDR_ERANGE;
  }
  return VBDR_OK;
}

vbdr_status vbdr_plan_bytes(const vbdr_t *h, uint64_t n_hosts, uint64_t *bytes) {
  return vbdr_plan_bytes_kind(h, n_hosts, VBDR_PLAN_AUTO, bytes);
}

vbdr_status vbdr_plan_build_kind(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts,
                                 uint32_t kind, void *d_plan, uint64_t bytes, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (kind > VBDR_PLAN_SORTED) return fail(h, VBDR_EINVAL, "unknown plan kind");
  PlanGeom g;
  PassPlanGeom pg;
  SpGeom sg;
  const int which = choose_plan(h, n_hosts, kind, &g, &pg, &sg);
  if (which < 0) return fail(h, VBDR_ERANGE, "no plan of this kind for this pool / host count");
  if (which == 2) {
    if (!d_hosts || !d_plan || (reinterpret_cast<uintptr_t>(d_plan) & 255u))
      return fail(h, VBDR_EINVAL, "d_hosts and a 256-byte aligned d_plan are required");
    if (bytes < sg.bytes) return fail(h, VBDR_ENOMEM, "plan buffer too small");
    if (vbdr_status s = check_async(h, "before plan_build")) return s;
    cudaStream_t cs = S(stream);
    const vbdr_launch::PlanLayout pl = sp_layout(sg, d_plan, n_hosts);
    cudaError_t e = vbdr_launch::sp_build(pl, d_hosts, n_hosts, h->cfg.m, h->p.A0, h->p.mask,
                                          pl.error, cs);
    if (e == cudaSuccess)
      e = vbdr_launch::sp_fill(pl, d_hosts, n_hosts, h->cfg.m, h->p.A0, h->p.mask, cs);
    if (e == cudaSuccess) e = vbdr_launch::plan_lct(pl.lct, h->cfg.m, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) return cuda_fail(h, e, "plan_build");
    h->info.launches += 5;
    h->plans[d_plan] = pl;
    return VBDR_OK;
  }
  if (which == 1) {
    if (!d_hosts || !d_plan || (reinterpret_cast<uintptr_t>(d_plan) & 255u))
      return fail(h, VBDR_EINVAL, "d_hosts and a 256-byte aligned d_plan are required");
    if (bytes < pg.bytes) return fail(h, VBDR_ENOMEM, "plan buffer too small");
    if (vbdr_status s = check_async(h, "before plan_build")) return s;
    cudaStream_t cs = S(stream);
    uint8_t *b = static_cast<uint8_t *>(d_plan);
    vbdr_launch::PlanLayout pl{};
    pl.kind = 1;
    pl.n_hosts = n_hosts;
    pl.hosts = reinterpret_cast<uint32_t *>(b + pg.off_hosts);
    pl.pid = b + pg.off_pid;
    pl.passes = pg.passes;
    cudaError_t e = cudaMemcpyAsync(pl.hosts, d_hosts, 4 * n_hosts, cudaMemcpyDeviceToDevice, cs);
    if (e == cudaSuccess)
      e = vbdr_launch::passplan_build(d_hosts, n_hosts, h->cfg.m, h->p.A0, h->p.mask,
                                      est_params(h).pass_log2, pl.pid, cs);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) return cuda_fail(h, e, "plan_build");
    h->info.launches += 1;
    h->plans[d_plan] = pl;
    return VBDR_OK;
  }
  if (!d_hosts || !d_plan || (reinterpret_cast<uintptr_t>(d_plan) & 255u))
    return fail(h, VBDR_EINVAL, "d_hosts and a 256-byte aligned d_plan are required");
  if (bytes < g.bytes) return fail(h, VBDR_ENOMEM, "plan buffer too small");
  if (vbdr_status s = check_async(h, "before plan_build")) return s;
  const vbdr_launch::PlanLayout pl = plan_layout(g, d_plan, n_hosts);
  cudaStream_t cs = S(stream);
  cudaError_t e = vbdr_launch::plan_build(pl, d_hosts, n_hosts, h->cfg.m, h->p.A0, h->p.mask,
                                          pl.range_size, cs);
  uint32_t max_range = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&max_range, pl.max_range, 4, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "plan_build");
  h->info.launches += 6;
  if (max_range > vbdr_launch::plan_ent_cap(pl.block_log2)) {
    h->plans.erase(d_plan);
    return fail(h, VBDR_ERANGE, "a register block holds more entries than shared memory stages");
  }
  h->plans[d_plan] = pl;
  return VBDR_OK;
}

vbdr_status vbdr_plan_build(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts, void *d_plan,
                            uint64_t bytes, void *stream) {
  return vbdr_plan_build_kind(h, d_hosts, n_hosts, VBDR_PLAN_AUTO, d_plan, bytes, stream);
}

static vbdr_status estimate_with_plan(vbdr_t *h, const void *d_plan, double *d_out, uint64_t *d_S,
                                      uint32_t *d_V, void *stream) {
  if (!h) return VBDR_EINVAL;
  auto it = h->plans.find(d_plan);
  if (it == h->plans.end()) return fail(h, VBDR_EINVAL, "unknown plan (build it with this handle)");
  if (vbdr_status s = check_async(h, "before estimate_plan")) return s;
  const vbdr_launch::PlanLayout &pl = it->second;
  if (pl.kind == 2) {
    const cudaError_t e = vbdr_launch::estimate_sp(est_params(h), pl, pl.n_hosts, d_out,
                                                   reinterpret_cast<unsigned long long *>(d_S),
                                                   d_V, S(stream));
    if (e != cudaSuccess) return cuda_fail(h, e, "estimate_plan launch");
    h->info.launches += 1;
    return VBDR_OK;
  }
  if (pl.kind == 1) {
    const cudaError_t e = vbdr_launch::estimate_passplan(
        est_params(h), pl.hosts, pl.n_hosts, pl.pid, pl.passes, d_out,
        reinterpret_cast<unsigned long long *>(d_S), d_V, S(stream));
    if (e != cudaSuccess) return cuda_fail(h, e, "estimate_plan launch");
    h->info.launches += pl.passes;
    return VBDR_OK;
  }
  const cudaError_t e = vbdr_launch::estimate_plan(
      est_params(h), pl, pl.n_hosts, d_out, reinterpret_cast<unsigned long long *>(d_S), d_V,
      S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "estimate_plan launch");
  h->info.launches += 1;
  return VBDR_OK;
}

vbdr_status vbdr_estimate_plan(vbdr_t *h, const void *d_plan, double *d_out, void *stream) {
  if (!d_out) return fail(h, VBDR_EINVAL, "null d_out");
  return estimate_with_plan(h, d_plan, d_out, nullptr, nullptr, stream);
}

vbdr_status vbdr_estimate_plan_host(vbdr_t *h, const void *d_plan, double *d_out_stage,
                                    double *h_out, void *stream) {
  if (!h || !d_out_stage || !h_out) return VBDR_EINVAL;
  if (vbdr_status s = estimate_with_plan(h, d_plan, d_out_stage, nullptr, nullptr, stream)) return s;
  const uint64_t n = h->plans[d_plan].n_hosts;
  const cudaError_t e =
      cudaMemcpyAsync(h_out, d_out_stage, 8ull * n, cudaMemcpyDeviceToHost, S(stream));
  if (e != cudaSuccess) return cuda_fail(h, e, "estimate_plan_host");
  return VBDR_OK;
}

vbdr_status vbdr_host_sums_plan(vbdr_t *h, const void *d_plan, uint64_t *d_S, uint32_t *d_V,
                                void *stream) {
  if (!d_S || !d_V) return fail(h, VBDR_EINVAL, "null d_S / d_V");
  return estimate_with_plan(h, d_plan, nullptr, d_S, d_V, stream);
}

vbdr_status vbdr_plan_check(vbdr_t *h, const void *d_plan, void *stream) {
  if (!h) return VBDR_EINVAL;
  auto it = h->plans.find(d_plan);
  if (it == h->plans.end()) return fail(h, VBDR_EINVAL, "unknown plan");
  if (it->second.kind != 0) return VBDR_OK;  // pass ids / sorted: nothing is staged
  unsigned long long err = 0;
  cudaStream_t cs = S(stream);
  cudaError_t e = cudaMemcpyAsync(&err, it->second.error, 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "plan_check");
  if (err) return fail(h, VBDR_ECUDA, "a staged plan transfer timed out");
  return VBDR_OK;
}

vbdr_status vbdr_plan_release(vbdr_t *h, const void *d_plan) {
  if (!h) return VBDR_EINVAL;
  h->plans.erase(d_plan);
  return VBDR_OK;
}

vbdr_status vbdr_estimate(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts, double *d_out,
                          void *stream) {
  if (!h) return VBDR_EINVAL;
  if (n_hosts == 0) return VBDR_OK;
  if (!d_hosts || !d_out) return fail(h, VBDR_EINVAL, "null d_hosts/d_out");
  if (vbdr_status s = check_async(h, "before estimate")) return s;
  uint32_t nl = 0;
  const cudaError_t e = vbdr_launch::estimate(est_params(h), d_hosts, n_hosts, d_out, nullptr,
                                              nullptr, S(stream), &nl);
  if (e != cudaSuccess) return cuda_fail(h, e, "estimate launch");
  h->info.launches += nl;
  return VBDR_OK;
}

vbdr_status vbdr_host_sums(vbdr_t *h, const uint32_t *d_hosts, uint64_t n_hosts, uint64_t *d_S,
                           uint32_t *d_V, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (n_hosts == 0) return VBDR_OK;
  if (!d_hosts || !d_S || !d_V) return fail(h, VBDR_EINVAL, "null pointer");
  if (vbdr_status s = check_async(h, "before host_sums")) return s;
  uint32_t nl = 0;
  const cudaError_t e = vbdr_launch::estimate(est_params(h), d_hosts, n_hosts, nullptr,
                                              reinterpret_cast<unsigned long long *>(d_S), d_V,
                                              S(stream), &nl);
  if (e != cudaSuccess) return cuda_fail(h, e, "host_sums launch");
  h->info.launches += nl;
  return VBDR_OK;
}

vbdr_status vbdr_scan_slice_host(vbdr_t *h, const uint32_t *h_pairs, uint64_t n_pairs,
                                 uint32_t *d_stage, uint64_t stage_pairs, void *stream) {
  if (!h) return VBDR_EINVAL;
  if (n_pairs == 0) return VBDR_OK;
  if (!h_pairs || !d_stage || stage_pairs < 16 ||
      (reinterpret_cast<uintptr_t>(d_stage) & 15u))
    return fail(h, VBDR_EINVAL, "bad host pairs / staging buffer");
  cudaStream_t cs = S(stream);
  if (vbdr_status s = ensure_pipeline(h, cs)) return s;
  if (vbdr_status s = check_async(h, "before scan_host")) return s;
  // two halves of the staging buffer, each a multiple of 2 pairs (16 B)
  const uint64_t half = (stage_pairs / 2) & ~uint64_t(1);
  // A copy into a half waits only for the last scan that read that half
  // (ev_scanned, carried across calls): the host-to-device copies of the next
  // slice overlap this slice's slide and estimate.  Each chunk's scan waits
  // for its copy.
  cudaError_t e = cudaSuccess;
  uint64_t done = 0;
  for (uint64_t c = 0; done < n_pairs && e == cudaSuccess; ++c) {
    const int slot = (int)(c & 1u);
    const uint64_t cnt = (n_pairs - done) < half ? (n_pairs - done) : half;
    uint32_t *dst = d_stage + 2 * half * (uint64_t)slot;
    e = cudaStreamWaitEvent(h->copy_stream, h->ev_scanned[slot], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(dst, h_pairs + 2 * done, 8ull * cnt, cudaMemcpyHostToDevice,
                          h->copy_stream);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_copied[slot], h->copy_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, h->ev_copied[slot], 0);
    if (e == cudaSuccess) {
      e = h->stamps ? vbdr_launch::scan_stamps(h->p, scan_mode(h), dst, cnt, cs)
                    : vbdr_launch::scan(h->p, h->fast, scan_mode(h), dst, cnt, cs);
      h->info.launches += scan_launches(h, cnt);
    }
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_scanned[slot], cs);
    done += cnt;
  }
  if (e != cudaSuccess) return cuda_fail(h, e, "scan_host");
  return VBDR_OK;
}

vbdr_status vbdr_estimate_host(vbdr_t *h, const uint32_t *h_hosts, uint64_t n_hosts,
                               uint32_t *d_hosts_stage, double *d_out_stage, double *h_out,
                               void *stream) {
  if (!h) return VBDR_EINVAL;
  if (n_hosts == 0) return VBDR_OK;
  if (!h_hosts || !d_hosts_stage || !d_out_stage || !h_out)
    return fail(h, VBDR_EINVAL, "null pointer");
  cudaStream_t cs = S(stream);
  if (vbdr_status s = ensure_pipeline(h, cs)) return s;
  if (vbdr_status s = check_async(h, "before estimate_host")) return s;
  // The host ids travel on the copy stream like the pairs (all host-to-device
  // traffic in one FIFO, never queued behind compute); the estimate waits for
  // them, the next copy into the stage waits for the estimate that read it.
  cudaError_t e = cudaStreamWaitEvent(h->copy_stream, h->ev_hosts_free, 0);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_hosts_stage, h_hosts, 4ull * n_hosts, cudaMemcpyHostToDevice,
                        h->copy_stream);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_hosts_in, h->copy_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, h->ev_hosts_in, 0);
  uint32_t nl = 0;
  if (e == cudaSuccess)
    e = vbdr_launch::estimate(est_params(h), d_hosts_stage, n_hosts, d_out_stage, nullptr,
                              nullptr, cs, &nl);
  if (e == cudaSuccess) {
    h->info.launches += nl;
    e = cudaEventRecord(h->ev_hosts_free, cs);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h_out, d_out_stage, 8ull * n_hosts, cudaMemcpyDeviceToHost, cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "estimate_host");
  return VBDR_OK;
}

vbdr_status vbdr_export_ages(vbdr_t *h, uint16_t *h_ages, int mode, void *stream) {
  if (!h || !h_ages || (mode != 0 && mode != 1)) return VBDR_EINVAL;
  if (h->p.drv_n != h->p.n_phys)
    return fail(h, VBDR_ESTATE, "a register-sharded handle exports ages with export_ages_at");
  const uint64_t n = h->p.n_phys;
  const uint32_t W = h->p.W;
  std::vector<uint32_t> words;
  try {
    words.resize((size_t)(W * n));
  } catch (...) {
    return fail(h, VBDR_ENOMEM, "host buffer");
  }
  cudaStream_t cs = S(stream);
  cudaError_t e = cudaMemcpyAsync(words.data(), h->p.drv, 4ull * W * n, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "export_ages");
  for (uint64_t j = 0; j < n; ++j)
    decode_ages(h, [&](uint32_t w) { return words[(size_t)(w * n + j)]; }, mode,
                h_ages + j * h->p.L);
  return VBDR_OK;
}

vbdr_status vbdr_export_ages_at(vbdr_t *h, const uint64_t *d_idx, uint64_t n_idx,
                                uint32_t *d_scratch, uint16_t *h_ages, int mode, void *stream) {
  if (!h || (n_idx && (!d_idx || !d_scratch || !h_ages)) || (mode != 0 && mode != 1))
    return VBDR_EINVAL;
  if (n_idx == 0) return VBDR_OK;
  const uint32_t W = h->p.W;
  std::vector<uint32_t> words;
  try {
    words.resize((size_t)(W * n_idx));
  } catch (...) {
    return fail(h, VBDR_ENOMEM, "host buffer");
  }
  cudaStream_t cs = S(stream);
  cudaError_t e = vbdr_launch::gather_words(h->p, d_idx, n_idx, d_scratch, cs);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(words.data(), d_scratch, 4ull * W * n_idx, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "export_ages_at");
  h->info.launches += 1;
  for (uint64_t i = 0; i < n_idx; ++i)
    decode_ages(h, [&](uint32_t w) { return words[(size_t)(i * W + w)]; }, mode,
                h_ages + i * h->p.L);
  return VBDR_OK;
}

vbdr_status vbdr_export_regmax(vbdr_t *h, uint8_t *h_regmax, void *stream) {
  if (!h || !h_regmax) return VBDR_EINVAL;
  cudaStream_t cs = S(stream);
  cudaError_t e = cudaMemcpyAsync(h_regmax, regmax_of(h, h->p.tick - 1u), h->p.n_phys,
                                  cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "export_regmax");
  return VBDR_OK;
}

vbdr_status vbdr_export_pool_sums(vbdr_t *h, uint64_t *h_S_tot, uint64_t *h_V_tot, void *stream) {
  if (!h || !h_S_tot || !h_V_tot) return VBDR_EINVAL;
  const uint32_t closed = h->p.tick - 1u;
  unsigned long long v[2];
  cudaStream_t cs = S(stream);
  cudaError_t e = cudaMemcpyAsync(v, h->p.acc + 2 * (closed & 3u), sizeof v,
                                  cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return cuda_fail(h, e, "export_pool_sums");
  *h_S_tot = v[0];
  *h_V_tot = v[1];
  return VBDR_OK;
}

}  // extern "C"
