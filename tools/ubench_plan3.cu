// ubench_plan3.cu -- plan-based estimate, v3: warp-scheduled ROUNDS.
// Research microbenchmark (host-side scheduler; the product builds on the GPU).
//
// v2 (k_plan.cu) gives every thread its own run of entries: a warp iterates to
// the LONGEST run of its 32 lanes (Poisson tail, ~63 % lane efficiency) and
// every random table byte / accumulator costs ~3.5 bank-conflict wavefronts.
// v3 lets ANY lane of a warp serve any of the warp's 224 host slots: the plan
// packs the warp's entries of one phase into rounds of 32 (one per lane) with
// distinct hosts per round (so the read-modify-write of a u32 accumulator in
// shared memory is race-free) and, as far as the greedy scheduler manages,
// distinct table banks and accumulator banks per round.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                      \
    }                                                                               \
  } while (0)

#ifndef BLOCK_LOG2
#define BLOCK_LOG2 16
#endif
#ifndef SLACK
#define SLACK 0
#endif
#ifndef PIPE
#define PIPE 0
#endif
#ifndef WORDLD
#define WORDLD 0
#endif
#ifndef NOACC
#define NOACC 0
#endif
#ifndef ILP
#define ILP 0
#endif
#ifndef NOTAB
#define NOTAB 0
#endif
#ifndef NOENT
#define NOENT 0
#endif
#ifndef ACC64
#define ACC64 0
#endif
#ifndef ATOM
#define ATOM 0
#endif
#ifndef SCHED
#define SCHED 0
#endif
#ifndef SYNCW
#define SYNCW 1
#endif
#ifndef THREADS_
#define THREADS_ 512
#define SLOTS_ 7
#endif
constexpr int THREADS = THREADS_, WARPS = THREADS / 32, SLOTS = SLOTS_, BLOCK = 1 << BLOCK_LOG2;
constexpr int PHASES = (1 << 22) / BLOCK;
constexpr int ACC_W = SLOTS * 32 + 32;  // per warp: 224 host slots + 32 trash lanes
#ifndef ENT_CAP_
#define ENT_CAP_ (BLOCK_LOG2 == 16 ? 8192 : 4608)
#endif
constexpr int ENT_CAP = ENT_CAP_;
constexpr int STRIDE = (WARPS + 4) / 4 * 4;  // warp round starts per key (WARPS + 1 used), 16-byte padded

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

struct __align__(128) Smem {
  uint8_t tab[2][BLOCK];
  uint32_t ent[2][ENT_CAP];
  uint32_t start[2][STRIDE];
  uint32_t acc[WARPS][ACC_W];
#if ACC64
  unsigned long long acc64_[WARPS][ACC_W];
#endif
  uint64_t bar[2];
};

__global__ void __launch_bounds__(THREADS, 1)
k_plan3(const uint8_t *__restrict__ table, const uint32_t *__restrict__ entries,
        const uint32_t *__restrict__ starts, const uint32_t *__restrict__ range_base, uint32_t L,
        unsigned long long *out) {
  extern __shared__ __align__(128) uint8_t raw[];
  Smem &sm = *reinterpret_cast<Smem *>(raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = lane; i < ACC_W; i += 32) sm.acc[w][i] = 0u;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto bulk = [&](void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
  };
  auto issue = [&](int ph) {
    const int b = ph & 1;
    const size_t key = (size_t)blockIdx.x * PHASES + ph;
    const uint32_t e0 = range_base[key], e1 = range_base[key + 1];
    const uint32_t ebytes = (e1 - e0) * 4;
#if NOTAB
    const uint32_t tbytes = ph < 2 ? BLOCK : 0;  // experiment: table staged once per buffer
#else
    const uint32_t tbytes = BLOCK;
#endif
#if NOENT
    const uint32_t xbytes = ph < 2 ? ebytes : 0;  // experiment: entries staged once per buffer
#else
    const uint32_t xbytes = ebytes;
#endif
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&sm.bar[b])),
                 "r"(tbytes + xbytes + STRIDE * 4) : "memory");
    if (tbytes) bulk(sm.tab[b], table + (size_t)ph * BLOCK, BLOCK, &sm.bar[b]);
    if (xbytes) bulk(sm.ent[b], entries + e0, ebytes, &sm.bar[b]);
    bulk(sm.start[b], starts + key * STRIDE, STRIDE * 4, &sm.bar[b]);
  };
  if (tid == 0) issue(0);
  uint32_t *acc = sm.acc[w];
  uint32_t sink = 0;
#if ACC64
  unsigned long long *acc64 = sm.acc64_[w];
  for (int i = lane; i < ACC_W; i += 32) acc64[i] = 0ull;
#endif
  for (int ph = 0; ph < PHASES; ++ph) {
    const int b = ph & 1;
    if (tid == 0 && ph + 1 < PHASES) issue(ph + 1);
    const uint32_t parity = (ph >> 1) & 1;
    uint32_t done = 0;
    for (uint32_t spin = 0; !done; ++spin) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(done) : "r"(smem_u32(&sm.bar[b])), "r"(parity) : "memory");
      if (spin > (1u << 24)) { if (tid == 0) atomicAdd(out, 1ull << 40); return; }
    }
    const uint8_t *tab = sm.tab[b];
    const uint32_t r0 = sm.start[b][w], r1 = sm.start[b][w + 1];
    const uint32_t *ent = sm.ent[b] + lane;
#if PIPE
    // software pipeline: the entry and table loads of round r+1 are issued
    // before the accumulator update of round r (only the updates are ordered)
    if (r0 < r1) {
      uint32_t v = ent[r0 * 32];
      uint32_t M = tab[v & (BLOCK - 1)];
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t vn = r + 1 < r1 ? ent[(r + 1) * 32] : 0u;
        const uint32_t Mn = tab[vn & (BLOCK - 1)];
        acc[v >> 16] += (1u << (L - M)) + ((uint32_t)(M == 0) << 24);
        __syncwarp();
        v = vn;
        M = Mn;
      }
    }
#elif ATOM && ILP
    // batches of ILP rounds: all loads first, then the atomics
    uint32_t r = r0;
    for (; r + ILP <= r1; r += ILP) {
      uint32_t v[ILP], M[ILP];
#pragma unroll
      for (int j = 0; j < ILP; ++j) v[j] = ent[(r + j) * 32];
#if WORDLD
#pragma unroll
      for (int j = 0; j < ILP; ++j) {
        const uint32_t o = v[j] & (BLOCK - 1);
        M[j] = (reinterpret_cast<const uint32_t *>(tab)[o >> 2] >> ((o & 3) * 8)) & 0xFFu;
      }
#else
#pragma unroll
      for (int j = 0; j < ILP; ++j) M[j] = tab[v[j] & (BLOCK - 1)];
#endif
#pragma unroll
      for (int j = 0; j < ILP; ++j)
#if NOACC
        sink += (v[j] >> 16) ^ ((1u << (L - M[j])) + ((uint32_t)(M[j] == 0) << 24));
#else
        atomicAdd(&acc[v[j] >> 16], (1u << (L - M[j])) + ((uint32_t)(M[j] == 0) << 24));
#endif
    }
    for (; r < r1; ++r) {
      const uint32_t v = ent[r * 32];
      const uint32_t M = tab[v & (BLOCK - 1)];
      atomicAdd(&acc[v >> 16], (1u << (L - M)) + ((uint32_t)(M == 0) << 24));
    }
#elif ATOM
    // shared-memory atomics: no ordering between rounds needed
#pragma unroll 4
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t v = ent[r * 32];
      const uint32_t M = tab[v & (BLOCK - 1)];
#if ACC64
      atomicAdd(&acc64[v >> 16], (1ull << (L - M)) + ((unsigned long long)(M == 0) << 40));
#else
      atomicAdd(&acc[(v >> 16) & (NOENT ? 255u : 0xFFFFu)], (1u << (L - M)) + ((uint32_t)(M == 0) << 24));
#endif
    }
#else
    for (uint32_t r = r0; r < r1; ++r) {
      const uint32_t v = ent[r * 32];
      const uint32_t M = tab[v & (BLOCK - 1)];
      const uint32_t a = v >> 16;
      acc[a] += (1u << (L - M)) + ((uint32_t)(M == 0) << 24);
#if SYNCW
      __syncwarp();
#endif
    }
#endif
    __syncthreads();
  }
  unsigned long long t = sink;
  for (int i = lane; i < ACC_W; i += 32) t += sm.acc[w][i];
  if (t == 42) *out = t;
}

// ------------------------------------------------------------------ host
struct Ent { uint32_t off; uint16_t host; };

// Greedy: pass 1 places entries (most loaded table bank first) into the
// first of R rounds with a free lane, the host absent and both banks free;
// pass 2 places the rest where the host is absent at the least conflict.
static void schedule(std::vector<Ent> &es, std::vector<uint32_t> &out, int slack, double &wf) {
  const int n = (int)es.size();
  int R = std::max(1, (n + 31) / 32 + slack);
  std::vector<std::vector<uint32_t>> rounds(R);
#if SCHED == 4
  // per round: degree-ordered greedy with bank capacity 1, then 2, then 3
  // (atomics: a repeated host only costs a conflict)
  R = std::max(1, (n + 31) / 32);
  rounds.assign(R, {});
  {
    std::vector<Ent> rem(es);
    for (int r = 0; r < R; ++r) {
      const int target = std::min<int>(32, ((int)rem.size() + (R - r) - 1) / (R - r));
      int dt[32] = {0}, da[32] = {0};
      for (auto &e : rem) { dt[(e.off >> 2) & 31]++; da[e.host & 31]++; }
      std::vector<int> order(rem.size());
      for (size_t i = 0; i < rem.size(); ++i) order[i] = (int)i;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return dt[(rem[x].off >> 2) & 31] + da[rem[x].host & 31] >
               dt[(rem[y].off >> 2) & 31] + da[rem[y].host & 31];
      });
      std::vector<char> taken(rem.size(), 0);
      int ut[32] = {0}, ua[32] = {0}, cnt = 0;
      for (int cap = 1; cap <= 32 && cnt < target; ++cap)
        for (int i : order) {
          if (cnt >= target) break;
          if (taken[i]) continue;
          const int t = (rem[i].off >> 2) & 31, a = rem[i].host & 31;
          if (ut[t] < cap && ua[a] < cap) { taken[i] = 1; ut[t]++; ua[a]++; cnt++; }
        }
      std::vector<Ent> next;
      for (size_t i = 0; i < rem.size(); ++i)
        if (taken[i]) rounds[r].push_back(rem[i].off | (uint32_t)rem[i].host << 16);
        else next.push_back(rem[i]);
      rem.swap(next);
    }
  }
  if (false)
#elif SCHED == 3
  R = std::max(1, (n + 31) / 32);
  rounds.assign(R, {});
  for (int i = 0; i < n; ++i) rounds[i / 32].push_back(es[i].off | (uint32_t)es[i].host << 16);
  if (false)
#elif SCHED == 1
  // stripe: sorted by table bank, entry i -> round i mod R (atomics only)
  std::stable_sort(es.begin(), es.end(), [&](const Ent &x, const Ent &y) {
    return ((x.off >> 2) & 31) < ((y.off >> 2) & 31);
  });
  R = std::max(1, (n + 31) / 32);
  rounds.assign(R, {});
  for (int i = 0; i < n; ++i) rounds[i % R].push_back(es[i].off | (uint32_t)es[i].host << 16);
  if (false)
#endif
  {
  std::vector<std::vector<uint8_t>> hs(R, std::vector<uint8_t>(SLOTS * 32, 0));
  std::vector<uint32_t> T(R, 0), A(R, 0);
  int tl[32] = {0};
  for (auto &e : es) tl[(e.off >> 2) & 31]++;
  std::stable_sort(es.begin(), es.end(), [&](const Ent &x, const Ent &y) {
    return tl[(x.off >> 2) & 31] > tl[(y.off >> 2) & 31];
  });
  std::vector<Ent> left;
  for (auto &e : es) {
    const uint32_t tb = 1u << ((e.off >> 2) & 31), ab = 1u << (e.host & 31);
    bool ok = false;
    for (int r = 0; r < R && !ok; ++r) {
      if (rounds[r].size() >= 32 || hs[r][e.host] || (T[r] & tb) || (A[r] & ab)) continue;
      rounds[r].push_back(e.off | (uint32_t)e.host << 16);
      hs[r][e.host] = 1; T[r] |= tb; A[r] |= ab; ok = true;
    }
    if (!ok) left.push_back(e);
  }
  for (auto &e : left) {
    const uint32_t tb = 1u << ((e.off >> 2) & 31), ab = 1u << (e.host & 31);
    int best = -1, bc = 99;
    for (int r = 0; r < (int)rounds.size(); ++r) {
      if (rounds[r].size() >= 32 || hs[r][e.host]) continue;
      const int c = ((T[r] & tb) ? 1 : 0) + 2 * ((A[r] & ab) ? 1 : 0);
      if (c < bc) { bc = c; best = r; }
    }
    if (best < 0) {
      rounds.emplace_back(); hs.emplace_back(SLOTS * 32, 0); T.push_back(0); A.push_back(0);
      best = (int)rounds.size() - 1;
    }
    rounds[best].push_back(e.off | (uint32_t)e.host << 16);
    hs[best][e.host] = 1; T[best] |= tb; A[best] |= ab;
  }
  }
  for (auto &r : rounds) {
    // wavefront estimate: entry 1 + max table-bank multiplicity + 2 x acc-bank multiplicity
    int tm[32] = {0}, am[32] = {0}, mt = 0, ma = 0;
    std::vector<uint32_t> words;
    for (uint32_t v : r) {
      const uint32_t word = (v & 0xFFFF) >> 2;
      if (std::find(words.begin(), words.end(), word) == words.end()) {
        words.push_back(word);
        mt = std::max(mt, ++tm[word & 31]);
      }
      ma = std::max(ma, ++am[(v >> 16) & 31]);
    }
    wf += 1 + mt + 2 * ma;
    for (int l = 0; l < 32; ++l)
      out.push_back(l < (int)r.size() ? r[l] : (uint32_t)(SLOTS * 32 + l) << 16);
  }
}

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t table_bytes = (size_t)PHASES * BLOCK;
  uint8_t *table;
  CK(cudaMalloc(&table, table_bytes));
  std::vector<uint8_t> ht(table_bytes);
  for (size_t i = 0; i < table_bytes; ++i) ht[i] = (uint8_t)(1 + (i * 2654435761u >> 28) % 6);
  CK(cudaMemcpy(table, ht.data(), table_bytes, cudaMemcpyHostToDevice));
  // 500k hosts x 128 gathers over sms CTAs x 16 warps (host -> warp slot)
  const int H = 500000, G = 128;
  const size_t nkeys = (size_t)sms * PHASES;
  std::vector<uint32_t> range_base(nkeys + 1), starts(nkeys * STRIDE, 0), ent;
  ent.reserve(72u << 20);
  uint64_t rng = 88172645463325252ull;
  auto rnd = [&]() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; };
  const int T = sms * THREADS;
  double wf = 0;
  size_t maxrange = 0, nent = 0;
  for (int c = 0; c < sms; ++c) {
    // per (phase, warp) entry lists for this CTA
    std::vector<std::vector<Ent>> lists((size_t)PHASES * WARPS);
    for (int t = 0; t < THREADS; ++t)
      for (int s = 0; s < SLOTS; ++s) {
        const long h = (long)s * T + (long)c * THREADS + t;
        if (h >= H) continue;
        for (int i = 0; i < G; ++i) {
          const uint32_t p = (uint32_t)(rnd() & ((1u << 22) - 1));
          lists[(size_t)(p >> BLOCK_LOG2) * WARPS + t / 32].push_back(
              {p & (BLOCK - 1), (uint16_t)(s * 32 + (t & 31))});
          ++nent;
        }
      }
    for (int ph = 0; ph < PHASES; ++ph) {
      const size_t key = (size_t)c * PHASES + ph;
      range_base[key] = (uint32_t)ent.size();
      uint32_t rounds = 0;
      for (int w = 0; w < WARPS; ++w) {
        starts[key * STRIDE + w] = rounds;
        const size_t before = ent.size();
        schedule(lists[(size_t)ph * WARPS + w], ent, SLACK, wf);
        rounds += (uint32_t)((ent.size() - before) / 32);
      }
      starts[key * STRIDE + WARPS] = rounds;
      maxrange = std::max(maxrange, (size_t)rounds * 32);
    }
  }
  range_base[nkeys] = (uint32_t)ent.size();
  printf("block %d B, %d phases, %zu entries -> %zu slots (%.1f%% padding, %.1f MB), "
         "max per CTA-phase %zu (cap %d), est. %.2f wavefronts / 32 entries\n",
         BLOCK, PHASES, nent, ent.size(), 100.0 * (ent.size() - nent) / nent, ent.size() * 4e-6,
         maxrange, ENT_CAP, wf / nent * 32);
  if (maxrange > ENT_CAP) return 3;
  uint32_t *d_ent, *d_st, *d_rb;
  unsigned long long *out;
  CK(cudaMalloc(&d_ent, ent.size() * 4 + 64));
  CK(cudaMalloc(&d_st, starts.size() * 4));
  CK(cudaMalloc(&d_rb, range_base.size() * 4));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(out, 0, 8));
  CK(cudaMemcpy(d_ent, ent.data(), ent.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_st, starts.data(), starts.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rb, range_base.data(), range_base.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(k_plan3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem)));
  printf("smem %zu KB\n", sizeof(Smem) / 1024);
  void *flush;
  CK(cudaMalloc(&flush, 512u << 20));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaMemset(flush, rep, 512u << 20));
    CK(cudaEventRecord(e0));
    k_plan3<<<sms, THREADS, sizeof(Smem)>>>(table, d_ent, d_st, d_rb, 10, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    unsigned long long h;
    CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
    if (h >> 40) { printf("mbarrier timeout\n"); return 2; }
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("plan v3 (L2 flushed): %.3f ms = %.1f G entries/s\n", ms, nent / ms / 1e6);
  }
  return 0;
}
