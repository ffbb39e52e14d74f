// eval_thread.cu — K2t: one candidate per THREAD (32 candidates per warp).
//
// Same computation as eval.cu's one-candidate-per-warp K2 (Alg. 2's
// per-partition body, over the exact chain tables of
// R-FACT; readings R9-R18), restructured so that a warp instruction does
// useful work for 32 candidates instead of spreading one candidate's n slots
// over lanes: every per-slot / per-pipeline loop is a short sequential loop
// in one thread, with the thread's small arrays in shared memory at an odd
// word stride (lanes touching the same index hit distinct banks).  Each
// thread walks a run of consecutive candidate indices, carrying the
// composition from one lexicographic successor to the next.
//
// The dependency shift (R10) is evaluated per LEVEL of the sorted coarse
// multiset, not per slot: G_i is ascending, so among the slots whose needed
// position falls in one level the first one dominates, and the first slot
// reaching position p is found by walking a slot pointer over the sorted
// "thresholds" (the first slot each moved EF counts for).  Cost O(levels +
// moves) instead of O(n).
#include "optimus_dev.cuh"

namespace optimus {
namespace {

#ifndef K2T_THREADS
#define K2T_THREADS 128
#endif
constexpr int kTThreads = K2T_THREADS;
#ifndef K2T_RUN
#define K2T_RUN 32
#endif
constexpr int kTRun = K2T_RUN;            // most consecutive candidates per thread and claim
#ifndef K2T_MINRUN
#define K2T_MINRUN 1
#endif
constexpr int kTMinRun = K2T_MINRUN;      // fewest consecutive candidates per thread and claim
#ifndef K2T_GSS
#define K2T_GSS 1
#endif
#ifndef K2T_GSS_DEN
#define K2T_GSS_DEN 2  // claims of (remaining / 2 warps): the first claims of all warps take half the work, not all of it (config 4 K2: -4% on 1 rank, -17% at world 2)
#endif
constexpr int kTGss = K2T_GSS, kTGssDen = K2T_GSS_DEN;  // guided claim = remaining * GSS / (GSS_DEN * warps), capped
#ifndef K2T_MINB
#define K2T_MINB 6  // fast kernel: resident blocks per SM the register cap aims at (smem allows 6)
#endif
#ifndef K2T_GMINB
#define K2T_GMINB 5  // general kernel
#endif
#ifndef K2T_BIN_UNRANK
#define K2T_BIN_UNRANK 40  // unranking binary-searches a part when n - m + 1 exceeds this (16 measured 4% slower on config 3)
#endif
#ifndef K2T_MINB_WIDE
#define K2T_MINB_WIDE 5  // fast kernel of the n > 32 instances (small per-thread state: registers decide)
#endif
// per-thread scratch for n <= B slots and m <= BM pipelines, an odd number of
// words: (32, 32) 260 bytes; (64, 64) 516; (128, 64) 780; (128, 128) 1028;
// (64, 16) 364; (128, 16) 684 (at least N, c, the fast path's masks E[B + 2] and thresholds[B]; the
// general path's byte arrays; an odd number of words)
template <int B, int BM = B>
__host__ __device__ constexpr int tstride() {
  return ((4 * BM + 4 * B > 2 * BM + 5 * B + 8 ? 4 * BM + 4 * B : 2 * BM + 5 * B + 8) + 4) | 4;
}
// dynamic shared memory of a K2 mode 1 block: the per-thread scratch
template <int B, int BM>
__host__ __device__ constexpr int tsmem() { return kTThreads * tstride<B, BM>(); }
// the fast kernel's: the composition and the level masks only (16-bit masks
// when m <= 16), an odd number of words
template <int BM>
struct FMask {
  using T = uint32_t;
};
template <>
struct FMask<16> {
  using T = uint16_t;
};
template <int B, int BM>
__host__ __device__ constexpr int fstride() {
  return ((BM + (B + 2) * (int)sizeof(typename FMask<BM>::T) + 3) / 4 * 4) | 4;
}
template <int B, int BM>
__host__ __device__ constexpr int fsmem() { return kTThreads * fstride<B, BM>(); }
// the general kernel's: teval's byte arrays; the level masks only at B = 32
template <int B, int BM>
__host__ __device__ constexpr int gstride() { return B == 32 ? tstride<B, BM>() : (4 * BM + 4 * B + 4) | 4; }
template <int B, int BM>
__host__ __device__ constexpr int gsmem() { return kTThreads * gstride<B, BM>(); }

// Per-thread scratch (bytes 0..8B-1, B = 32 shown).  The three phases of one
// candidate use disjoint live sets, so bytes 2B..8B-1 are shared between them:
//   all      N[0..31] c[32..63]
//   forward  cnt[64..97] thr[98..129]
//   ordering seen[64..95] kb[96..127] mvj[128..159] mvk[160..191] own[192..223] rk[224..255]
//   backward cb[64..95] Qcb[96..127] own rk   (kb_j = N_j - cb_j is implied)
// K2 mode 1's dynamic shared memory: per-thread scratch, then the warps'
// general-path queues.  Scratch arrays are addressed by 32-bit offsets into
// it (SB), so every access is a shared-window LDS/STS wherever the view goes.
extern __shared__ __align__(16) unsigned char k2sm[];

struct SB {
  uint32_t o;  // byte offset in k2sm
  __device__ __forceinline__ uint8_t& operator[](int i) const { return k2sm[o + i]; }
  __device__ __forceinline__ uint32_t& w(int i) const { return reinterpret_cast<uint32_t*>(k2sm + o)[i]; }  // o % 4 == 0
  __device__ __forceinline__ SB operator+(int i) const { return SB{o + (uint32_t)i}; }
};

struct TS {
  SB N;     // composition N_j
  SB c;     // coarse (not yet moved) forward microbatches c_j
  SB cnt;   // cnt[t] = #{j : c_j >= t}, t = 1..n (cnt[n+1] = 0)
  SB thr;   // committed forward thresholds: first slot (1-based) each moved EF counts for, ascending
  SB own;   // owner pipeline of LLM microbatch slot i (global ordering)
  SB rk;    // rank of D_i within its owner's sorted deadlines
  SB cb;    // coarse backward microbatches per pipeline
  SB kb;    // ordering: slots given to each pipeline so far
  SB Qcb;   // Qcb[i] = #{owner's moved backward EF <= D_i}
  SB seen;  // ordering: active pipeline list
  SB mvj;   // ordering: moved entries sorted by (value, key): pipeline
  SB mvk;   //                                                  chain index
};

template <int B, int BM>
__device__ __forceinline__ TS ts_at(uint32_t b) {
  TS s;
  s.N = SB{b};                         // [BM]
  s.c = SB{b + BM};                    // [BM]
  const SB x{b + 2 * BM};              // phase-shared region
  s.cnt = x;                           // [B + 2]
  s.thr = x + B + 2;                   // [B]
  s.seen = x;                          // [BM]
  s.kb = x + BM;                       // [BM]
  s.mvj = x + 2 * BM;                  // [B]
  s.mvk = x + 2 * BM + B;              // [B]
  s.own = x + 2 * BM + 2 * B;          // [B]
  s.rk = x + 2 * BM + 3 * B;           // [B]
  s.cb = x;                            // [BM]
  s.Qcb = x + BM;                      // [B], ends before own
  return s;
}

#ifndef K2T_TV_OFF
struct TV {
  const int64_t* o;  // the table's address (32-bit offsets from Cfg::tables measured 1-2% slower)
};
#else
struct TV {
  uint32_t o;  // element offset in Cfg::tables
};
#endif

#ifndef K2T_TV_OFF
#define TVOF(x) TV{c.tables + (x)}
#else
#define TVOF(x) TV{(uint32_t)(x)}
#endif

struct TPlan {
  int e, P, rt, m, kmax, np1;
  unsigned rtm;            // row of pipeline j = (j * rtm) >> 16 (exact for j < 128, rt <= 128)
  bool strict;            // PRE_EF strictly increasing: pre entries order by (t, j)
  bool fast;              // strict and m <= 32: tfast (pipeline sets as 32-bit masks) applies
  uint64_t first, count;
  // the plan's tables as 32-bit element offsets from T (registers: one
  // pointer instead of ten)
  const int64_t* T;       // Cfg::tables
  TV preEF;               // PRE_EF(t), t = 0..n (row P-1 of PRE_F)
  TV preBEF;              // PREB_EF(t)
  TV devF, devB;
  TV kj;                  // findCritical keys per pipeline and count (PlanDesc::kj), u64
  TV inbF, bpF, lenF, inbB, lenB;
#ifndef K2T_TV_OFF
  __device__ __forceinline__ int64_t at(TV v, int i) const { return __ldg(&v.o[i]); }
  __device__ __forceinline__ const int64_t* ptr(TV v) const { return v.o; }
#else
  __device__ __forceinline__ int64_t at(TV v, int i) const { return __ldg(&T[v.o + i]); }
  __device__ __forceinline__ const int64_t* ptr(TV v) const { return T + v.o; }
#endif
};

__device__ __forceinline__ int row_of(const TPlan& p, int j) { return (int)(((unsigned)j * p.rtm) >> 16); }

__device__ void tplan(const Cfg& c, int e, TPlan& p) {
  const PlanDesc& d = c.plans[e];
  p.e = e;
  p.P = d.P;
  p.rt = d.rt;
  p.rtm = 65536u / (unsigned)d.rt + 1u;
  p.m = d.m;
  p.kmax = d.kmax;
  p.np1 = c.n + 1;
  p.first = d.first;
  p.count = d.count;
  p.T = c.tables;
  p.preEF = TVOF((d.preF + (int64_t)(d.P - 1) * (c.n + 1)));
  p.preBEF = TVOF((d.preB + (int64_t)(d.P - 1) * (c.n + 1)));
  p.devF = TVOF(d.devF);
  p.devB = TVOF(d.devB);
  p.kj = TVOF(d.kj);
  p.inbF = TVOF(d.inbF);
  p.bpF = TVOF(d.bpF);
  p.lenF = TVOF(d.lenF);
  p.inbB = TVOF(d.inbB);
  p.lenB = TVOF(d.lenB);
  p.strict = (__ldg(&c.tables[d.pflags]) & 1) != 0;
  p.fast = p.strict && d.m <= 32;
}

__device__ int tfind_plan(const Cfg& c, uint64_t g) {
  #pragma unroll 1
  for (int e = 0; e < c.E; ++e) {
    const PlanDesc& d = c.plans[e];
    if (d.count && g >= d.first && g < d.first + d.count) return e;
  }
  return -1;
}

// Lexicographic unranking (R17) into N[0..m); binomial rows of stride B + 1.
// Part j's value x is the smallest x whose cumulative count
// S(x) = sum_{y<=x} C(rem - y - 1, parts - 2) = C(rem - 1, parts - 1) - C(rem - x - 1, parts - 1)
// exceeds the rank (hockey stick): a linear scan over x when the range of x
// is short, a binary search on C(rem - x - 1, parts - 1) when it is long
// (large n, few pipelines: the scan's length differs from lane to lane).
// (plain loads: bt may be a shared-memory table)
template <typename T>
__device__ __forceinline__ void tunrank_t(const T* bt, int S, int n, int m, T r, TS& s) {
  int rem = n;
  const bool bin = n - m + 1 > K2T_BIN_UNRANK;
  #pragma unroll 1
  for (int j = 0; j < m - 1; ++j) {
    const int parts = m - j;
    int x = 1;
    if (!bin) {
      const T* row = bt + (parts - 2);
      #pragma unroll 1
      for (; x <= rem - (parts - 1); ++x) {
        const T cnt = row[(rem - x - 1) * S];
        if (r < cnt) break;
        r -= cnt;
      }
    } else {
      const T* col = bt + (parts - 1);
      const T tot = col[(rem - 1) * S];  // C(rem - 1, parts - 1)
      const T thr = tot - r;                     // find the smallest x with C(rem - x - 1, parts - 1) < thr
      int lo = 1, hi = rem - parts + 1;
      #pragma unroll 1
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (col[(rem - mid - 1) * S] < thr) hi = mid; else lo = mid + 1;
      }
      x = lo;
      r -= tot - col[(rem - x) * S];  // S(x - 1)
    }
    s.N[j] = (uint8_t)x;
    rem -= x;
  }
  s.N[m - 1] = (uint8_t)rem;
}

template <int B>
__device__ __forceinline__ void tunrank(const Cfg& c, const uint32_t* b32, const TPlan& p, int n, uint64_t rank, TS& s) {
  // plans of < 2^32 compositions: every count met is below 2^32 too (b32:
  // the 32-bit table, staged in shared memory by the B = 32 kernels)
  if (p.count <= 0xffffffffull)
    tunrank_t<uint32_t>(b32, B + 1, n, p.m, (uint32_t)rank, s);
  else
    tunrank_t<uint64_t>(c.binom, B + 1, n, p.m, rank, s);
}

// the kernels' 32-bit binomial table: staged in shared memory at B = 32 (33 x 33 words)
template <int B>
__device__ __forceinline__ const uint32_t* stage_binom32(const Cfg& c, uint32_t* sm) {
  if (B != 32) return c.binom32;
  for (int i = threadIdx.x; i < 33 * 33; i += blockDim.x) sm[i] = __ldg(&c.binom32[i]);
  return sm;
}

// Lexicographic successor of N (m parts); false past the last composition.
// A composition packed into 64 bits for k2_general's queue: N_j - 1 in
// kPackBits bits each, for m <= kPackParts (N_j <= B).
template <int B>
__host__ __device__ constexpr int kPackBits() { return B <= 32 ? 5 : B <= 64 ? 6 : 7; }
template <int B>
__host__ __device__ constexpr int kPackParts() { return 64 / kPackBits<B>(); }
template <int B>
__device__ __forceinline__ uint64_t tpack(const SB N, int m) {
  uint64_t v = 0;
#pragma unroll 1
  for (int j = m - 1; j >= 0; --j) v = v << kPackBits<B>() | (uint64_t)(N[j] - 1);
  return v;
}
template <int B>
__device__ __forceinline__ void tunpack(uint64_t v, int m, const SB N) {
#pragma unroll 1
  for (int j = 0; j < m; ++j, v >>= kPackBits<B>()) N[j] = (uint8_t)((v & ((1u << kPackBits<B>()) - 1u)) + 1u);
}

__device__ bool tnext(int m, TS& s) {
  if (m < 2) return false;
  const int last = s.N[m - 1];
  if (last > 1) {  // common step: one microbatch from part m-1 to part m-2
    s.N[m - 2] += 1;
    s.N[m - 1] = (uint8_t)(last - 1);
    return true;
  }
  int S = last, jj = m - 2;
  #pragma unroll 1
  for (; jj >= 0; --jj) {  // largest jj whose suffix can still give one away
    if (S > m - 1 - jj) break;
    S += s.N[jj];
  }
  if (jj < 0) return false;
  s.N[jj] += 1;
  int j = jj + 1;  // parts jj+1 .. m-2 become 1 (word stores where aligned; N is 4-byte aligned)
  #pragma unroll 1
  for (; j < m - 1 && (j & 3); ++j) s.N[j] = 1;
  #pragma unroll 1
  for (; j + 4 <= m - 1; j += 4) s.N.w(j >> 2) = 0x01010101u;
  #pragma unroll 1
  for (; j < m - 1; ++j) s.N[j] = 1;
  s.N[m - 1] = (uint8_t)(S - 1 - (m - 2 - jj));
  return true;
}

// Forward dependency shift (R10).  Slot i needs sorted pre position
// need_i = i - q(i), q(i) = #{thresholds <= i} (the M committed ones plus
// the trial one bp; n+1 = never); INF if some need_i > sum c; else the max
// over levels t of PRE_EF(t) - G_{s(t)}, s(t) = first slot reaching the
// level's first position (slots reaching later positions of the level have
// larger G).
__device__ __forceinline__ int64_t tdep_fwd(const TPlan& p, const int64_t* G, int n, int sumc, int bp, const TS& s,
                                            int M) {
  // max_i need_i: need rises by one per slot and drops by one per threshold
  int maxneed = 0;
  {
    int k = 0, q = 0;
    bool used = false;
    #pragma unroll 1
    for (;;) {
      const int a = k < M ? s.thr[k] : n + 1, b = used ? n + 1 : bp;
      const int nb = min(a, b);
      maxneed = max(maxneed, min(nb, n + 1) - 1 - q);
      if (nb > n) break;
      if (a <= b) ++k; else used = true;
      ++q;
    }
  }
  if (maxneed > sumc) return kInf;
  int64_t best = kNegInf;
  int i = 0, q = 0, k = 0;
  bool used = false;
  #pragma unroll 1
  for (int t = 1, pos = 0; pos < maxneed; ++t) {
    const int start = pos + 1;
    i = max(i, start + q);
    #pragma unroll 1
    for (;;) {  // thresholds up to slot i lower its need: move right
      const int a = k < M ? s.thr[k] : n + 1, b = used ? n + 1 : bp;
      if (min(a, b) > i) break;
      if (a <= b) ++k; else used = true;
      ++q;
      i = start + q;
    }
    best = max(best, p.at(p.preEF, t) - G[i - 1]);
    pos += s.cnt[t];
  }
  return best;
}

__device__ __forceinline__ void assign_slot(const int64_t* preBEF, const int64_t* D, const TS& s, int j, int& slot,
                                            int64_t& dep_b) {
  const int r = s.N[j] - s.kb[j];  // rank of this slot's deadline within pipeline j (R15)
  OPT_CHECK(slot < 128 && r >= 1 && r <= 128);
  s.kb[j] += 1;
  s.own[slot] = (uint8_t)j;
  s.rk[slot] = (uint8_t)r;
  dep_b = max(dep_b, __ldg(&preBEF[r]) - D[slot]);  // initial backward shift
  ++slot;
}

// Global ordering (R14), PRE_EF strict: pre entries (value PRE_EF(t) - Df,
// key (j, t-1)) come level by level in pipeline order (active pipelines
// compacted per level), merged with the moved EFs (INB_F[a_j][k], key
// (j, c_j + k)) sorted by (value, key).  Fills own[] / rk[]; returns the
// initial backward shift max_i PREB_EF(rk_i) - D_i.
__device__ int64_t order_strict(const TPlan& p, const int64_t* D, int m, int64_t Df, TS& s) {
  const int rt = p.rt, kmax = p.kmax;
  auto mval = [&](int q) { return p.at(p.inbF, row_of(p, s.mvj[q]) * kmax + s.mvk[q]); };
  auto mkey = [&](int q) { return ((int)s.mvj[q] << 8) | (s.c[s.mvj[q]] + s.mvk[q]); };
  int nm = 0;
  #pragma unroll 1
  for (int j = 0, a = 0, r = 0; j < m; ++j) {
    const int cj = s.c[j], kfj = s.N[j] - cj;
    s.kb[j] = 0;
    #pragma unroll 1
    for (int k = 0; k < kfj; ++k) {  // insertion sort of the moved entries
      const int64_t v = p.at(p.inbF, a * kmax + k);
      const int key = (j << 8) | (cj + k);
      int q = nm;
      while (q > 0) {
        const int64_t pv = mval(q - 1);
        if (pv < v || (pv == v && mkey(q - 1) < key)) break;
        s.mvj[q] = s.mvj[q - 1];
        s.mvk[q] = s.mvk[q - 1];
        --q;
      }
      s.mvj[q] = (uint8_t)j;
      s.mvk[q] = (uint8_t)k;
      ++nm;
    }
    if (++r == rt) { r = 0; ++a; }
  }
  const SB act = s.seen;
  int na = 0;
  #pragma unroll 1
  for (int j = 0; j < m; ++j)
    if (s.c[j] > 0) act[na++] = (uint8_t)j;
  int slot = 0, mi = 0;
  int64_t dep_b = kNegInf;
  int64_t mv = nm > 0 ? mval(0) : INT64_MAX;  // value of the next moved entry
  #pragma unroll 1
  for (int t = 1; na > 0; ++t) {
    const int64_t v = p.at(p.preEF, t) - Df;
    while (mv < v) {  // moved entries below this level's value precede all of it
      assign_slot(p.ptr(p.preBEF), D, s, s.mvj[mi], slot, dep_b);
      ++mi;
      mv = mi < nm ? mval(mi) : INT64_MAX;
    }
    int nn = 0;
    if (mv == v) {  // equal values: merge by key
      #pragma unroll 1
      for (int q = 0; q < na; ++q) {
        const int j = act[q];
        const int key = (j << 8) | (t - 1);
        while (mv == v && mkey(mi) < key) {
          assign_slot(p.ptr(p.preBEF), D, s, s.mvj[mi], slot, dep_b);
          ++mi;
          mv = mi < nm ? mval(mi) : INT64_MAX;
        }
        assign_slot(p.ptr(p.preBEF), D, s, j, slot, dep_b);
        if (s.c[j] > t) act[nn++] = (uint8_t)j;
      }
    } else {
      #pragma unroll 1
      for (int q = 0; q < na; ++q) {
        const int j = act[q];
        assign_slot(p.ptr(p.preBEF), D, s, j, slot, dep_b);
        if (s.c[j] > t) act[nn++] = (uint8_t)j;
      }
    }
    na = nn;
  }
  while (mi < nm) assign_slot(p.ptr(p.preBEF), D, s, s.mvj[mi++], slot, dep_b);
  return dep_b;
}

// Global ordering (R14) for any PRE_EF (levels of equal value grouped, so
// ties order by (j, t-1)); moved entries extracted in key order by repeated
// minimum search above the last key taken.
// (rare: only plans whose coarse EFs tie; out of line, with plain arguments so
// that the caller's plan and scratch views stay in registers)
__device__ __noinline__ int64_t order_general(const int64_t* preEF, const int64_t* preBEF, const int64_t* inbF, int rt,
                                              int kmax, const int64_t* D, int m, int64_t Df, bool moved, uint32_t oN,
                                              uint32_t oc, uint32_t okb, uint32_t oown, uint32_t ork) {
  TS s;
  s.N = SB{oN};
  s.c = SB{oc};
  s.kb = SB{okb};
  s.own = SB{oown};
  s.rk = SB{ork};
  struct {
    const int64_t *preEF, *preBEF, *inbF;
    __device__ __forceinline__ int64_t at(const int64_t* v, int i) const { return __ldg(&v[i]); }
    __device__ __forceinline__ const int64_t* ptr(const int64_t* v) const { return v; }
  } p{preEF, preBEF, inbF};
  int maxc = 0;
  #pragma unroll 1
  for (int j = 0; j < m; ++j) {
    maxc = max(maxc, (int)s.c[j]);
    s.kb[j] = 0;
  }
  int slot = 0;
  int64_t dep_b = kNegInf, lastv = kNegInf, mv = kInf;
  int lastk = -1, mk = 0, mj = -1;
  auto next_moved = [&]() {
    mv = kInf;
    mj = -1;
    if (!moved) return;
    #pragma unroll 1
    for (int j = 0, a = 0, r = 0; j < m; ++j) {
      const int cj = s.c[j], kfj = s.N[j] - cj;
      #pragma unroll 1
      for (int k = 0; k < kfj; ++k) {
        const int64_t v = p.at(p.inbF, a * kmax + k);
        const int key = (j << 8) | (cj + k);
        if ((v > lastv || (v == lastv && key > lastk)) && (v < mv || (v == mv && key < mk))) {
          mv = v;
          mk = key;
          mj = j;
        }
      }
      if (++r == rt) { r = 0; ++a; }
    }
  };
  next_moved();
  #pragma unroll 1
  for (int t1 = 1; t1 <= maxc;) {
    int t2 = t1;
    const int64_t pv = p.at(p.preEF, t1);
    while (t2 < maxc && p.at(p.preEF, t2 + 1) == pv) ++t2;
    const int64_t v = pv - Df;
    #pragma unroll 1
    for (int j = 0; j < m; ++j)
      #pragma unroll 1
      for (int t = t1; t <= min(t2, (int)s.c[j]); ++t) {
        const int key = (j << 8) | (t - 1);
        while (mj >= 0 && (mv < v || (mv == v && mk < key))) {
          assign_slot(p.ptr(p.preBEF), D, s, mj, slot, dep_b);
          lastv = mv;
          lastk = mk;
          next_moved();
        }
        assign_slot(p.ptr(p.preBEF), D, s, j, slot, dep_b);
        lastv = v;
        lastk = key;
      }
    t1 = t2 + 1;
  }
  while (mj >= 0) {
    assign_slot(p.ptr(p.preBEF), D, s, mj, slot, dep_b);
    lastv = mv;
    lastk = mk;
    next_moved();
  }
  return dep_b;
}

// Initial backward shift when no forward chain moved and PRE_EF is strict:
// the order is (t, j), slot of (t, j) gets rank N_j - t + 1; own/rk are not
// materialised.
__device__ __forceinline__ int64_t order_fast(const TPlan& p, const int64_t* D, int m, TS& s) {
  const SB actN = s.seen;  // N_j of the pipelines still active, in pipeline order
  #pragma unroll 1
  for (int j = 0; j < m; ++j) actN[j] = s.N[j];
  int na = m, pos = 0;
  int64_t best = kNegInf;
  #pragma unroll 1
  for (int t = 1; na > 0; ++t) {
    int nn = 0;
    #pragma unroll 1
    for (int q = 0; q < na; ++q) {
      const int Nj = actN[q];
      best = max(best, p.at(p.preBEF, Nj - t + 1) - D[pos++]);
      if (Nj > t) actN[nn++] = (uint8_t)Nj;
    }
    na = nn;
  }
  return best;
}

// Backward dependency shift (R15) after the ordering; trial pipeline js
// (-1: none) with trial chain end efb.
__device__ int64_t tdep_bwd(const TPlan& p, const int64_t* D, int n, int js, int64_t efb, const TS& s) {
  int64_t best = kNegInf;
  #pragma unroll 1
  for (int i = 0; i < n; ++i) {
    const int o = s.own[i];
    const int64_t d = D[i];
    const int cbo = s.cb[o] - (o == js ? 1 : 0);
    const int need = s.rk[i] - s.Qcb[i] - (o == js && efb <= d ? 1 : 0);
    if (need > cbo) return kInf;
    if (need > 0) best = max(best, p.at(p.preBEF, need) - d);
  }
  return best;
}

struct TStats {
  unsigned v[12];  // per-candidate loop counts (optimus_eval_stats); [8] fast path, [9] general path, [10] claims, [11] unranks
};

// decode a findCritical key: pipeline js and its DEV value (-inf, js = -1 if none)
__device__ __forceinline__ int64_t crit_value(const TPlan& p, TV dev, const SB cnt8, uint32_t best,
                                              int& js) {
  if (best < 128u) { js = -1; return kNegInf; }
  js = 127 - (int)(best & 127u);
  return p.at(dev, row_of(p, js) * p.np1 + cnt8[js]);
}

// findCritical (R11): argmax over pipelines with count > 0 of DEV[row][count],
// ties -> lowest j.  cnt8 = the per-pipeline counts.  Compares the 32-bit
// keys rank(DEV[row][count]) << 7 | (127 - j) (m <= 128): the max key is the
// max DEV at the lowest j; rank 0 (count 0) never wins over a count > 0.
__device__ __forceinline__ int64_t critical(const TPlan& p, TV dev, int half, const SB cnt8, int m,
                                            int& js) {
  const uint32_t* key = reinterpret_cast<const uint32_t*>(p.ptr(p.kj)) + half;  // KJ[j][c] word `half`
  const int np1 = p.np1;
  uint32_t best = 0;
#pragma unroll 2
  for (int j = 0; j < m; ++j) best = max(best, __ldg(&key[2 * (j * np1 + cnt8[j])]));
  return crit_value(p, dev, cnt8, best, js);
}

// the two largest forward keys over the pipelines' current counts
__device__ __forceinline__ void critical2(const TPlan& p, const SB cnt8, int m, uint32_t& k0, uint32_t& k1) {
  const uint32_t* key = reinterpret_cast<const uint32_t*>(p.ptr(p.kj));
  const int np1 = p.np1;
  uint32_t a = 0, b = 0;
#pragma unroll 2
  for (int j = 0; j < m; ++j) {
    const uint32_t k = __ldg(&key[2 * (j * np1 + cnt8[j])]);
    b = max(b, min(a, k));
    a = max(a, k);
  }
  k0 = a;
  k1 = b;
}

// One candidate, sequentially in this thread.
// EXPLAIN (NEXT-1, one candidate): xo[8 + t] = pipeline of the t-th committed
// forward move, xo[8 + n + t] = of the t-th backward move; xo[1..4] = Df, Db,
// forward / backward move counts.
// Forward dependency shift (R10) on 32-bit level masks (B = 32 instance):
// thresholds T_1 <= .. <= T_K (sorted bytes, n + 1 = never), levels from
// E[x] = {j : c_j = x} (E[0]: c_j = 0).  max_i need_i = max over k of
// T_k - k with T_{K+1} = n + 1; INF if that exceeds the coarse entries;
// else the level walk of tdep_fwd (first slot of a level: start + thresholds
// passed).
__device__ __forceinline__ int64_t tdep_mask(const TPlan& p, const int64_t* G, int n, int sumc, const uint32_t* E,
                                             uint32_t all, const SB thr, int K) {
  int maxneed = n - K;
#pragma unroll 1
  for (int k = 0; k < K; ++k) maxneed = max(maxneed, (int)thr[k] - (k + 1));
  if (maxneed > sumc) return kInf;
  int64_t best = kNegInf;
  uint32_t A = all & ~E[0];
  int k = 0;
#pragma unroll 1
  for (int t = 1, pos = 0; pos < maxneed; ++t) {
    int i = pos + 1 + k;
    while (k < K && (int)thr[k] <= i) { ++k; ++i; }
    OPT_CHECK(i >= 1 && i <= n && t <= n);
    best = max(best, p.at(p.preEF, t) - G[i - 1]);
    pos += __popc(A);
    A &= ~E[t];
  }
  return best;
}

// Global ordering (R14) and the initial backward shift for strict plans on
// level masks, when every moved entry sorts after every coarse one.  Coarse
// values PRE_EF(t) - Df rise with t, a pipeline's moved ones INB_F[a][k] with
// k: compare the largest coarse value with the smallest moved one; false if
// they may interleave.  Otherwise pipeline j's entries are its c_j coarse ones
// (level t: slot pos_t + |A_t below j|, rank N_j - t + 1) followed by its
// moved ones (slot sum c + place among the moved, rank kf_j - k).  D is
// non-increasing in the slot, so for a rank r > max kf the largest term is at
// the coarse entry of jmax (largest N, highest j) at level N_max - r + 1, and
// ranks r <= max kf are dominated by a moved entry of that rank.  E[x] =
// {j : c_j = x} (read only); mv (after E[max N]) receives the sorted moved
// entries.
__device__ __forceinline__ bool tsep(const TPlan& p, const int64_t* D, const TS& s, const uint32_t* E, uint32_t all,
                                     uint32_t MV, int maxN, int jmax, int sumc, int64_t Df, const SB mv, int64_t& dep_b) {
  const int kmax = p.kmax;
  int maxc = maxN;
#pragma unroll 1
  while (maxc > 0 && E[maxc] == 0u) --maxc;
  if (MV != 0u && maxc > 0) {
    const int64_t vpre = p.at(p.preEF, maxc) - Df;
#pragma unroll 1
    for (uint32_t b = MV; b; b &= b - 1)
      if (p.at(p.inbF, row_of(p, __ffs(b) - 1) * kmax) <= vpre) return false;
  }
  int maxkf = 0;
#pragma unroll 1
  for (uint32_t b = MV; b; b &= b - 1) {
    const int j = __ffs(b) - 1;
    maxkf = max(maxkf, (int)s.N[j] - (int)s.c[j]);
  }
  const uint32_t below = (1u << jmax) - 1u;
  uint32_t A = all & ~E[0];
  int64_t best = kNegInf;
#pragma unroll 1
  for (int u = 1, pos = 0; u <= maxN - maxkf; ++u) {
    OPT_CHECK(pos + __popc(A & below) < kMaxN && maxN - u + 1 >= 1);
    best = max(best, p.at(p.preBEF, maxN - u + 1) - D[pos + __popc(A & below)]);
    pos += __popc(A);
    A &= ~E[u];
  }
  // moved entries sorted by (value, key): inserted in (j, k) order, so a
  // stable insertion by value keeps key order among equal values (a single
  // moved pipeline's are already in order); kept as (j, k) byte pairs in mv
  // for the first backward trial (tbwd1)
  int nm = 0;
  const bool one = (MV & (MV - 1)) == 0u;
#pragma unroll 1
  for (uint32_t b = MV; b; b &= b - 1) {
    const int j = __ffs(b) - 1, a = row_of(p, j), kfj = (int)s.N[j] - (int)s.c[j];
#pragma unroll 1
    for (int k = 0; k < kfj; ++k) {
      int q = nm++;
      if (!one) {
        const int64_t v = p.at(p.inbF, a * kmax + k);
#pragma unroll 1
        for (; q > 0 && p.at(p.inbF, row_of(p, mv[2 * q - 2]) * kmax + mv[2 * q - 1]) > v; --q) {
          mv[2 * q] = mv[2 * q - 2];
          mv[2 * q + 1] = mv[2 * q - 1];
        }
      }
      mv[2 * q] = (uint8_t)j;
      mv[2 * q + 1] = (uint8_t)k;
    }
  }
#pragma unroll 1
  for (int q = 0; q < nm; ++q) {
    const int j = mv[2 * q];
    OPT_CHECK(sumc + q < kMaxN);
    best = max(best, p.at(p.preBEF, (int)s.N[j] - (int)s.c[j] - (int)mv[2 * q + 1]) - D[sumc + q]);
  }
  dep_b = best;
  return true;
}

// First backward trial (R13 in mirrored time, R15) on tsep's ordering: no
// backward move yet (Qcb = 0, cb = N), js gives one coarse backward
// microbatch whose chain ends at EFb.  Only js's entries change (need = rank -
// [EFb <= D]; INF if js's first entry, rank N_js, loses its cover).  The
// others' maximum: every moved entry of theirs, and their coarse entries of
// the ranks r > kf_o = their largest kf, whose largest slot is at jx (largest
// N among them, highest j) on level N_jx - r + 1 (smaller ranks are
// dominated by a moved entry of that rank, whose slot is later).
__device__ __forceinline__ int64_t tbwd1(const TPlan& p, const int64_t* D, const TS& s, const uint32_t* E,
                                         uint32_t all, const SB mv, int nm, int sumc, int m, int jmax, int js,
                                         int64_t EFb) {
  const int Njs = s.N[js], cjs = s.c[js];
  int64_t best = kNegInf;
  int kfo = 0;
#pragma unroll 1
  for (int q = 0; q < nm; ++q) {
    const int j = mv[2 * q], k = mv[2 * q + 1], kfj = (int)s.N[j] - (int)s.c[j];
    const int64_t d = D[sumc + q];
    if (j != js) {
      best = max(best, p.at(p.preBEF, kfj - k) - d);
      kfo = max(kfo, kfj);
    } else {
      if (k == 0 && cjs == 0 && EFb > d) return kInf;  // js's first entry is this moved one
      const int need = kfj - k - (EFb <= d ? 1 : 0);
      if (need > 0) best = max(best, p.at(p.preBEF, need) - d);
    }
  }
  int jx = jmax, Nx = s.N[jmax];
  if (jmax == js) {  // the others' largest N, highest j
    jx = -1;
    Nx = 0;
#pragma unroll 1
    for (int j = 0; j < m; ++j)
      if (j != js && (int)s.N[j] >= Nx) { Nx = s.N[j]; jx = j; }
  }
  const int ux = jx >= 0 ? Nx - kfo : 0;  // others' coarse levels that count
  const uint32_t below_s = (1u << js) - 1u, below_x = jx >= 0 ? (1u << jx) - 1u : 0u;
  uint32_t A = all & ~E[0];
#pragma unroll 1
  for (int t = 1, pos = 0, tl = max(ux, cjs); t <= tl; ++t) {
    if (t <= cjs) {
      const int64_t d = D[pos + __popc(A & below_s)];
      if (t == 1 && EFb > d) return kInf;  // js's first entry (coarse, level 1)
      const int need = Njs - t + 1 - (EFb <= d ? 1 : 0);
      if (need > 0) best = max(best, p.at(p.preBEF, need) - d);
    }
    if (t <= ux) best = max(best, p.at(p.preBEF, Nx - t + 1) - D[pos + __popc(A & below_x)]);
    pos += __popc(A);
    A &= ~E[t];
  }
  return best;
}

// One candidate, sequentially in this thread (the general path).
// B = 32 (kMask): the forward loop runs on level masks E (uint32 words at
// E, zero on entry; left dirty, the caller zeroes them) with the thresholds
// after them, and for strict plans the ordering's initial backward shift is
// taken level by level when every moved EF sorts after every coarse one
// (then owners and ranks are materialised only if a backward move is tried).
// EXPLAIN (NEXT-1, one candidate): xo[8 + t] = pipeline of the t-th committed
// forward move, xo[8 + n + t] = of the t-th backward move; xo[1..4] = Df, Db,
// forward / backward move counts.
template <int B, bool EXPLAIN = false>
__device__ int64_t teval(const Cfg& c, const TPlan& p, const int64_t* G, const int64_t* D, int64_t T_end, TS& s,
                         uint32_t* E, TStats& st, int64_t* xo = nullptr, int js1 = -1, int64_t dep1 = 0) {
  constexpr bool kMask = B == 32;
  const int n = c.n, m = p.m, kmax = p.kmax;
  const uint32_t all = m >= 32 ? 0xffffffffu : (1u << m) - 1u;
  const SB thr = kMask ? SB{(uint32_t)((reinterpret_cast<unsigned char*>(E) - k2sm) + 4 * (B + 2))} : s.thr;
  // ---------------- coarse init (R9) -------------------------------------
  if (!kMask) {
#pragma unroll 1
    for (int t = 0; t < (n + 5) / 4; ++t) s.cnt.w(t) = 0u;  // cnt[0..n+1] (4-aligned)
  }
  // the first findCritical of both phases runs on N: one pass for both keys
  uint32_t kf0 = 0, kf1 = 0, kb0 = 0;
  int maxN = 0;
#pragma unroll 1
  for (int j = 0, off = 0; j < m; ++j, off += p.np1) {
    const int Nj = s.N[j];
    s.c[j] = (uint8_t)Nj;
    if (kMask) E[Nj] |= 1u << j;
    else s.cnt[Nj] += 1;
    maxN = max(maxN, Nj);
    const uint64_t k = __ldg(reinterpret_cast<const uint64_t*>(p.ptr(p.kj)) + off + Nj);
    kf1 = max(kf1, min(kf0, (uint32_t)k));  // the two largest forward keys (keys are distinct: j in the low bits)
    kf0 = max(kf0, (uint32_t)k);
    kb0 = max(kb0, (uint32_t)(k >> 32));
  }
  const int jmax = kMask ? 31 - __clz(E[maxN]) : 0;  // highest j with N_j = max N
  if (!kMask) {
#pragma unroll 1
    for (int t = maxN - 1; t >= 1; --t) s.cnt[t] += s.cnt[t + 1];  // histogram -> #{j : c_j >= t}
  }
  int sumc = n, M = 0, itf = 0, atf = 0, itb = 0, atb = 0;
  uint32_t MV = 0;  // pipelines with a committed forward move (kMask)
  // ---------------- forward OptimizeSchedule (R10-R13) --------------------
  // initial forward shift (no thresholds, no trial): the first slot of each
  // level t sits at position sum_{t' < t} cnt[t'] (tdep_fwd with M = 0)
  int64_t dep = kNegInf;
  if (kMask && js1 >= 0) {
    // resume after the fast path's first forward iteration, which committed
    // pipeline js1's move with forward shift dep1 (tfast: the same pick and
    // trial as this loop's first iteration; B = 32 plans only)
    const uint32_t bit = 1u << js1;
    const int cjs = s.c[js1];
    E[cjs] &= ~bit;
    E[cjs - 1] |= bit;
    thr[0] = (uint8_t)p.at(p.bpF, row_of(p, js1) * kmax);
    s.c[js1] = (uint8_t)(cjs - 1);
    MV = bit;
    M = 1;
    dep = dep1;
    --sumc;
    itf = atf = 1;
    kf0 = cjs > 1 ? __ldg(reinterpret_cast<const uint32_t*>(p.ptr(p.kj)) + 2 * (js1 * p.np1 + cjs - 1)) : 0u;
  } else {
    uint32_t A = all;
#pragma unroll 1
    for (int t = 1, pos = 0; pos < n; ++t) {
      dep = max(dep, p.at(p.preEF, t) - G[pos]);
      if (kMask) {
        pos += __popc(A);
        A &= ~E[t];
      } else {
        pos += s.cnt[t];
      }
    }
  }
  int64_t Delta;
#pragma unroll 1
  for (;;) {
    ++itf;
    int js;
    // findCritical (R11): the picks are a merge of the pipelines' key lists,
    // each non-increasing in the count, so while the last pick's next key
    // still beats the runner-up (kf1, untouched by the pick) it is the max
    if (itf > 1 && kf0 <= kf1) critical2(p, s.c, m, kf0, kf1);
    const int64_t dev = crit_value(p, p.devF, s.c, kf0, js);
    Delta = max((int64_t)0, max(dev, dep));
    if (Delta == 0 || sumc == 0) break;
    const int as = row_of(p, js), cjs = s.c[js], kfj = s.N[js] - cjs;
    if (kfj >= (int)p.at(p.lenF, as)) break;  // ScheduleKernels fails (R12)
    ++atf;
    const int bp = (int)p.at(p.bpF, as * kmax + kfj);  // EF_i + L <= F_i holds for slots >= bp
    int64_t dep2;
    int q = M;
    if (kMask) {  // trial move: js one level down, threshold bp inserted in order
      const uint32_t bit = 1u << js;
      OPT_CHECK(cjs >= 1 && cjs <= B && M < B);
      E[cjs] &= ~bit;
      E[cjs - 1] |= bit;
#pragma unroll 1
      for (; q > 0 && (int)thr[q - 1] > bp; --q) thr[q] = thr[q - 1];
      thr[q] = (uint8_t)bp;
      dep2 = tdep_mask(p, G, n, sumc - 1, E, all, thr, M + 1);
      if (dep2 > Delta) {  // checkEncLLMDep fails (R13): undo, phase ends
        E[cjs - 1] &= ~bit;
        E[cjs] |= bit;
#pragma unroll 1
        for (; q < M; ++q) thr[q] = thr[q + 1];
        break;
      }
      s.c[js] = (uint8_t)(cjs - 1);
      MV |= bit;
      ++M;
    } else {
      s.c[js] = (uint8_t)(cjs - 1);  // trial move
      s.cnt[cjs] -= 1;
      dep2 = tdep_fwd(p, G, n, sumc - 1, bp, s, M);
      if (dep2 > Delta) {  // checkEncLLMDep fails (R13): undo, phase ends
        s.c[js] = (uint8_t)cjs;
        s.cnt[cjs] += 1;
        break;
      }
      ++M;  // commit: insert the threshold
#pragma unroll 1
      for (; q > 0 && s.thr[q - 1] > bp; --q) s.thr[q] = s.thr[q - 1];
      s.thr[q] = (uint8_t)bp;
    }
    if (EXPLAIN) xo[8 + M - 1] = js;
    dep = dep2;
    --sumc;
    // the pick's next key (count c_js - 1); below the runner-up: rescan next time
    kf0 = s.c[js] > 0 ? __ldg(reinterpret_cast<const uint32_t*>(p.ptr(p.kj)) + 2 * (js * p.np1 + s.c[js])) : 0u;
  }
  const int64_t Df = Delta;
  // ---------------- global ordering (R14) -------------------------------
  bool have_order = true;
  int64_t dep_b = kNegInf;
  bool done_b = false;
  const SB mv{(uint32_t)((reinterpret_cast<unsigned char*>(E) - k2sm) + 4 * (maxN + 1))};  // after E[maxN]
  if (kMask && p.strict && tsep(p, D, s, E, all, MV, maxN, jmax, sumc, Df, mv, dep_b)) {
    have_order = false;  // owners and ranks materialised if a backward move is tried
    done_b = true;
  }
  if (!done_b) {
    have_order = M > 0 || !p.strict;
    dep_b = !have_order ? order_fast(p, D, m, s)
            : p.strict  ? order_strict(p, D, m, Df, s)
                        : order_general(p.ptr(p.preEF), p.ptr(p.preBEF), p.ptr(p.inbF), p.rt, p.kmax, D, m, Df, M > 0, s.N.o, s.c.o, s.kb.o, s.own.o, s.rk.o);
  }
  // ---------------- backward OptimizeSchedule (R15) ------------------------
  int sumcb = n;
  bool init_b = false;
  #pragma unroll 1
  for (;;) {
    ++itb;
    int js;
    const int64_t dev = !init_b ? crit_value(p, p.devB, s.N, kb0, js) : critical(p, p.devB, 1, s.cb, m, js);
    Delta = max((int64_t)0, max(dev, dep_b));
    if (Delta == 0 || sumcb == 0) break;
    const int as = row_of(p, js), kfj = s.N[js] - s.c[js];
    const int kbj = init_b ? s.N[js] - s.cb[js] : 0;
    const int64_t rowoff = (int64_t)as * (kmax + 1) + kfj;
    if (kbj >= (int)p.at(p.lenB, rowoff)) break;
    const int64_t EFb = p.at(p.inbB, rowoff * kmax + kbj);
    ++atb;
    int64_t dep2 = kNegInf;
    bool have2 = false;
    if (!have_order) {
      if (kMask && !init_b) {  // first trial on tsep's ordering, nothing materialised
        dep2 = tbwd1(p, D, s, E, all, mv, M, sumc, m, jmax, js, EFb);
        if (dep2 > Delta) break;
        have2 = true;  // the move commits: owners and ranks for the rest of the phase
      }
      order_strict(p, D, m, Df, s);  // materialise owners and ranks (same order, same initial shift)
      have_order = true;
    }
    if (!init_b) {  // backward moves are rare: per-pipeline state on first use
      #pragma unroll 1
      for (int j = 0; j < m; ++j) s.cb[j] = s.N[j];
      #pragma unroll 1
      for (int i = 0; i < n; ++i) s.Qcb[i] = 0;
      init_b = true;
    }
    if (!have2) dep2 = tdep_bwd(p, D, n, js, EFb, s);
    if (dep2 > Delta) break;
    #pragma unroll 1
    for (int i = 0; i < n; ++i) s.Qcb[i] += (s.own[i] == js && EFb <= D[i]) ? 1 : 0;
    s.cb[js] -= 1;
    if (EXPLAIN) xo[8 + n + (n - sumcb)] = js;
    dep_b = dep2;
    --sumcb;
  }
  if (EXPLAIN) {
    xo[1] = Df;
    xo[2] = Delta;
    xo[3] = M;
    xo[4] = n - sumcb;
    #pragma unroll 1
    for (int j = 0; j < m; ++j) {
      xo[8 + 2 * n + j] = s.N[j];
      xo[8 + 2 * n + m + j] = s.c[j];
      xo[8 + 2 * n + 2 * m + j] = init_b ? s.cb[j] : s.N[j];
    }
  }
  st.v[0] += 1;
  st.v[1] += m;
  st.v[2] += m * itf;
  st.v[3] += itf;
  st.v[4] += atf;
  st.v[5] += m * itb;
  st.v[6] += itb;
  st.v[7] += atb;
  st.v[9] += 1;
  return T_end + Df + Delta;  // R16
}

// ---------------------------------------------------------------------------
// Fast path (plans with PRE_EF strictly increasing and m <= 32): the whole
// candidate when neither phase commits a move, i.e. the first attempt of
// each OptimizeSchedule phase fails (R11-R13) or is never made.  Returns
// false as soon as a first move would commit; the candidate then goes to the
// general path (teval), which evaluates it from the start.  (Letting the
// fast path run the forward loop further measured slower: the warp waits for
// its longest loop, which the general path's full batches absorb better.)
//
// Pipeline sets are 32-bit masks.  E[x] = {j : N_j = x}; the walk over levels
// t = 1..max N turns it into A_t = {j : N_j >= t} (stored back in E[t]), so
// the slot of the coarse entry (t, j) in the global ordering without moved
// entries (R14: level-major, j within a level) is pos_t + |A_t below j|.
//   * forward (R10): the first slot of level t is pos_t; a trial move of js
//     (one threshold bp, R10's closed form) removes js from level N_js.
//   * ordering + initial backward shift (R14, R15): slot (t, j) has rank
//     N_j - t + 1 and D is non-increasing in the slot, so for each rank r the
//     term PREB_EF(r) - D[slot] is largest at the largest slot of rank r:
//     level N_max - r + 1 of jmax, the highest j with N_j = N_max.  One entry
//     per level instead of one per slot.
//   * backward trial of jb (no backward move yet, Qcb = 0): only jb's entries
//     change (need = r - [EFb <= D]); the others' maximum is the shift above,
//     or, when jb = jmax, the same walk over j2 (largest N among j != jmax).
// Leaves E zeroed.  MT: the mask word (16 bits for instances of m <= 16).
template <int B, typename MT>
__device__ __forceinline__ bool tfast(const TPlan& p, const int64_t* G, const int64_t* D, int n, const TS& s,
                                      MT* E, int64_t& Df, int64_t& Db, TStats& st, int& js1, int64_t& dep1) {
  const int m = p.m, np1 = p.np1;
  uint32_t kf0 = 0, kb0 = 0;
  int Nmax = 0;
  const uint64_t* kj = reinterpret_cast<const uint64_t*>(p.ptr(p.kj));
#pragma unroll 2
  for (int j = 0, off = 0; j < m; ++j, off += np1) {
    const int Nj = s.N[j];
    OPT_CHECK(Nj >= 1 && Nj <= n && Nj <= B);
    E[Nj] |= (MT)(1u << j);
    const uint64_t k = __ldg(kj + off + Nj);  // first findCritical of both phases (R11)
    kf0 = max(kf0, (uint32_t)k);
    kb0 = max(kb0, (uint32_t)(k >> 32));
    Nmax = max(Nmax, Nj);
  }
  const int jmax = 31 - __clz((uint32_t)E[Nmax]);  // highest j with N_j = N_max
  const uint32_t all = m == 32 ? 0xffffffffu : (1u << m) - 1u;
  const uint32_t below_max = (1u << jmax) - 1u;
  int64_t dep = kNegInf, depb = kNegInf;
  {
    uint32_t A = all;
#pragma unroll 1
    for (int t = 1, pos = 0; t <= Nmax; ++t) {
      const uint32_t e = E[t];
      E[t] = (MT)A;
      OPT_CHECK(t <= n && pos < n && pos + __popc(A & below_max) < n);
      dep = max(dep, p.at(p.preEF, t) - G[pos]);
      depb = max(depb, p.at(p.preBEF, Nmax - t + 1) - D[pos + __popc(A & below_max)]);
      pos += __popc(A);
      A &= ~e;
    }
  }
  bool general = false;
  js1 = -1;
  // ---- forward, first iteration
  int js;
  const int64_t dev = crit_value(p, p.devF, s.N, kf0, js);
  const int64_t Delta = max((int64_t)0, max(dev, dep));
  int atf = 0;
  if (Delta != 0) {
    const int as = row_of(p, js);
    if ((int)p.at(p.lenF, as) > 0) {
      ++atf;
      const int bp = (int)p.at(p.bpF, as * p.kmax);
      if (bp <= n) {  // else need_n = n > n - 1 coarse entries: INF, the move fails
        const int Njs = s.N[js];
        const uint32_t jsbit = 1u << js;
        int64_t dep2 = kNegInf;
#pragma unroll 1
        for (int t = 1, pos = 0; pos < n - 1; ++t) {
          uint32_t A = E[t];
          if (t == Njs) A &= ~jsbit;
          const int st1 = pos + 1;  // first position of level t (1-based): slot st1, or st1 + 1 past the threshold
          OPT_CHECK(t <= n && (st1 < bp ? st1 - 1 : st1) < n);
          dep2 = max(dep2, p.at(p.preEF, t) - G[st1 < bp ? st1 - 1 : st1]);
          pos += __popc(A);
        }
        general = dep2 <= Delta;  // checkEncLLMDep holds: the move commits
        if (general) {  // k2_general resumes after this commit
          js1 = js;
          dep1 = dep2;
        }
      }
    }
  }
  Df = Delta;
  int atb = 0;
  if (!general) {
    // ---- backward, first iteration (initial shift depb)
    int jb;
    const int64_t devb = crit_value(p, p.devB, s.N, kb0, jb);
    const int64_t Delta_b = max((int64_t)0, max(devb, depb));
    if (Delta_b != 0) {
      const int as = row_of(p, jb);
      const int64_t rowoff = (int64_t)as * (p.kmax + 1);  // kf = 0 forward chains
      if ((int)p.at(p.lenB, rowoff) > 0) {
        ++atb;
        const int64_t EFb = p.at(p.inbB, rowoff * p.kmax);
        if (EFb <= D[jb]) {  // else jb's rank-N slot (level 1, slot jb) loses its coarse entry: INF
          const int Njb = s.N[jb];
          const bool other2 = jb == jmax;
          int N2 = 0, j2 = 0;  // jb = jmax: the others' largest N and its highest j (E[t] holds A_t)
          if (other2) {
#pragma unroll 1
            for (N2 = Nmax; N2 > 0 && __popc(E[N2]) < 2; --N2) {}
            if (N2 > 0) j2 = 31 - __clz((uint32_t)E[N2] & ~(1u << jmax));
          }
          const int tl = max(Njb, N2);
          const uint32_t below_b = (1u << jb) - 1u, below_2 = (1u << j2) - 1u;
          int64_t dep2 = other2 ? kNegInf : depb;
#pragma unroll 1
          for (int t = 1, pos = 0; t <= tl; ++t) {
            const uint32_t A = E[t];
            if (t <= Njb) {
              const int sl = pos + __popc(A & below_b);
              const int64_t d = D[sl];
              const int need = Njb - t + 1 - (EFb <= d ? 1 : 0);
              if (need > 0) dep2 = max(dep2, p.at(p.preBEF, need) - d);
            }
            if (other2 && t <= N2) dep2 = max(dep2, p.at(p.preBEF, N2 - t + 1) - D[pos + __popc(A & below_2)]);
            pos += __popc(A);
          }
          general = dep2 <= Delta_b;  // a backward move commits: the general path
        }
      }
    }
    Db = Delta_b;
  }
#pragma unroll 1
  for (int t = 1; t <= Nmax; ++t) E[t] = 0;
  if (!general) {
    st.v[0] += 1;
    st.v[1] += m;
    st.v[2] += m;
    st.v[3] += 1;
    st.v[4] += atf;
    st.v[5] += m;
    st.v[6] += 1;
    st.v[7] += atb;
    st.v[8] += 1;
  }
  return !general;
}

// positions of this rank (block-cyclic over [begin, end)) below global index x >= begin
__device__ __forceinline__ uint64_t rank_pos(const EvalArgs& A, uint64_t x) {
  const uint64_t r = x - A.begin, fb = r / A.block, rem = r - fb * A.block, k = fb % A.world;
  return (fb / A.world) * A.block + (k > A.rank ? A.block : 0) + (k == A.rank ? rem : 0);
}

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tbetter(int64_t lat, uint64_t g, int64_t& bl, uint64_t& bg) {
  if (lat < bl || (lat == bl && g < bg)) { bl = lat; bg = g; }
}

// block argmin of the warps' bests into this block's partial (written on a
// range's first chunk, merged into on the later ones)
__device__ __forceinline__ void block_best(int64_t bl, uint64_t bg, int64_t* partials, int first) {
  __shared__ long long bl_sm[kTThreads / 32];
  __shared__ unsigned long long bg_sm[kTThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
    const uint64_t og = __shfl_xor_sync(0xffffffffu, bg, o);
    tbetter(ol, og, bl, bg);
  }
  if (lane == 0) { bl_sm[warp] = bl; bg_sm[warp] = bg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t l = INT64_MAX;
    uint64_t gg = UINT64_MAX;
    if (!first) { l = partials[2 * blockIdx.x]; gg = (uint64_t)partials[2 * blockIdx.x + 1]; }
    for (int w = 0; w < kTThreads / 32; ++w) tbetter(bl_sm[w], bg_sm[w], l, gg);
    partials[2 * blockIdx.x] = l;
    partials[2 * blockIdx.x + 1] = (int64_t)gg;
  }
}

__device__ __forceinline__ void flush_stats(const TStats& st, unsigned long long* stats) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    unsigned v = st.v[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && stats && v) atomicAdd(&stats[i], (unsigned long long)v);
  }
}

// K2 mode 1, fast kernel: every candidate of this rank's shard (range) or of
// the index list (EXPLICIT) through tfast; the candidates it hands over (and
// every candidate of a plan it does not cover: m > 32 or PRE_EF not strictly
// increasing) go to the global queue for k2_general, one warp-reserved batch
// of kGqBatch slots at a time (unused slots marked ~0).
template <bool EXPLICIT, int B, int BM>
__global__ void __launch_bounds__(kTThreads, B == 32 ? K2T_MINB : K2T_MINB_WIDE)
    k2_fast(Cfg c, EvalArgs A) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k2_general may become resident as blocks leave
  __shared__ int64_t G[B], D[B];
  __shared__ uint32_t bsm[B == 32 ? 33 * 33 : 1];
  const uint32_t* b32 = stage_binom32<B>(c, bsm);
  __shared__ uint64_t plo[EXPLICIT ? 1 : kMaxE], pn[EXPLICIT ? 1 : kMaxE];
  __shared__ int pstate[EXPLICIT ? 1 : kMaxE];  // 0 not known ready, 1 ready
  __shared__ uint64_t psum[EXPLICIT ? 1 : kMaxE + 1];  // this rank's positions of the plans before k2order[k]
  const int lane = threadIdx.x & 31, n = c.n;
  const int64_t T_end = c.scal[1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    G[i] = c.F[i] - c.L;          // EF_i + L <= F_i
    D[i] = T_end - c.B[i] - c.L;  // EB_i >= B_i + L (mirrored)
  }
  if (!EXPLICIT)
    for (int e = threadIdx.x; e < c.E; e += blockDim.x) {  // this rank's positions of plan e
      const PlanDesc& d = c.plans[e];
      const uint64_t x0 = max(A.begin, d.first), x1 = min(A.end, d.first + d.count);
      const uint64_t lo = x0 < x1 ? rank_pos(A, x0) : 0, hi = x0 < x1 ? rank_pos(A, x1) : 0;
      plo[e] = lo;
      pn[e] = hi - lo;
      pstate[e] = 0;
    }
  __syncthreads();
  if (!EXPLICIT && threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int k = 0; k < c.n_k2order; ++k) {
      psum[k] = acc;
      acc += pn[c.k2order[k]];
    }
    psum[c.n_k2order] = acc;
  }
  __syncthreads();
  TS s;  // the fast path only keeps the composition and its masks per thread
  s.N = SB{(uint32_t)(threadIdx.x * fstride<B, BM>())};
  using MT = typename FMask<BM>::T;
  MT* E = reinterpret_cast<MT*>(k2sm + threadIdx.x * fstride<B, BM>() + BM);  // tfast's masks (zero)
  for (int t = 0; t < B + 2; ++t) E[t] = 0;
  TPlan p;
  p.e = -1;
  TStats st = {{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
  int64_t bl = INT64_MAX;
  uint64_t bg = UINT64_MAX;
  const unsigned lt_mask = (1u << lane) - 1u;
  unsigned qb = 0, qe = 0;  // this warp's reserved queue slots [qb, qe) (warp-uniform)
  // one candidate per lane (valid lanes): fast path, else into the queue
  auto step = [&](bool valid, uint64_t g, uint64_t out, int e) {
    bool pend = false;
    int js1 = -1;
    int64_t dep1 = 0;
    if (valid) {
      int64_t Df, Db;
      if (p.fast && tfast<B, MT>(p, G, D, n, s, E, Df, Db, st, js1, dep1)) {
        const int64_t lat = T_end + Df + Db;  // R16
        if (A.lat_out) A.lat_out[out] = lat;
        tbetter(lat, g, bl, bg);
      } else {
        pend = true;
      }
    }
    const unsigned want = __ballot_sync(0xffffffffu, pend);
    if (!want) return;
    const unsigned k = __popc(want);
    if (qb + k > qe) {  // a new batch; the rest of the old one stays unused
      for (unsigned x = qb + lane; x < qe; x += 32) A.gq[x] = ~0ull;
      unsigned r = 0;
      if (lane == 0) r = atomicAdd(A.gqn, (unsigned)kGqBatch);
      r = __shfl_sync(0xffffffffu, r, 0);
      OPT_CHECK(r + kGqBatch <= A.gqcap);
      qb = r;
      qe = r + kGqBatch;
    }
    if (pend) {  // (the index g may use 64 bits; lat_out positions stay below 2^56)
      const unsigned x = qb + __popc(want & lt_mask);
      A.gq[x] = g;
      A.gqo[x] = out | (uint64_t)e << 56;
      if (p.m <= kPackParts<B>()) {  // the composition (no unranking in k2_general) and the first forward commit
        const bool r = B == 32 && js1 >= 0 && kPackBits<B>() * p.m + 4 <= 64 && js1 < 15;
        A.gqc[x] = tpack<B>(s.N, p.m) | (r ? (uint64_t)(js1 + 1) << (kPackBits<B>() * p.m) : 0ull);
        if (r) A.gqd[x] = dep1;
      }
    }
    qb += k;
  };
  if (EXPLICIT) {
    const uint64_t nchunks = (A.count + 31) / 32;
    for (;;) {
      unsigned long long ch = 0;
      if (lane == 0) ch = atomicAdd(A.counter, 1ull);
      ch = __shfl_sync(0xffffffffu, ch, 0);
      if (ch >= nchunks) break;
      const uint64_t i = ch * 32 + lane;
      bool valid = false;
      uint64_t g = 0;
      int e = -1;
      if (i < A.count) {
        g = A.index[i];
        e = tfind_plan(c, g);
        if (e >= 0) {
          if (e != p.e) tplan(c, e, p);
          tunrank<B>(c, b32, p, n, g - p.first, s);
          valid = true;
        }
      }
      step(valid, g, i, e);
    }
  } else {
    // This rank's positions of the plans, concatenated in k2order: plan
    // k2order[k] holds [psum[k], psum[k + 1]) of this order space, its
    // positions of the block-cyclic sharding over [begin, end) being
    // [plo[e], plo[e] + pn[e]).  A warp claims 32 * r consecutive order
    // positions with one atomic (r from kTRun down to kTMinRun as the
    // remaining work shrinks: guided self-scheduling) and evaluates them
    // plan segment by plan segment, r consecutive candidates per lane, each
    // segment once K1 has completed its plan (this launch may overlap K1;
    // K1 finishes plans in k2order).
    const uint64_t nwarps = (uint64_t)gridDim.x * (kTThreads / 32);
    const uint64_t T = psum[c.n_k2order];
    int k = 0;  // plan cursor in k2order (claims only move forward)
    for (;;) {
      unsigned long long x0 = 0, tk = 0;
      if (lane == 0) {
        const unsigned long long seen = *(volatile unsigned long long*)A.counter;
        const unsigned long long left = T > seen ? T - seen : 0;
        tk = min(32ull * kTRun, max(32ull * kTMinRun, left * kTGss / (kTGssDen * nwarps) / 32 * 32));
        x0 = left ? atomicAdd(A.counter, tk) : T;
      }
      x0 = __shfl_sync(0xffffffffu, x0, 0);
      tk = __shfl_sync(0xffffffffu, tk, 0);
      if (x0 >= T) break;
      const uint64_t x1 = min((uint64_t)(x0 + tk), T);
#ifndef K2T_GSTATS
      st.v[10] += lane == 0;
#endif
      for (uint64_t x = x0; x < x1;) {
        while (psum[k + 1] <= x) ++k;
        const int e = c.k2order[k];
        const uint64_t xb = min(x1, psum[k + 1]);
        if (__shfl_sync(0xffffffffu, pstate[e], 0) == 0) {  // wait for K1 to complete plan e
          if (lane == 0) {
            volatile int* pst = pstate;  // shared by the block's warps; only ever raised
            // poll relaxed (an acquire load invalidates L1), acquire once when complete
            while (pst[e] == 0 && ld_relaxed(&c.pdone[e]) < plan_items(c.plans[e])) __nanosleep(500);
            (void)ld_acquire(&c.pdone[e]);
            pst[e] = 1;
          }
          __syncwarp();  // the lanes' table reads follow lane 0's acquire
        }
        if (e != p.e) tplan(c, e, p);
        const int r = (int)((xb - x + 31) / 32);
        const uint64_t p0 = plo[e] + (x - psum[k]) + (uint64_t)lane * r, pend = plo[e] + (xb - psum[k]);
        uint64_t g = 0;
        for (int it = 0; it < r; ++it) {  // the same trip count on every lane (warp-synchronous queue)
          const uint64_t q = p0 + it;
          const bool valid = q < pend;
          if (valid) {
            if (it == 0 || q % A.block == 0) {  // (re)locate: positions -> global indices jump at rank blocks
              const uint64_t rb = q / A.block;
              g = A.begin + (rb * A.world + A.rank) * (uint64_t)A.block + (q - rb * A.block);
              tunrank<B>(c, b32, p, n, g - p.first, s);
#ifndef K2T_GSTATS
              st.v[11] += 1;
#endif
            } else {
              ++g;
              tnext(p.m, s);
            }
          }
          step(valid, g, g - A.begin, e);
        }
        x = xb;
      }
    }
  }
  for (unsigned x = qb + lane; x < qe; x += 32) A.gq[x] = ~0ull;  // the tail of this warp's last batch
  flush_stats(st, A.stats);
  block_best(bl, bg, A.partials, A.first_chunk);
}

// K2 mode 1, general kernel: the queued candidates through teval (the whole
// algorithm), warps taking 32 queue slots at a time.
template <int B, int BM>
__global__ void __launch_bounds__(kTThreads, B == 32 ? K2T_GMINB : BM == 16 ? (B == 64 ? 4 : 2) : B == 64 ? 3 : BM == 64 ? 2 : 1)
    k2_general(Cfg c, EvalArgs A) {
  __shared__ int64_t G[B], D[B];
  __shared__ uint32_t bsm[B == 32 ? 33 * 33 : 1];
  const uint32_t* b32 = stage_binom32<B>(c, bsm);
  const int lane = threadIdx.x & 31, n = c.n;
  const int64_t T_end = c.scal[1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    G[i] = c.F[i] - c.L;
    D[i] = T_end - c.B[i] - c.L;
  }
  __syncthreads();
  TS s = ts_at<B, BM>((uint32_t)(threadIdx.x * gstride<B, BM>()));
  uint32_t* E = reinterpret_cast<uint32_t*>(k2sm + threadIdx.x * gstride<B, BM>() + 2 * BM);  // (B = 32 only)
  if (B == 32)
    for (int t = 0; t < B + 2; ++t) E[t] = 0u;
  TPlan p;
  p.e = -1;
  TStats st = {{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
  int64_t bl = INT64_MAX;
  uint64_t bg = UINT64_MAX;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the fast kernel (programmatic dependency) has finished
  const uint64_t total = *reinterpret_cast<volatile unsigned*>(A.gqn);
  for (;;) {
    unsigned long long ch = 0;
    if (lane == 0) ch = atomicAdd(A.counter2, 32ull);
    ch = __shfl_sync(0xffffffffu, ch, 0);
    if (ch >= total) break;
    const uint64_t i = ch + lane;
    const uint64_t g = i < total ? A.gq[i] : ~0ull;
    if (g != ~0ull) {
      const uint64_t qo = A.gqo[i];
      const int e = (int)(qo >> 56);
      if (e != p.e) tplan(c, e, p);
      int js1 = -1;
      int64_t dep1 = 0;
      if (p.m <= kPackParts<B>()) {
        const uint64_t v = A.gqc[i];
        tunpack<B>(v, p.m, s.N);
        if (B == 32 && kPackBits<B>() * p.m + 4 <= 64) js1 = (int)(v >> (kPackBits<B>() * p.m)) - 1;
        if (js1 >= 0) dep1 = A.gqd[i];
      } else {
        tunrank<B>(c, b32, p, n, g - p.first, s);
      }
      const int64_t lat = teval<B>(c, p, G, D, T_end, s, E, st, nullptr, js1, dep1);
      if (A.lat_out) A.lat_out[qo & ((1ull << 56) - 1)] = lat;
      tbetter(lat, g, bl, bg);
      if (B == 32)
        for (int t = 0; t < B + 2; ++t) E[t] = 0u;  // teval leaves its masks and scratch dirty
    }
  }
  flush_stats(st, A.stats);
  block_best(bl, bg, A.partials2, A.first_chunk);
  // the last block out resets the queue and claim counters for the next
  // chunk or call (every block read the queue length before leaving), so
  // that no memset separates K1 from the next fast kernel (its programmatic
  // dependent launch)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(A.gdone, 1u) == gridDim.x - 1) {
      *A.gqn = 0u;
      *A.counter2 = 0ull;
      *A.counter = 0ull;
      for (int e = 0; e < A.nplans; ++e) A.pclaim[e] = 0ull;
      __threadfence();
      *A.gdone = 0u;
    }
  }
}

// NEXT-1: one candidate's decisions (the schedule's moves), for emission.
// out: [0] lat, [1] Df, [2] Db, [3] forward moves, [4] backward moves,
// [5] plan, [6] m, [7] n, [8, 8+n) forward move pipelines, [8+n, 8+2n)
// backward ones, then N[m], c_final[m], cb_final[m].  One thread works.
template <int B, int BM>
__global__ void __launch_bounds__(kTThreads) k2_explain(Cfg c, uint64_t g, int64_t* out) {
  __shared__ int64_t G[B], D[B];
  __shared__ uint32_t bsm[B == 32 ? 33 * 33 : 1];
  const uint32_t* b32 = stage_binom32<B>(c, bsm);
  const int n = c.n;
  const int64_t T_end = c.scal[1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    G[i] = c.F[i] - c.L;
    D[i] = T_end - c.B[i] - c.L;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int e = tfind_plan(c, g);
  out[0] = -1;
  if (e < 0) return;
  TPlan p;
  tplan(c, e, p);
  TS s = ts_at<B, BM>(0u);
  uint32_t* E = reinterpret_cast<uint32_t*>(k2sm + 2 * BM);
  for (int t = 0; t < B + 2; ++t) E[t] = 0u;
  tunrank<B>(c, b32, p, n, g - p.first, s);
  TStats st = {{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}};
  out[5] = e;
  out[6] = p.m;
  out[7] = n;
  out[0] = teval<B, true>(c, p, G, D, T_end, s, E, st, out);
}

// NEXT-4: the global ordering (R14) of an explained candidate, slot by slot:
// out[2 i] = the pipeline whose forward finish is LLM microbatch i, out[2 i +
// 1] = that finish (LLM-relative: coarse PRE_EF(t) - Df, moved INB_F).  One
// thread, the plain definition: every entry, sorted by (value, pipeline,
// local index).  xo = optimus_explain's device output.
__global__ void k_order_dump(Cfg c, const int64_t* xo, int64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int n = c.n, e = (int)xo[5], m = (int)xo[6];
  const int64_t Df = xo[1];
  const int64_t* N = xo + 8 + 2 * n;
  const int64_t* cf = N + m;
  const PlanDesc& d = c.plans[e];
  const int64_t* preEF = c.tables + d.preF + (int64_t)(d.P - 1) * (n + 1);
  const int64_t* inbF = c.tables + d.inbF;
  int q = 0;
  for (int j = 0; j < m; ++j) {
    const int a = j / d.rt;
    for (int u = 0; u < (int)N[j]; ++u) {  // j's entries in local order: coarse t = 1..c_j, then moved
      const int64_t v = u < cf[j] ? preEF[u + 1] - Df : inbF[(int64_t)a * d.kmax + (u - cf[j])];
      int x = q++;
      // insertion by (value, pipeline, local): later (j, u) keys are larger
      while (x > 0 && out[2 * (x - 1) + 1] > v) {
        out[2 * x] = out[2 * (x - 1)];
        out[2 * x + 1] = out[2 * (x - 1) + 1];
        --x;
      }
      out[2 * x] = j;
      out[2 * x + 1] = v;
    }
  }
}

}  // namespace

template <int B, int BM>
static void k2t_attrs() {
  constexpr int smem = tsmem<B, BM>(), fsm = fsmem<B, BM>();
  cudaFuncSetAttribute(k2_fast<false, B, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);
  cudaFuncSetAttribute(k2_fast<false, B, BM>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(k2_fast<true, B, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, fsm);
  cudaFuncSetAttribute(k2_fast<true, B, BM>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(k2_general<B, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, gsmem<B, BM>());
  cudaFuncSetAttribute(k2_general<B, BM>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaFuncSetAttribute(k2_explain<B, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// K2 mode 1 instance for n slots and at most mmax pipelines in a plan with
// candidates: 0 = (32, 32), 1 = (64, 64), 2 = (128, 64), 3 = (128, 128),
// 4 = (64, 16), 5 = (128, 16)
__host__ __device__ constexpr int tinstance(int n, int mmax) {
  return n <= 32 ? 0 : n <= 64 ? (mmax <= 16 ? 4 : 1) : mmax <= 16 ? 5 : mmax <= 64 ? 2 : 3;
}

template <int B, int BM>
static int grid_b(int sms) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2_fast<false, B, BM>, kTThreads, fsmem<B, BM>());
  return max(1, per) * sms;
}

template <int B, int BM>
static int ggrid_b(int sms) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2_general<B, BM>, kTThreads, gsmem<B, BM>());
  return max(1, per) * sms;
}

int eval_thread_instance(int n, int mmax) { return tinstance(n, mmax); }

// dynamic shared memory opt-in of every instance (once per device, capi's device_info)
void eval_thread_attrs() {
  k2t_attrs<32, 32>();
  k2t_attrs<64, 64>();
  k2t_attrs<128, 64>();
  k2t_attrs<128, 128>();
  k2t_attrs<64, 16>();
  k2t_attrs<128, 16>();
}

// persistent grids of instance i: fast kernel, general kernel
int eval_thread_grid(int sms, int i) {
  switch (i) {
    case 0: return grid_b<32, 32>(sms);
    case 1: return grid_b<64, 64>(sms);
    case 2: return grid_b<128, 64>(sms);
    case 4: return grid_b<64, 16>(sms);
    case 5: return grid_b<128, 16>(sms);
    default: return grid_b<128, 128>(sms);
  }
}

int eval_general_grid(int sms, int i) {
  switch (i) {
    case 0: return ggrid_b<32, 32>(sms);
    case 1: return ggrid_b<64, 64>(sms);
    case 2: return ggrid_b<128, 64>(sms);
    case 4: return ggrid_b<64, 16>(sms);
    case 5: return ggrid_b<128, 16>(sms);
    default: return ggrid_b<128, 128>(sms);
  }
}

template <int B, int BM>
static void explain_b(const Cfg& c, uint64_t g, int64_t* d_out, cudaStream_t st) {
  k2_explain<B, BM><<<1, kTThreads, (size_t)tsmem<B, BM>(), st>>>(c, g, d_out);
}

cudaError_t launch_order_dump(const Cfg& c, const int64_t* d_explain, int64_t* d_out, cudaStream_t st) {
  k_order_dump<<<1, 32, 0, st>>>(c, d_explain, d_out);
  return cudaGetLastError();
}

cudaError_t launch_explain(const Cfg& c, uint64_t g, int64_t* d_out, cudaStream_t st) {
  switch (tinstance(c.n, c.mmax)) {
    case 0: explain_b<32, 32>(c, g, d_out, st); break;
    case 1: explain_b<64, 64>(c, g, d_out, st); break;
    case 2: explain_b<128, 64>(c, g, d_out, st); break;
    case 4: explain_b<64, 16>(c, g, d_out, st); break;
    case 5: explain_b<128, 16>(c, g, d_out, st); break;
    default: explain_b<128, 128>(c, g, d_out, st); break;
  }
  return cudaGetLastError();
}

// K2 mode 1: the range (or index list) a chunk at a time, so that the queue
// (gqcap slots, less the batches every fast warp may leave half used) holds
// every candidate a chunk can hand over; per chunk the fast kernel (the first
// one overlapping K1 by programmatic dependent launch) then the general one.
// Range chunks are whole multiples of block x world global indices from
// begin, so the block-cyclic shard is the same as in one launch.
template <int B, int BM>
static cudaError_t launch_eval_thread_b(const Cfg& c, const EvalArgs& a0, cudaStream_t st) {
  const uint64_t margin = (uint64_t)kGqBatch * a0.grid * (kTThreads / 32);
  if (a0.gqcap <= margin) return cudaErrorInvalidValue;
  const uint64_t room = a0.gqcap - margin;
  EvalArgs a = a0;
  a.first_chunk = 1;
  cudaError_t e = cudaSuccess;
  auto chunk = [&](bool pdl) -> cudaError_t {
    cudaError_t r = cudaSuccess;  // (queue and claim counters are zero: load, then k2_general's last block)
    if (a.index) {
      k2_fast<true, B, BM><<<a.grid, kTThreads, fsmem<B, BM>(), st>>>(c, a);
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)a.grid);
      cfg.blockDim = dim3(kTThreads);
      cfg.dynamicSmemBytes = fsmem<B, BM>();
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl ? 1 : 0;  // may start while K1 (which triggers at its start) still runs
      r = cudaLaunchKernelEx(&cfg, k2_fast<false, B, BM>, c, a);
      if (r != cudaSuccess) return r;
    }
    {  // programmatic dependent launch: its prologue overlaps the fast kernel's tail
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)a.grid2);
      cfg.blockDim = dim3(kTThreads);
      cfg.dynamicSmemBytes = gsmem<B, BM>();
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      r = cudaLaunchKernelEx(&cfg, k2_general<B, BM>, c, a);
      if (r != cudaSuccess) return r;
    }
    a.first_chunk = 0;
    return cudaGetLastError();
  };
  if (a0.index) {
    uint64_t off = 0;
    do {
      a.index = a0.index + off;
      a.count = min(room, a0.count - off);
      a.lat_out = a0.lat_out ? a0.lat_out + off : nullptr;
      if ((e = chunk(false)) != cudaSuccess) return e;
      off += a.count;
    } while (off < a0.count);
  } else {
    const uint64_t per = (uint64_t)a0.block * a0.world;
    const uint64_t C = max((uint64_t)1, room / a0.block) * per;
    uint64_t b = a0.begin;
    do {
      a.begin = b;
      a.end = min(a0.end, b + C);
      a.lat_out = a0.lat_out ? a0.lat_out + (b - a0.begin) : nullptr;
      if ((e = chunk(b == a0.begin)) != cudaSuccess) return e;
      b = a.end;
    } while (b < a0.end);
  }
  return cudaSuccess;
}

// chunks launch_eval_thread_b splits a call into (two kernels each)
int eval_thread_chunks(const EvalArgs& a) {
  const uint64_t margin = (uint64_t)kGqBatch * a.grid * (kTThreads / 32);
  if (a.gqcap <= margin) return 1;
  const uint64_t room = a.gqcap - margin;
  if (a.index) return (int)max((uint64_t)1, (a.count + room - 1) / room);
  const uint64_t C = max((uint64_t)1, room / a.block) * (uint64_t)a.block * a.world;
  return (int)max((uint64_t)1, (a.end - a.begin + C - 1) / C);
}

cudaError_t launch_eval_thread(const Cfg& c, const EvalArgs& a, cudaStream_t st) {
  switch (tinstance(c.n, c.mmax)) {
    case 0: return launch_eval_thread_b<32, 32>(c, a, st);
    case 1: return launch_eval_thread_b<64, 64>(c, a, st);
    case 2: return launch_eval_thread_b<128, 64>(c, a, st);
    case 4: return launch_eval_thread_b<64, 16>(c, a, st);
    case 5: return launch_eval_thread_b<128, 16>(c, a, st);
    default: return launch_eval_thread_b<128, 128>(c, a, st);
  }
}

}  // namespace optimus
