// chains.cu — per-plan tables and K1, the kernel-level first-fit chain tables.
//
// PAPER.md §4.2: InitSchedule (coarse: encoder forwards before
// the LLM, backwards after it) and ScheduleKernels/AssignKernels: move one
// microbatch of an encoder pipeline into the bubbles interleaved with LLM
// compute at kernel granularity, upstream stage before downstream stage for
// forward, reverse order for backward, encoder comm never in TP bubbles
// (Design decision 3).  §4.4: kernels of all encoder
// branches are scheduled as one encoder.  Readings R6-R9, R12, R15 and the
// exact factorisation R-FACT: every device instance is only
// touched by its own pipeline's moves and TP siblings share geometry, so the
// k-th forward chain of ANY pipeline of PP-row a ends at INB_F[a][k], and
// the k-th backward chain after kf forward chains at INB_B[a][kf][k].
//
// K1 (k1_chains), one launch, one block per unit, one warp per encoder stage:
//   forward units (plan, row): successive forward chains until the first
//   failure, publishing a versioned snapshot of the fill state after each;
//   backward units (plan, row, kf): mirrored backward chains on top of
//   forward version kf, started as soon as it is published.  The last E
//   blocks build the per-plan tables K2 reads: coarse GPipe fill tables
//   PRE_F / PRE_B (R9), the critical-path tables DEV_F / DEV_B (R11) and
//   their order ranks.
// First fit: while kernels fit the current interval of their resource, 32
// kernels are placed at once by a max-plus scan over the warp; otherwise a
// window of 32 consecutive intervals lives in registers (lane i = interval
// base+i) and one ballot tests all 32, skipping blocks that end before the
// ready time or cannot hold the kernel.
#include <algorithm>
#include <cstdio>

#include "optimus_dev.cuh"

namespace optimus {
namespace {

constexpr unsigned FULL = 0xffffffffu;

#ifndef K1_SCALAR
#define K1_SCALAR 4  // kernels placed one by one before a 32-wide batch is tried
#endif
#ifndef K1_GROUPS
#define K1_GROUPS 2  // most chains of one unit in flight (1: one chain after the other; config 2 build: 1 -> 0.99 ms, 2 -> 0.70, 4 -> 0.71, 12 -> 0.72)
#endif

#ifdef K1_TRACE  // development instrumentation: per K1 work item start / end (globaltimer ns), item, block
#define K1_STATS
__device__ unsigned long long g_k1trace[16384][4];
__device__ unsigned long long g_k1stats[4096][32][14];
#endif

#ifdef K1_STATS  // development instrumentation (OPTIMUS_NVCC_EXTRA=-DK1_STATS): per-warp event counts
// 0 place_stage prologs, 1 unit setup, 2 slow placements, 3 vwait cycles,
// 4 placement loop, 5 upstream-stage waits, 6 total, 7 slow cycles, 8 publish, 9 fast rounds,
// 10 window advances, 11 advance cycles, 12 slow found in the current window, 13 flush cycles
__shared__ unsigned long long k1st[32][14];
__shared__ int k1item;
#define K1ST(i, v) do { if ((threadIdx.x & 31) == 0) k1st[threadIdx.x >> 5][i] += (v); } while (0)
#ifndef K1ST_MIN
#define K1ST_MIN 150000
#endif
#else
#define K1ST(i, v) do { } while (0)
#endif

// ------------------------------------------------------------ plan tables
__device__ void plan_tables(const Cfg& c, int e) {
  const PlanDesc pd = c.plans[e];
  if (pd.count == 0) return;
  const int P = pd.P, n = c.n;
  __shared__ int64_t tau_f[kMaxP], tau_b[kMaxP];
  // stage sums tau[s] over the stage's layers of every branch (R8)
  for (int s = threadIdx.x; s < P; s += blockDim.x) {
    int64_t tf = 0, tb = 0;
    for (int b = 0; b < c.nb; ++b) {
      const int L = c.blayers[b];
      const int nl = (s + 1) * L / P - s * L / P;
      const int idf = enc_list_id(b, pd.ti, c.ntp, 0), idb = enc_list_id(b, pd.ti, c.ntp, 1);
      int64_t sf = 0, sb = 0;
      for (int i = c.loff[idf]; i < c.loff[idf + 1]; ++i) sf += c.lns[i];
      for (int i = c.loff[idb]; i < c.loff[idb + 1]; ++i) sb += c.lns[i];
      tf += nl * sf;
      tb += nl * sb;
    }
    tau_f[s] = tf;
    tau_b[s] = tb;
  }
  __syncthreads();
  int64_t* preF = c.tables + pd.preF;
  int64_t* preB = c.tables + pd.preB;
  // GPipe fill from 0 (R9): end(s,x) = max(end(s,x-1), end(s-1,x)+p2p) + tau[s]
  if (threadIdx.x < 2) {
    int64_t* E = threadIdx.x == 0 ? preF : preB;
    const int64_t* tau = threadIdx.x == 0 ? tau_f : tau_b;
    for (int s = 0; s < P; ++s) E[s * (n + 1)] = 0;
    for (int x = 1; x <= n; ++x)
      for (int s = 0; s < P; ++s) {
        int64_t st = E[s * (n + 1) + x - 1];
        if (s > 0) st = max(st, E[(s - 1) * (n + 1) + x] + c.enc_p2p);
        E[s * (n + 1) + x] = st + tau[s];
      }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // K2's fast path needs PRE_EF strictly increasing (the pre entries of a level then order by j)
    bool strict = true;
    for (int t = 1; t < n; ++t) strict = strict && preF[(P - 1) * (n + 1) + t + 1] > preF[(P - 1) * (n + 1) + t];
    c.tables[pd.pflags] = strict ? 1 : 0;
  }
  // DEV[a][cnt] = max_s(end(s, cnt) - w_{aP+s}) (forward; w' = T_end - z backward)
  const int64_t T_end = c.scal[1];
  for (int i = threadIdx.x; i < pd.rp * (n + 1); i += blockDim.x) {
    const int a = i / (n + 1), cnt = i % (n + 1);
    int64_t df = kNegInf, db = kNegInf;
    if (cnt > 0)
      for (int s = 0; s < P; ++s) {
        df = max(df, preF[s * (n + 1) + cnt] - c.w[a * P + s]);
        db = max(db, preB[s * (n + 1) + cnt] - (T_end - c.z[a * P + s]));
      }
    c.tables[pd.devF + i] = df;
    c.tables[pd.devB + i] = db;
  }
  __syncthreads();
  // order ranks of the DEV entries (K2's findCritical compares 32-bit keys
  // rank << 7 | 127 - j): rank = #{entries < v}, >= rp for cnt > 0, 0 at cnt 0
  const int V = pd.rp * (n + 1);
  uint32_t* key = reinterpret_cast<uint32_t*>(c.tables + pd.devK);
  for (int i = threadIdx.x; i < 2 * V; i += blockDim.x) {
    const int64_t* dv = c.tables + (i < V ? pd.devF : pd.devB);
    const int ii = i < V ? i : i - V;
    const int64_t v = dv[ii];
    uint32_t r = 0;
    if (ii % (n + 1) != 0)
      for (int q = 0; q < V; ++q) r += dv[q] < v ? 1u : 0u;
    key[i] = r;
  }
  __syncthreads();
  // per-pipeline keys with the lowest-j tie rule folded in (K2 mode 1)
  uint64_t* kj = reinterpret_cast<uint64_t*>(c.tables + pd.kj);
  for (int i = threadIdx.x; i < pd.m * (n + 1); i += blockDim.x) {
    const int j = i / (n + 1), cnt = i % (n + 1), a = j / pd.rt;
    const uint32_t lo = (uint32_t)(127 - j);
    const uint32_t kf = key[a * (n + 1) + cnt] << 7 | lo, kb = key[V + a * (n + 1) + cnt] << 7 | lo;
    kj[i] = (uint64_t)kf | (uint64_t)kb << 32;
  }
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(FULL, v, o));
  return v;
}

// ------------------------------------------------------ first-fit machinery
// Register view of one (LLM stage, resource) interval list of one unit.
// Snapshots of the forward fill state are versioned per 32-interval block:
// version v = the state after v forward chains, own[b] = the version whose
// buffer holds block b (-1: never written, fill = start).
// Forward (M = false): intervals as in the template; chain k writes every
// block it touches into version k+1's buffer and points own[b] there, so
// version k+1 = own map after chain k, no copies.  Mirrored (M = true,
// R15): interval i' is real interval count-1-i' in time t -> T_end - t; its
// end is T_end minus the fill pointer of forward version kf (own = kf's map);
// the unit's own fill state lives in `fill`, valid in the blocks marked in wm.
template <bool M>
struct VR {
  int count, ver;        // forward: version this chain writes
  uint32_t* wm;          // mirror: 32-blocks of fill written so far (smem)
  const int64_t* S;
  const int64_t* H;
  int64_t* fill;         // mirror: this unit's fill array
  int64_t* bm;           // largest capacity hi - lo of each 32-block (smem; lowered as blocks fill)
  int16_t* own;          // owner version per 32-block (smem): forward current, mirror kf's (-1: never written)
  int64_t* snap0;        // this list in version 0's buffer; version o at + o * vstride
  int64_t vstride;
  int64_t T_end;
  // chain pipeline (several chains of one stage in flight on different
  // warps, chain k trailing chain k-1): a 32-block is "passed" by a chain
  // once its window has left it; later chains only read passed blocks.
  volatile int* pprev;   // blocks passed by chain k-1 on this list (smem; nullptr: chain k-1 is complete)
  volatile int* pmine;   // blocks passed by this chain (nullptr: nobody trails it)
  const volatile int* stopp;  // first void chain of the unit
  int16_t* gown;         // forward: version k+1's published owner map of this list (passed blocks written on pass)
  int passed, k;
  __device__ __forceinline__ int64_t hi_at(int i) const {
    if (!M) return H[i];
    const int r = count - 1 - i;
    const int o = own[r >> 5];
    return T_end - (o < 0 ? S[r] : __ldcg(&snap0[o * vstride + r]));  // published by another block: L2
  }
  __device__ __forceinline__ int64_t start_at(int i) const { return M ? T_end - H[count - 1 - i] : S[i]; }
  __device__ __forceinline__ int64_t lo_at(int i) const {
    if (M) return ((wm[i >> 10] >> ((i >> 5) & 31)) & 1u) ? fill[i] : start_at(i);
    const int o = own[i >> 5];
    return o < 0 ? S[i] : snap0[o * vstride + i];
  }
};

// A window of 32 consecutive intervals in registers (lane l = interval
// base+l), and the "current" interval of
// the chain-stage as warp-uniform scalars (cur = -1: none): the interval
// the last kernel of this resource went into; every earlier interval ends
// at or before `ready` from then on, so first fit can start there.
struct Win {
  int base, cur;
  bool dirty;
  int64_t lo, hi;
  int64_t clo, chi;  // fill pointer / end of interval cur (clo authoritative); both -inf when cur < 0
};

template <bool M>
__device__ __forceinline__ void win_fetch(const VR<M>& V, int b, int64_t& lo, int64_t& hi) {
  const int i = b + (threadIdx.x & 31);
  if (i < V.count) {
    hi = V.hi_at(i);
    lo = V.lo_at(i);
  } else {
    hi = kNegInf;
    lo = 0;
  }
}

// Blocks [V.passed, nb) of this list are final for the chains that trail
// this one: publish their owners (forward) and the pass count.  Every lane
// fences its own stores (window flushes) before lane 0 releases the count.
template <bool M>
__device__ __forceinline__ void vpass(VR<M>& V, int nb) {
  if (nb <= V.passed) return;
  const int lane = threadIdx.x & 31;
  if (!M && V.gown)
    for (int b = V.passed + lane; b < nb; b += 32) V.gown[b] = V.own[b];
  if (V.pmine) {
    __threadfence_block();
    __syncwarp();
    if (lane == 0) *V.pmine = nb;
  }
  V.passed = nb;
}

// Wait until the previous chain has passed block b of this list (false:
// this chain is void, an earlier one failed).  Decisions on lane 0's reads.
template <bool M>
__device__ __forceinline__ bool vwait(const VR<M>& V, int b) {
  if (!V.pprev) return true;
  if (__shfl_sync(FULL, *V.pprev, 0) > b) {
    __threadfence_block();
    return true;
  }
#ifdef K1_STATS
  const long long tv0 = clock64();
#endif
  for (;;) {
    if (__shfl_sync(FULL, *V.pprev, 0) > b) break;
    if (V.k >= __shfl_sync(FULL, *V.stopp, 0)) return false;
    __nanosleep(32);
  }
#ifdef K1_STATS
  K1ST(3, clock64() - tv0);
#endif
  __threadfence_block();
  return true;
}

template <bool M>
__device__ __forceinline__ bool win_open(VR<M>& V, Win& w, int b) {
  w.base = b;
  w.cur = -1;
  w.clo = kNegInf;  // no current interval: the fast path's max-plus terms must stay inert
  w.chi = kNegInf;
  w.dirty = false;
  // the blocks before the ready time are never touched by this chain: their
  // owners are final once the previous chain has passed them
  if (!vwait(V, b >> 5)) return false;
  vpass(V, b >> 5);
  win_fetch(V, b, w.lo, w.hi);
  return true;
}

__device__ __forceinline__ void win_sync_cur(Win& w) {
  if (w.cur >= 0 && (threadIdx.x & 31) == w.cur - w.base) w.lo = w.clo;
  w.cur = -1;
  w.clo = kNegInf;
  w.chi = kNegInf;
}

template <bool M>
__device__ __forceinline__ void win_flush(VR<M>& V, Win& w) {
  win_sync_cur(w);
  if (!w.dirty) return;
  const int lane = threadIdx.x & 31;
  const int i = w.base + lane;
  OPT_CHECK(M || (V.ver >= 0 && V.ver <= 32767));
  if (i < V.count) (M ? V.fill : V.snap0 + V.ver * V.vstride)[i] = w.lo;  // forward: the whole block
  // the block's largest capacity, an upper bound for the skip test: one
  // 32-bit redux over capacities saturated at 2^32 - 1 (read back as +inf)
  const int64_t c64 = i < V.count ? w.hi - w.lo : 0;
  const unsigned c32 = __reduce_max_sync(FULL, c64 >= 0xFFFFFFFFll ? 0xFFFFFFFFu : (unsigned)max(c64, (int64_t)0));
  if (lane == 0) {
    V.bm[w.base >> 5] = c32 == 0xFFFFFFFFu ? kInf : (int64_t)c32;
    if (M) atomicOr(&V.wm[w.base >> 10], 1u << ((w.base >> 5) & 31));  // chains in flight share the word
    else V.own[w.base >> 5] = (int16_t)V.ver;
  }
  w.dirty = false;
  __syncwarp();
}

// Place one kernel of duration d at or after `ready` (R12): the first
// interval (time order) with end > ready and max(ready, lo) + d <= end.
// Slow path, after the kernel did not fit the current interval (the fast
// path in place_stage): a ballot over the 32-interval window, then the
// following windows.
// first 32-block >= b that ends after `ready` and whose largest capacity
// can hold d (CI if none): ci = block ends, bm = block capacities
__device__ __forceinline__ int next_block(const int64_t* ci, const int64_t* bm, int CI, int b, int64_t ready,
                                          int64_t d) {
  const int lane = threadIdx.x & 31;
  for (; b < CI; b += 32) {
    const int k = b + lane;
    const unsigned m = __ballot_sync(FULL, k < CI && ci[k] > ready && bm[k] >= d);
    if (m) return b + __ffs(m) - 1;
  }
  return CI;
}

template <bool M>
__device__ __forceinline__ bool place_slow(VR<M>& V, Win& w, int64_t d, int64_t& ready, const int64_t* ci,
                                           const int64_t* bm, int CI) {
  win_sync_cur(w);
  for (;;) {
    const int blk = w.base >> 5;
    {  // the window first (registers; the block indices only filter)
      const int64_t x = max(ready, w.lo);
      const unsigned b = __ballot_sync(FULL, x + d <= w.hi);  // (d >= 1: such an end is after ready)
      if (b) {
#ifdef K1_STATS
        K1ST(12, 1);
#endif
        const int f = __ffs(b) - 1;
        const int64_t xf = __shfl_sync(FULL, x, f);
        w.chi = __shfl_sync(FULL, w.hi, f);
        w.cur = w.base + f;
        w.clo = xf + d;
        w.dirty = true;
        ready = xf + d;
        return true;
      }
    }
#ifdef K1_STATS
    const long long ta0 = clock64();
#endif
    win_flush(V, w);
#ifdef K1_STATS
    K1ST(13, clock64() - ta0);
    K1ST(10, 1);
#endif
    const int nb = next_block(ci, bm, CI, blk + 1, ready, d);
    if (32 * nb >= V.count) return false;
    if (!vwait(V, nb)) return false;
    vpass(V, nb);
    // (no prefetch of the following window: measured 7-9% slower builds)
    win_fetch(V, 32 * nb, w.lo, w.hi);
    w.base = 32 * nb;
#ifdef K1_STATS
    K1ST(11, clock64() - ta0);
#endif
  }
}

// Per-warp shared memory of a K1 unit.
struct UnitSm {
  int64_t* seq;       // [NK] flattened kernels of the whole encoder, stage-major: duration | comm << 63
  int* soff;          // [P+1] stage offsets into seq
  uint32_t* wm;       // [P][2][MW] blocks of the fill arrays written so far
  int64_t* ci;        // [P][2][CI] coarse index: end of the last interval of each 32-block
  int64_t* bm;        // [P][2][CI] largest base capacity of each 32-block (this orientation)
  int16_t* own;       // [P][2][CI] snapshot block owners (forward: current, mirror: snapshot kf); int16: versions reach kmax = n - m + 1 <= 128
  int64_t* pe;        // [NK + P] stage-local exclusive duration prefix: pe[s + x] = sum of d over [soff[s], x), x in [soff[s], soff[s+1]]
  uint32_t* lcp;      // [NK] 1 + the last comm kernel <= x of its stage (low 16 bits), 1 + the last compute kernel (high; 0: none)
  int CI, MW;
};

__host__ __device__ inline size_t unit_smem_bytes(int NK, int P, int CI) {
  const int MW = (CI + 31) / 32;
  return ((size_t)NK * 8 + 15) / 16 * 16 + ((size_t)(P + 1) * 4 + 15) / 16 * 16 +
         ((size_t)P * 2 * MW * 4 + 15) / 16 * 16 + (size_t)P * 2 * CI * 8 * 2 + ((size_t)P * 2 * CI * 2 + 15) / 16 * 16 +
         (size_t)(NK + P) * 8 + ((size_t)NK * 4 + 15) / 16 * 16;
}

__device__ UnitSm carve(unsigned char* p, int NK, int P, int CI) {
  UnitSm u;
  u.seq = (int64_t*)p;
  p += ((size_t)NK * 8 + 15) / 16 * 16;
  u.soff = (int*)p;
  p += ((size_t)(P + 1) * 4 + 15) / 16 * 16;
  u.wm = (uint32_t*)p;
  p += ((size_t)P * 2 * ((CI + 31) / 32) * 4 + 15) / 16 * 16;
  u.ci = (int64_t*)p;
  u.bm = u.ci + (size_t)P * 2 * CI;
  p += (size_t)P * 2 * CI * 8 * 2;
  u.own = (int16_t*)p;
  p += ((size_t)P * 2 * CI * 2 + 15) / 16 * 16;
  u.pe = (int64_t*)p;
  p += (size_t)(NK + P) * 8;
  u.lcp = (uint32_t*)p;
  u.CI = CI;
  u.MW = (CI + 31) / 32;
  return u;
}

// Flatten stage s of the encoder's kernel lists (R8; §4.4 branches in order,
// P:478) for plan pd (one warp per stage): stage s = for each branch its layers
// [floor(sL/P), floor((s+1)L/P)); mirrored time runs each layer's backward
// list in reverse (R15).
__device__ void build_seq(const Cfg& c, const PlanDesc& pd, bool mirror, UnitSm& U, int s) {
  const int lane = threadIdx.x & 31, P = pd.P;
  int pos = 0;  // kernels of the stages before s
  for (int t = 0; t < s; ++t)
    for (int b = 0; b < c.nb; ++b) {
      const int L = c.blayers[b], id = enc_list_id(b, pd.ti, c.ntp, mirror ? 1 : 0);
      pos += ((t + 1) * L / P - t * L / P) * (c.loff[id + 1] - c.loff[id]);
    }
  if (lane == 0) U.soff[s] = pos;
  for (int b = 0; b < c.nb; ++b) {
    const int L = c.blayers[b];
    const int l0 = s * L / P, l1 = (s + 1) * L / P;
    const int id = enc_list_id(b, pd.ti, c.ntp, mirror ? 1 : 0);
    const int off = c.loff[id], len = c.loff[id + 1] - off;
    const int cnt = (l1 - l0) * len;
    for (int x = lane; x < cnt; x += 32) {
      const int k = x % len;
      const int kk = mirror ? off + len - 1 - k : off + k;
      U.seq[pos + x] = c.lns[kk] | (c.lkind[kk] != 0 ? INT64_MIN : 0);
    }
    pos += cnt;
  }
  if (lane == 0 && s == P - 1) U.soff[P] = pos;
  __syncwarp();
  // the fast path's run tables: duration prefix and last kernel of each kind
  const int i0 = U.soff[s];
  int64_t carry = 0;
  int lc = 0, lp = 0;
  if (lane == 0) U.pe[s + i0] = 0;
  for (int b = i0; b < pos; b += 32) {
    const int x = b + lane;
    const int64_t v = x < pos ? U.seq[x] : 0;
    int64_t d = v & INT64_MAX;
    int mc = x < pos && v < 0 ? x - i0 + 1 : 0, mp = x < pos && v >= 0 ? x - i0 + 1 : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t t = __shfl_up_sync(FULL, d, o);
      const int tc = __shfl_up_sync(FULL, mc, o), tp = __shfl_up_sync(FULL, mp, o);
      if (lane >= o) {
        d += t;
        mc = max(mc, tc);
        mp = max(mp, tp);
      }
    }
    mc = max(mc, lc);
    mp = max(mp, lp);
    if (x < pos) {
      U.pe[s + x + 1] = carry + d;
      U.lcp[x] = (uint32_t)(mc ? mc + i0 : 0) | (uint32_t)(mp ? mp + i0 : 0) << 16;
    }
    carry += __shfl_sync(FULL, d, 31);
    lc = __shfl_sync(FULL, mc, 31);
    lp = __shfl_sync(FULL, mp, 31);
  }
}

// view of list r of stage s of row a; fill = this unit's fill array of the
// stage, snap0 = the stage's snapshot version-0 array (both [icapc + icapm])
template <bool M>
__device__ VR<M> make_view(const Cfg& c, const PlanDesc& pd, int a, int s, int r, int64_t* fill, const UnitSm& U,
                           int64_t* snap0, int ver) {
  const int q = a * pd.P + s;
  VR<M> V;
  V.count = r == 0 ? c.ncomp[q] : c.ncomm[q];
  V.S = r == 0 ? c.comp_lo + (int64_t)q * c.icapc : c.comm_lo + (int64_t)q * c.icapm;
  V.H = r == 0 ? c.comp_hi + (int64_t)q * c.icapc : c.comm_hi + (int64_t)q * c.icapm;
  V.fill = fill ? fill + (r ? c.icapc : 0) : nullptr;
  V.ver = ver;
  V.bm = U.bm + (2 * s + r) * U.CI;
  V.own = U.own + (2 * s + r) * U.CI;
  V.snap0 = snap0 + (r ? c.icapc : 0);
  V.vstride = (int64_t)pd.rp * pd.P * (c.icapc + c.icapm);
  V.wm = U.wm + (2 * s + r) * U.MW;
  V.T_end = c.scal[1];
  V.pprev = nullptr;
  V.pmine = nullptr;
  V.stopp = nullptr;
  V.gown = nullptr;
  V.passed = 0;
  V.k = 0;
  return V;
}

// coarse index of one view: ci[k] = end of interval min(count-1, 32k+31)
template <bool M>
__device__ void build_ci(const VR<M>& V, int64_t* ci, int CI) {
  const int nblk = (V.count + 31) / 32;
  for (int k = threadIdx.x & 31; k < CI; k += 32)
    ci[k] = k < nblk ? V.hi_at(min(V.count - 1, 32 * k + 31)) : kInf;
  __syncwarp();
}

// first 32-block whose last interval ends after `ready`
__device__ __forceinline__ int ci_search(const int64_t* ci, int CI, int64_t ready) {
  const int lane = threadIdx.x & 31;
  for (int b = 0; b < CI; b += 32) {
    const int k = b + lane;
    const unsigned m = __ballot_sync(FULL, k < CI && ci[k] > ready);
    if (m) return 32 * (b + __ffs(m) - 1);
  }
  return 32 * CI;
}

struct UnitCtx {
  int P, a;
  int64_t* fill;   // mirror: this unit's fill state, slot-major: [P][icapc + icapm]
  int64_t* snap0;  // version 0 of this row's forward snapshots, same layout (version o at + o * rp * P * icap)
};

// Place stage s of one chain starting at `ready` (R12; mirrored lists and
// w' = T_end - z for backward, R15).  On success *end = the stage's last
// kernel end.  On failure the stage's fill state may be partly modified
// (the unit stops).
// REC (schedule emission, NEXT-1): rec[q] = {stage, comm, start, end} of
// kernel q of the chain (q = index in the flattened stage-major list).
// the chain pipeline's links of one chain-stage (per resource r)
struct Link {
  volatile int* pprev[2];      // pass counts of chain k-1 (nullptr: no wait)
  volatile int* pmine[2];      // this chain's pass counts (nullptr: nobody trails)
  int16_t* gown[2];            // forward: version k+1's owner maps (nullptr: not published)
  const volatile int* stopp;
};

template <bool M, bool REC = false>
__device__ bool place_stage(const Cfg& c, const PlanDesc& pd, const UnitCtx& X, UnitSm& U, int s, int k,
                            int64_t ready, int64_t* end, const Link& lk, int64_t* rec = nullptr) {
#ifdef K1_STATS
  const long long tp0 = clock64();
#endif
  const int icap = c.icapc + c.icapm;
  int64_t* f0 = M ? X.fill + (int64_t)s * icap : nullptr;
  int64_t* s0 = X.snap0 + (int64_t)s * icap;
  VR<M> V0 = make_view<M>(c, pd, X.a, s, 0, f0, U, s0, k + 1);
  VR<M> V1 = make_view<M>(c, pd, X.a, s, 1, f0, U, s0, k + 1);
  V0.pprev = lk.pprev[0];
  V1.pprev = lk.pprev[1];
  V0.pmine = lk.pmine[0];
  V1.pmine = lk.pmine[1];
  V0.gown = lk.gown[0];
  V1.gown = lk.gown[1];
  V0.stopp = V1.stopp = lk.stopp;
  V0.passed = V1.passed = 0;
  V0.k = V1.k = k;
  Win w0, w1;  // compute-free / comm-free windows of this stage
  if (!win_open(V0, w0, ci_search(U.ci + (2 * s) * U.CI, U.CI, ready))) return false;
  if (!win_open(V1, w1, ci_search(U.ci + (2 * s + 1) * U.CI, U.CI, ready))) return false;
  const int i1 = U.soff[s + 1];
  const int64_t* seq = U.seq;
  const int i0 = U.soff[s];
  int i = i0;
#ifdef K1_STATS
  const long long t0 = clock64();
  K1ST(0, t0 - tp0);
#endif
  for (;;) {
    // scalar steps first (warp-uniform, the sequential definition): after a
    // slow placement the next kernels often leave the current intervals
    // within a few steps, where a 32-wide batch would mostly be wasted
    bool fits = true;
    int64_t vmiss = 0;  // the kernel the scalar steps could not place (fits == false)
#pragma unroll 1
    for (int ns = 0; ns < K1_SCALAR && i < i1; ++ns) {
      const int64_t v = seq[i];
      const bool comm = v < 0;
      const int64_t d = v & INT64_MAX;
      const int64_t e = max(ready, comm ? w1.clo : w0.clo) + d;
      if (e > (comm ? w1.chi : w0.chi)) {
        fits = false;
        vmiss = v;
        break;
      }
      if (REC && (threadIdx.x & 31) == 0) {
        int64_t* r = rec + (int64_t)i * 4;
        r[0] = s;
        r[1] = comm;
        r[2] = e - d;
        r[3] = e;
      }
      ready = e;
      if (comm) w1.clo = e;
      else w0.clo = e;
      ++i;
    }
    // fast path, runs of up to 32 kernels (lane l = kernel i+l): inside the
    // current intervals every kernel starts at the previous end (the fill
    // pointers never pass `ready`), so kernel l ends at ready + pe(i, l] and
    // "kernels i..x all fit" holds iff the last kernel of each kind up to x
    // ends within its resource's current interval (ends only grow with x):
    // two table lookups per lane and one ballot per run of 32
    const int64_t* pe = U.pe + s;
    while (fits && i < i1) {
      const int lane = threadIdx.x & 31;
      const int64_t base = ready - pe[i];
      const int64_t thc = w1.chi - base, thp = w0.chi - base;
      const int x = i + lane;
      bool ok = true;
      if (x < i1) {
        const uint32_t q = U.lcp[x];
        const int lc = (int)(q & 0xffffu) - 1, lp = (int)(q >> 16) - 1;
        ok = (lc < i || pe[lc + 1] <= thc) && (lp < i || pe[lp + 1] <= thp);
      }
      const unsigned okm = __ballot_sync(FULL, ok);
      K1ST(9, 1);
      const int nv = min(32, i1 - i);
      const int f = min(nv, okm == FULL ? 32 : __ffs(~okm) - 1);  // kernels [i, i+f) fit
      if (REC && lane < f) {
        int64_t* r = rec + (int64_t)(i + lane) * 4;
        r[0] = s;
        r[1] = U.seq[i + lane] < 0;
        r[2] = base + pe[i + lane];
        r[3] = base + pe[i + lane + 1];
      }
      if (f > 0) {
        const uint32_t q = U.lcp[i + f - 1];
        const int lc = (int)(q & 0xffffu) - 1, lp = (int)(q >> 16) - 1;
        if (lc >= i) w1.clo = base + pe[lc + 1];
        if (lp >= i) w0.clo = base + pe[lp + 1];
        ready = base + pe[i + f];
        i += f;
      }
      if (f < nv) break;
    }
    if (i >= i1) break;
    const int64_t v = fits ? seq[i] : vmiss;
    K1ST(2, 1);
#ifdef K1_STATS
    const long long ts0 = clock64();
#endif
    const bool ok = v < 0 ? place_slow(V1, w1, v & INT64_MAX, ready, U.ci + (2 * s + 1) * U.CI,
                                       U.bm + (2 * s + 1) * U.CI, U.CI)
                          : place_slow(V0, w0, v & INT64_MAX, ready, U.ci + (2 * s) * U.CI, U.bm + (2 * s) * U.CI,
                                       U.CI);
    if (REC && ok && (threadIdx.x & 31) == 0) {
      int64_t* r = rec + (int64_t)i * 4;
      r[0] = s;
      r[1] = v < 0;
      r[2] = ready - (v & INT64_MAX);
      r[3] = ready;
    }
#ifdef K1_STATS
    K1ST(7, clock64() - ts0);
#endif
    if (!ok) return false;
    ++i;
  }
#ifdef K1_STATS
  K1ST(4, clock64() - t0);
#endif
  win_flush(V0, w0);
  win_flush(V1, w1);
  // the rest of both lists: final once the previous chain is complete
  if (!vwait(V0, U.CI - 1) || !vwait(V1, U.CI - 1)) return false;
  vpass(V0, U.CI);
  vpass(V1, U.CI);
  __syncwarp();
  *end = ready;
  return true;
}


struct K1Launch {
  int NK, Pmax, CI, KM;  // KM = max kmax
};

__host__ __device__ inline size_t k1_smem_bytes(const K1Launch& L) {
  return unit_smem_bytes(L.NK, L.Pmax, L.CI) + (size_t)L.Pmax * L.KM * (8 + 4 + 8) + 16;
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

// One K1 unit per block, warp w = stage s of chain group g (s = w mod P,
// g = w div P, G = W div P groups): group g places chains k = g, g + G, ...
// A wavefront over stages and a pipeline over chains: chain k of stage s
// starts when chain k of stage s-1 has ended (shared-memory flags), and
// reads a 32-interval block of a list only once chain k-1 has passed it
// (its window left the block: the block's fill state and owner are final).
// Chain k's kernels never start before chain k-1's (same ready times or
// later, fill pointers only advance), so it trails chain k-1 and ends after
// it.  Forward (M = false): successive chains on fresh instances; chain k
// publishes version k+1 of each stage's fill state (the owner map, block by
// block as it passes them; flags[k+1] counts the stages), and the unit ends
// with flags[0] = 1.  Backward (M = true): mirrored chains on top of forward
// version kf, started once it is published (or skipped when the forward
// unit ended with fewer chains).  Both stop at the first failure; chains
// after it are void (they quit at their next wait).
template <bool M, bool REC = false>
__device__ __forceinline__ void k1_unit(const Cfg& c, const K1Launch& L, int e, int a, int kf, int klimit = 1 << 30,
                                        int64_t* rec = nullptr) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int stop_at;  // first chain index known to fail (chains >= it are void)
  __shared__ int go;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const PlanDesc pd = c.plans[e];
  const int P = pd.P, icap = c.icapc + c.icapm;
  // chain groups: REC replays one chain after the other
  const int G = REC ? 1 : max(1, min((int)(blockDim.x >> 5) / P, K1_GROUPS));
  const int s = w % P, g = w / P;
  int* flags = c.k1flags + pd.flag_base + (int64_t)a * (pd.kmax + 1);
  OPT_CHECK(pd.flag_base + (int64_t)(a + 1) * (pd.kmax + 1) <= c.nflags && kf <= pd.kmax);
  if (M && kf > 0) {  // wait for forward version kf of this row
    if (threadIdx.x == 0) {
      // poll relaxed (an acquire load invalidates the SM's L1, which the
      // running units on this SM read their intervals through); acquire once
      int ok;
      for (;;) {
        if (ld_relaxed(&flags[kf]) >= P) { ok = 1; break; }
        if (ld_relaxed(&flags[0]) != 0) { ok = ld_acquire(&flags[kf]) >= P; break; }
        __nanosleep(256);
      }
      (void)ld_acquire(&flags[kf]);
      go = ok;
    }
    __syncthreads();
    if (!go) return;  // uniform: no pipeline of this row has kf forward chains
  }
  const bool active = g < G;  // warps beyond G * P only join the barriers
  UnitSm U = carve(dsm, L.NK, L.Pmax, L.CI);
  const size_t ub = unit_smem_bytes(L.NK, L.Pmax, L.CI);
  volatile int* status = (volatile int*)(dsm + ub);  // [P][KM]: 0 pending, 1 done, 2 failed
  const size_t sb = (((size_t)L.Pmax * L.KM * 4 + 15) & ~size_t(15));
  volatile int64_t* endv = (volatile int64_t*)(dsm + ub + sb);
  volatile int* prog = (volatile int*)(dsm + ub + sb + (size_t)L.Pmax * L.KM * 8);  // [P][KM][2] blocks passed
  volatile int* stop = &stop_at;
  auto slot = [&](int k, int st) {
    OPT_CHECK(k >= 0 && k <= pd.kmax && st >= 0 && st < P);
    return pd.slot_base + ((int64_t)k * pd.rp + a) * P + st;
  };
#ifdef K1_STATS
  const long long tk0 = clock64();
  for (int i = threadIdx.x; i < 32 * 14; i += blockDim.x) k1st[i / 14][i % 14] = 0;
  __syncthreads();
#endif
  if (active && g == 0) build_seq(c, pd, M, U, s);
  for (int i = threadIdx.x; i < P * L.KM; i += blockDim.x) status[i] = 0;
  for (int i = threadIdx.x; i < 2 * P * L.KM; i += blockDim.x) prog[i] = 0;
  if (threadIdx.x == 0) stop_at = pd.kmax;
  int64_t* snap0 = c.snap + slot(0, 0) * icap;
  if (active && g == 0) {
    for (int r = 0; r < 2; ++r) {
      // block owners: forward starts untouched; mirror loads snapshot kf's map
      int16_t* own = U.own + (2 * s + r) * U.CI;
      const int16_t* gown = c.snap_own + (slot(kf, s) * 2 + r) * c.ci_n;
      for (int b = lane; b < U.CI; b += 32) own[b] = (M && kf > 0) ? (int16_t)__ldcg((const short*)&gown[b]) : (int16_t)-1;
      for (int b = lane; b < U.MW; b += 32) U.wm[(2 * s + r) * U.MW + b] = 0u;
      __syncwarp();
      VR<M> V = make_view<M>(c, pd, a, s, r, nullptr, U, snap0 + (int64_t)s * icap, 0);
      build_ci(V, U.ci + (2 * s + r) * U.CI, U.CI);
      const int64_t* bsrc = c.bmax + (((int64_t)(a * P + s) * 2 + r) * 2 + (M ? 1 : 0)) * c.ci_n;
      for (int k = lane; k < U.CI; k += 32) U.bm[(2 * s + r) * U.CI + k] = bsrc[k];
    }
  }
  __syncthreads();
  if (active) {
    const UnitCtx X{P, a, M ? c.bfill + slot(kf, 0) * icap : nullptr, snap0};
#ifdef K1_STATS
    K1ST(1, clock64() - tk0);
#endif
    const int64_t T_end = c.scal[1];
    const int q = a * P + s;
    const int64_t ws = M ? T_end - c.z[q] : c.w[q];
    const int kend = min(pd.kmax, klimit);
    // every decision on a value another warp may change is taken from lane
    // 0's read (broadcast), so that the warp never splits before its
    // full-mask collectives
    for (int k = g; k < kend; k += G) {
      if (k >= __shfl_sync(FULL, *stop, 0)) break;
      int64_t ready = ws;
      if (s > 0) {  // wait for chain k of the upstream stage
        int st;
        bool quit = false;
#ifdef K1_STATS
        const long long tw0 = clock64();
#endif
        for (;;) {
          st = __shfl_sync(FULL, status[(s - 1) * L.KM + k], 0);
          if (st != 0) break;
          if (k >= __shfl_sync(FULL, *stop, 0)) { quit = true; break; }
          __nanosleep(20);
        }
#ifdef K1_STATS
        K1ST(5, clock64() - tw0);
#endif
        if (quit || st == 2) {
          if (lane == 0) {
            atomicMin(&stop_at, k);
            status[s * L.KM + k] = 2;
          }
          break;
        }
        __threadfence_block();
        ready = max(endv[(s - 1) * L.KM + k] + c.enc_p2p, ws);
      }
      Link lk;
      for (int r = 0; r < 2; ++r) {
        lk.pprev[r] = (G > 1 && k > 0) ? prog + ((int64_t)s * L.KM + k - 1) * 2 + r : nullptr;
        lk.pmine[r] = (G > 1 && k + 1 < kend) ? prog + ((int64_t)s * L.KM + k) * 2 + r : nullptr;
        lk.gown[r] = (!M && !REC) ? c.snap_own + (slot(k + 1, s) * 2 + r) * c.ci_n : nullptr;
      }
      lk.stopp = stop;
      int64_t end;
      if (!place_stage<M, REC>(c, pd, X, U, s, k, ready, &end, lk,
                               REC ? rec + (int64_t)k * U.soff[P] * 4 : nullptr)) {
        if (lane == 0) {
          atomicMin(&stop_at, k);
          status[s * L.KM + k] = 2;
        }
        break;
      }
      if (lane == 0) {
        endv[s * L.KM + k] = end;
        __threadfence_block();
        status[s * L.KM + k] = 1;
        if (!REC && s == P - 1) {
          if (M) c.tables[pd.inbB + ((int64_t)a * (pd.kmax + 1) + kf) * pd.kmax + k] = end;
          else c.tables[pd.inbF + (int64_t)a * pd.kmax + k] = end;
        }
      }
      __syncwarp();
      if (!M && !REC) {  // publish version k+1 of this stage (its owner map went out block by block)
#ifdef K1_STATS
        const long long tq0 = clock64();
#endif
        __threadfence();  // this lane's block and map stores before the count
        __syncwarp();
        if (lane == 0) atomicAdd(&flags[k + 1], 1);
#ifdef K1_STATS
        K1ST(8, clock64() - tq0);
#endif
      }
    }
  }
#ifdef K1_STATS
  K1ST(6, clock64() - tk0);
#ifdef K1_TRACE
  if (lane == 0 && k1item < 4096)
    for (int q = 0; q < 14; ++q) g_k1stats[k1item][w][q] = k1st[w][q];
#else
  if (active && lane == 0 && k1st[w][6] > K1ST_MIN)
    printf("K1ST M=%d e=%d a=%d kf=%d s=%d/%d g=%d/%d prolog=%llu setup=%llu slow=%llu x=%llu pcyc=%llu wcyc=%llu tot=%llu scyc=%llu\n",
           (int)M, e, a, kf, s, P, g, G, k1st[w][0], k1st[w][1], k1st[w][2], k1st[w][3], k1st[w][4], k1st[w][5], k1st[w][6], k1st[w][7]);
#endif
#endif
  __syncthreads();
  if (REC) return;  // emission replay: the build's tables stay as they are
  if (threadIdx.x == 0) {  // chains completed by every stage
    int k = 0;
    while (k < pd.kmax && status[(P - 1) * L.KM + k] == 1) ++k;
    if (M) {
      c.tables[pd.lenB + (int64_t)a * (pd.kmax + 1) + kf] = k;
    } else {
      c.tables[pd.lenF + a] = k;
      __threadfence();
      atomicExch(&flags[0], 1);  // forward unit done: versions > lenF never come
    }
  }
  if (!M) {  // for K2's forward dependency test: the first slot each chain end can precede
    __syncthreads();
    const int len = (int)c.tables[pd.lenF + a];
    for (int k = threadIdx.x; k < len; k += blockDim.x) {
      const int64_t ef = c.tables[pd.inbF + (int64_t)a * pd.kmax + k];
      int lo = 0, hi = c.n;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (c.F[mid] - c.L >= ef) hi = mid; else lo = mid + 1;
      }
      c.tables[pd.bpF + (int64_t)a * pd.kmax + k] = lo + 1;
    }
  }
}

// Schedule emission (NEXT-1): replay the first klimit chains of one unit
// (forward: kf < 0; backward on forward version kf) with every kernel's
// placement recorded; the build's tables and snapshots are only read.
template <bool M>
__global__ void k1_record(Cfg c, K1Launch L, int e, int a, int kf, int klimit, int64_t* rec) {
  k1_unit<M, true>(c, L, e, a, M ? kf : 0, klimit, rec);
}

// Scheduling efficiency of one explained candidate (NEXT-1, §5.3.2 P:665,
// reading R-EFF): xo = optimus_explain's device output.  out (zeroed) gets
// [in-bubble work with the moves, without them (coarse only), total].
// Coarse microbatch x of stage s occupies [fill[s][x] - tau[s], fill[s][x])
// of the plan's GPipe tables (R9); only its part inside the natural bubble
// [0, w_q) (mirrored [0, T_end - z_q)) counts; moved chains count in full.
__global__ void k_eff(Cfg c, const int64_t* xo, unsigned long long* out) {
  const int n = c.n, e = (int)xo[5], m = (int)xo[6];
  const int64_t* N = xo + 8 + 2 * n;
  const int64_t* cf = N + m;
  const int64_t* cb = N + 2 * m;
  const PlanDesc pd = c.plans[e];
  const int P = pd.P;
  __shared__ int64_t tau_f[kMaxP], tau_b[kMaxP];
  for (int s = threadIdx.x; s < P; s += blockDim.x) {  // stage sums (R8), as the plan tables
    int64_t tf = 0, tb = 0;
    for (int b = 0; b < c.nb; ++b) {
      const int L = c.blayers[b], nl = (s + 1) * L / P - s * L / P;
      const int idf = enc_list_id(b, pd.ti, c.ntp, 0), idb = enc_list_id(b, pd.ti, c.ntp, 1);
      int64_t sf = 0, sb = 0;
      for (int i = c.loff[idf]; i < c.loff[idf + 1]; ++i) sf += c.lns[i];
      for (int i = c.loff[idb]; i < c.loff[idb + 1]; ++i) sb += c.lns[i];
      tf += nl * sf;
      tb += nl * sb;
    }
    tau_f[s] = tf;
    tau_b[s] = tb;
  }
  __syncthreads();
  const int64_t T_end = c.scal[1];
  const int64_t* fillF = c.tables + pd.preF;
  const int64_t* fillB = c.tables + pd.preB;
  auto coarse = [&](const int64_t* fill, int s, int64_t tau, int64_t bubble, int64_t count) {
    int64_t t = 0;
    for (int x = 1; x <= count; ++x) {
      const int64_t hi = fill[s * (n + 1) + x], lo = hi - tau;
      t += max((int64_t)0, min(hi, bubble) - max(lo, (int64_t)0));
    }
    return t;
  };
  for (int idx = threadIdx.x; idx < m * P; idx += blockDim.x) {
    const int j = idx / P, s = idx % P, q = (j / pd.rt) * P + s;
    const int64_t pre = c.w[q], post = T_end - c.z[q], tf = tau_f[s], tb = tau_b[s];
    const int64_t fine = (N[j] - cf[j]) * tf + (N[j] - cb[j]) * tb;
    atomicAdd(&out[0], (unsigned long long)(fine + coarse(fillF, s, tf, pre, cf[j]) + coarse(fillB, s, tb, post, cb[j])));
    atomicAdd(&out[1], (unsigned long long)(coarse(fillF, s, tf, pre, N[j]) + coarse(fillB, s, tb, post, N[j])));
    atomicAdd(&out[2], (unsigned long long)(N[j] * (tf + tb)));
  }
}

// Persistent: every block takes work items in list order (forward units
// first, so a backward unit only ever waits on items already taken by
// running blocks) until the list is exhausted, and counts each finished
// item in its plan's pdone (release).  The launch lets the dependent K2
// start at once (programmatic dependent launch): K2 takes a plan's
// candidates once pdone says its tables are complete.
// Block size 32 * p: register budgets per p range (MAXT threads, MINB blocks per SM).
__device__ __forceinline__ void k1_body(const Cfg& c, const K1Launch& L) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef PDL_PROBE  // development: K1 / K2 timeline (globaltimer ns) in the sync words
  unsigned long long* probe = reinterpret_cast<unsigned long long*>(c.k1next) + 1;
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&probe[0], t);
  }
#endif
  __shared__ int item;
  for (;;) {
    if (threadIdx.x == 0) item = atomicAdd(c.k1next, 1);
    __syncthreads();
    const int it = item;
    __syncthreads();
    if (it >= c.k1_total) {
#ifdef PDL_PROBE
      if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(&probe[1], t);
      }
#endif
      break;
    }
    const uint32_t u = (uint32_t)c.k1units[it];
    const int type = u >> 30, e = (u >> 16) & 0x3FFF, a = (u >> 8) & 255, kf = u & 255;
#ifdef K1_TRACE
    if (threadIdx.x == 0) k1item = it;
    unsigned long long tt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt0));
#endif
    if (type == 2) plan_tables(c, e);
    else if (type == 0) k1_unit<false>(c, L, e, a, 0);
    else k1_unit<true>(c, L, e, a, kf);
    __syncthreads();
#ifdef K1_TRACE
    if (threadIdx.x == 0 && it < 16384) {
      unsigned long long tt1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt1));
      g_k1trace[it][0] = tt0;
      g_k1trace[it][1] = tt1;
      g_k1trace[it][2] = u;
      g_k1trace[it][3] = blockIdx.x;
    }
#endif
    if (threadIdx.x == 0) {
      __threadfence();
#ifdef PDL_PROBE
      if (atomicAdd(&c.pdone[e], 1) == plan_items(c.plans[e]) - 1) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        printf("PLANREADY e=%d P=%d count=%llu at +%llu us\n", e, c.plans[e].P, (unsigned long long)c.plans[e].count,
               (t - probe[0]) / 1000);
      }
#else
      atomicAdd(&c.pdone[e], 1);
#endif
    }
  }
}

template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k1_chains(Cfg c, K1Launch L) { k1_body(c, L); }

#ifndef K1_MAXNREG
#define K1_MAXNREG 112
#endif
// 12-warp blocks (p <= 12), one per SM: registers capped below the whole
// file (164 uncapped, no spills at 112) so that K2 blocks fit beside the K1
// block while both run
__global__ void __maxnreg__(K1_MAXNREG) k1_chains12(Cfg c, K1Launch L) { k1_body(c, L); }

template <typename F>
static void k1_attrs(F f) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  // the whole unified L1 as shared memory: K2 blocks must fit next to the
  // K1 blocks while both run
#ifndef K1_NO_CARVEOUT
  cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
#endif
}

// K1 block: 12 warps up to p = 12 (every stage count P <= p gets 12 / P
// chain groups), then 16 and 32
__host__ __device__ inline int k1_threads(int p) { return p <= 12 ? 384 : (p <= 16 ? 512 : 1024); }
#ifndef K1_PER_SM
#define K1_PER_SM 1
#endif

template <typename F>
static int k1_grid_b(F f, const Cfg& c, size_t smem) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, k1_threads(c.p), smem);
  // one block per SM (occupancy permitting) leaves room on every SM for K2
  // blocks, which start as soon as the first plans are complete
  return std::max(1, std::min(c.k1_total, std::max(1, std::min(per, K1_PER_SM)) * c.sms));
}

}  // namespace


// K1 dynamic shared memory per block for the problem's sizes (checked at load)
size_t k1_smem_for(int nk, int p, int ci, int kmax_all) {
  K1Launch L;
  L.NK = std::max(1, nk);
  L.Pmax = p;
  L.CI = ci;
  L.KM = std::max(1, kmax_all);
  return k1_smem_bytes(L);
}

cudaError_t launch_eff(const Cfg& c, const int64_t* d_explain, unsigned long long* d_out, cudaStream_t st) {
  k_eff<<<1, 128, 0, st>>>(c, d_explain, d_out);
  return cudaGetLastError();
}

cudaError_t launch_record(const Cfg& c, int e, int a, int kf, int klimit, int64_t* d_rec, cudaStream_t st) {
  K1Launch L;
  L.NK = c.nk_max;
  L.Pmax = c.p;
  L.CI = (std::max(c.icapc, c.icapm) + 31) / 32;
  L.KM = std::max(1, c.kmax_all);
  const size_t smem = k1_smem_bytes(L);
  if (kf < 0) k1_record<false><<<1, 32 * c.p, smem, st>>>(c, L, e, a, 0, klimit, d_rec);
  else k1_record<true><<<1, 32 * c.p, smem, st>>>(c, L, e, a, kf, klimit, d_rec);
  return cudaGetLastError();
}

// large dynamic shared memory opt-in of every K1 variant (once per device, capi's device_info)
void chains_attrs() {
  k1_attrs(k1_chains12);
  k1_attrs(k1_chains<512, 1>);
  k1_attrs(k1_chains<1024, 1>);
  cudaFuncSetAttribute(k1_record<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k1_record<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
}

static K1Launch k1_launch_of(const Cfg& c) {
  K1Launch L;
  L.NK = c.nk_max;
  L.Pmax = c.p;
  L.CI = (std::max(c.icapc, c.icapm) + 31) / 32;
  L.KM = std::max(1, c.kmax_all);
  return L;
}

// persistent K1 grid for this problem (computed once at load)
int k1_grid(const Cfg& c) {
  const size_t smem = k1_smem_bytes(k1_launch_of(c));
  if (c.p <= 12) return k1_grid_b(k1_chains12, c, smem);
  if (c.p <= 16) return k1_grid_b(k1_chains<512, 1>, c, smem);
  return k1_grid_b(k1_chains<1024, 1>, c, smem);
}

cudaError_t launch_chain_tables(const Cfg& c, cudaStream_t st, int* launches) {
  const K1Launch L = k1_launch_of(c);
  const size_t smem = k1_smem_bytes(L);
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  if (launches) *launches += 1;
  const int grid = c.k1_grid;
  const int nt = k1_threads(c.p);
  if (c.p <= 12) k1_chains12<<<grid, nt, smem, st>>>(c, L);
  else if (c.p <= 16) k1_chains<512, 1><<<grid, nt, smem, st>>>(c, L);
  else k1_chains<1024, 1><<<grid, nt, smem, st>>>(c, L);
  return cudaGetLastError();
}

}  // namespace optimus

#ifdef K1_TRACE
extern "C" int optimus_debug_k1trace(void* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, optimus::g_k1trace, (size_t)n * 32);
}
extern "C" int optimus_debug_k1stats(void* out) {
  return (int)cudaMemcpyFromSymbol(out, optimus::g_k1stats, sizeof(optimus::g_k1stats));
}
extern "C" int optimus_debug_k1reset() {
  static unsigned long long z[16384][4];
  return (int)cudaMemcpyToSymbol(optimus::g_k1trace, z, sizeof(z));
}
#endif
