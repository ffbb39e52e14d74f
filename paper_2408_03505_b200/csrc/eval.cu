// eval.cu — K2 (one candidate per warp) and K3 (argmin reduction).
//
// For every candidate (encoder plan e, composition N of N_mb into m parts)
// this runs Alg. 2's per-partition body: coarse init,
// OptimizeSchedule(FWD), global ordering, OptimizeSchedule(BWD), lat; and
// Alg. 1's strict-< minimum, ties -> lowest global index (R18).
// All kernel-level placement was hoisted exactly into the chain tables
// (R-FACT, chains.cu), so the per-candidate loop is integer min/max/compare
// work over lanes:
//   lane j (< m)  = encoder pipeline j: c_j, kf_j, its DEV value
//   lane i (< n)  = LLM microbatch slot i: G_i = F_i - L, D_i = T_end - B_i - L,
//                   H(i+1) = sum_j min(c_j, i+1), the moved-EF counts
// Dependency shift (R10): need_i = i - #{moved EF <= G_i}; INF if need_i >
//   sum c; else PRE_EF(t_i) - G_i with t_i = min{t : H(t) >= need_i}.
// Backward (R15): per-pipeline sorted deadlines; slot i's rank within its
//   owner is the number of later slots with the same owner + 1.
#include "optimus_dev.cuh"

namespace optimus {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kEvalThreads = 256;
constexpr int kChunk = 64;  // consecutive candidates per warp work item

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
  // max of int64 via two 32-bit redux: high word, then low word among the winners
  const int hi = (int)(v >> 32);
  const int mh = __reduce_max_sync(FULL, hi);
  const unsigned lo = (unsigned)(v & 0xffffffffu);
  const unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  return (int64_t)(((uint64_t)(uint32_t)mh << 32) | ml);
}

__device__ __forceinline__ unsigned lanemask_le(int k) { return k >= 31 ? FULL : ((2u << k) - 1u); }
__device__ __forceinline__ unsigned lanemask_gt(int k) { return ~lanemask_le(k); }

struct PlanCache {
  int e, P, rt, m, kmax;
  int aj;         // lane j: its PP row a = j div r_t (R7)
  bool strict;    // PRE_EF strictly increasing (pre entries order by (t, j))
  uint64_t first, count;
  const int64_t* devF;
  const int64_t* devB;
  const int64_t* inbF;
  const int64_t* lenF;
  const int64_t* inbB;
  const int64_t* lenB;
  int64_t preEF;   // lane t-1 holds PRE_EF(t)  = end(P-1, t)   (t = lane+1)
  int64_t preBEF;  // lane t-1 holds PREB_EF(t)
};

__device__ void load_plan(const Cfg& c, int e, PlanCache& pc) {
  const PlanDesc& pd = c.plans[e];
  const int lane = threadIdx.x & 31, n = c.n;
  pc.e = e;
  pc.P = pd.P;
  pc.rt = pd.rt;
  pc.m = pd.m;
  pc.kmax = pd.kmax;
  pc.first = pd.first;
  pc.count = pd.count;
  pc.devF = c.tables + pd.devF;
  pc.devB = c.tables + pd.devB;
  pc.inbF = c.tables + pd.inbF;
  pc.lenF = c.tables + pd.lenF;
  pc.inbB = c.tables + pd.inbB;
  pc.lenB = c.tables + pd.lenB;
  const int t = min(lane + 1, n);
  pc.preEF = c.tables[pd.preF + (int64_t)(pd.P - 1) * (n + 1) + t];
  pc.preBEF = c.tables[pd.preB + (int64_t)(pd.P - 1) * (n + 1) + t];
  pc.aj = lane / pd.rt;
  const int64_t prev = __shfl_up_sync(FULL, pc.preEF, 1);
  pc.strict = __all_sync(FULL, lane == 0 || lane >= n || pc.preEF > prev);
}

__device__ int find_plan(const Cfg& c, uint64_t g) {
  for (int e = 0; e < c.E; ++e) {
    const PlanDesc& pd = c.plans[e];
    if (pd.count && g >= pd.first && g < pd.first + pd.count) return e;
  }
  return -1;
}

// Lexicographic unranking of a composition (R17): lane j gets N_j.
__device__ int unrank_lane(const Cfg& c, int n, int m, uint64_t rank) {
  const int lane = threadIdx.x & 31;
  int mine = 0, rem = n, j = 0;
  // every lane walks the same sequence (uniform, no divergence)
  for (; j < m - 1; ++j) {
    const int parts = m - j;
    int x = 1;
    for (; x <= rem - (parts - 1); ++x) {
      const uint64_t cnt = __ldg(&c.binom[(rem - x - 1) * (kMaxNWarp + 1) + (parts - 2)]);
      if (rank < cnt) break;
      rank -= cnt;
    }
    if (lane == j) mine = x;
    rem -= x;
  }
  if (lane == m - 1) mine = rem;
  return mine;
}

// Lexicographic successor (lane j holds N_j); returns false past the last.
__device__ bool next_composition(int m, int& N) {
  const int lane = threadIdx.x & 31;
  // exclusive suffix sum S_j = sum_{k>j} N_k
  int v = lane < m ? N : 0, incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_down_sync(FULL, incl, o);
    if (lane + o < 32) incl += y;
  }
  const int S = incl - v;
  const unsigned b = __ballot_sync(FULL, lane <= m - 2 && S > m - 1 - lane);
  if (!b) return false;
  const int jj = 31 - __clz(b);
  const int Sj = __shfl_sync(FULL, S, jj);
  if (lane == jj) N += 1;
  else if (lane > jj && lane < m - 1) N = 1;
  else if (lane == m - 1) N = Sj - 1 - (m - 2 - jj);
  return true;
}

// Level-boundary mask of the pre multiset: level t (lane t-1 holds H(t) =
// sum_j min(c_j, t) and cnt = #{j : c_j >= t}) occupies the 0-based sorted
// positions [H(t-1), H(t)); the levels 1..max c are all non-empty.
__device__ __forceinline__ unsigned level_mask(int H, int cnt) {
  return __reduce_or_sync(FULL, cnt > 0 ? 1u << (H - cnt) : 0u);
}

// Forward dependency shift (R10): need_i = i - #{moved EF <= G_i}; INF if
// need_i > sum c; else max over need_i > 0 of PRE_EF(t_i) - G_i, with t_i
// the level holding sorted position need_i - 1.
__device__ __forceinline__ int64_t dep_fwd(int n, unsigned B, int Qc, int sumc, int64_t G, int64_t preEF) {
  const int lane = threadIdx.x & 31;
  const int need = lane + 1 - Qc;
  if (__any_sync(FULL, lane < n && need > sumc)) return kInf;
  const int t = __popc(B & lanemask_le(max(need - 1, 0)));
  const int64_t pe = __shfl_sync(FULL, preEF, max(t - 1, 0));  // PRE_EF(t)
  return warp_max64(lane < n && need > 0 ? pe - G : kNegInf);
}

// Backward dependency shift (R15): slot i with owner o, rank r within o.
__device__ __forceinline__ int64_t dep_bwd(int n, int r, int Qcb, int cbo, int64_t D, int64_t preBEF) {
  const int lane = threadIdx.x & 31;
  const int need = r - Qcb;
  if (__any_sync(FULL, lane < n && need > cbo)) return kInf;
  const int64_t pe = __shfl_sync(FULL, preBEF, max(need, 1) - 1);  // PREB_EF(need)
  return warp_max64(lane < n && need > 0 ? pe - D : kNegInf);
}

// Per-warp work counters (warp-uniform), flushed with one atomic per warp:
// candidates, sum m, sum m*iters_f, iters_f, attempts_f, sum m*iters_b,
// iters_b, attempts_b.  The host turns them into algorithmic lane-ops
// (optimus_eval_stats).
struct Stats {
  unsigned v[8];
};

// Base state of the current composition N, carried across lexicographic
// successors: lane j: N_j and its DEV values; lane t-1: cnt(t) = #{j : N_j
// >= t}, H(t) = sum_j min(N_j, t).
struct Comp {
  int N, cnt, H;
  int64_t dvF, dvB;
};

__device__ void comp_init(const Cfg& c, const PlanCache& pc, int N, Comp& s) {
  __shared__ int hist_sm[kEvalThreads / 32][kMaxNWarp + 2];
  const int lane = threadIdx.x & 31, np1 = c.n + 1;
  int* sm = hist_sm[threadIdx.x >> 5];
  const bool isp = lane < pc.m;
  s.N = isp ? N : 0;
  s.dvF = isp ? __ldg(&pc.devF[pc.aj * np1 + N]) : kNegInf;
  s.dvB = isp ? __ldg(&pc.devB[pc.aj * np1 + N]) : kNegInf;
  sm[lane] = 0;
  if (lane < 2) sm[32 + lane] = 0;
  __syncwarp();
  if (isp) atomicAdd(&sm[N], 1);
  __syncwarp();
  int cnt = sm[lane + 1];
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_down_sync(FULL, cnt, o);
    if (lane + o < 32) cnt += y;
  }
  int H = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, H, o);
    if (lane >= o) H += y;
  }
  s.cnt = cnt;
  s.H = H;
  __syncwarp();
}

// Lexicographic successor with the base state kept up to date; the common
// step (last part > 1) moves one microbatch from part m-1 to part m-2.
__device__ bool comp_next(const Cfg& c, const PlanCache& pc, Comp& s) {
  const int lane = threadIdx.x & 31, m = pc.m, np1 = c.n + 1;
  if (m < 2) return false;
  const int y = __shfl_sync(FULL, s.N, m - 1);
  if (y > 1) {
    const int x = __shfl_sync(FULL, s.N, m - 2);
    s.cnt += (lane == x ? 1 : 0) - (lane == y - 1 ? 1 : 0);  // cnt(x+1) += 1, cnt(y) -= 1
    s.H += (lane >= x ? 1 : 0) - (lane >= y - 1 ? 1 : 0);
    if (lane == m - 2 || lane == m - 1) {
      s.N += lane == m - 2 ? 1 : -1;
      s.dvF = __ldg(&pc.devF[pc.aj * np1 + s.N]);
      s.dvB = __ldg(&pc.devB[pc.aj * np1 + s.N]);
    }
    return true;
  }
  int N = s.N;
  if (!next_composition(m, N)) return false;
  comp_init(c, pc, N, s);
  return true;
}

// One candidate: returns lat (uniform across the warp).
__device__ int64_t eval_one(const Cfg& c, const PlanCache& pc, const Comp& base, int64_t G, int64_t D, int64_t T_end,
                            Stats& st) {
  __shared__ int ord_sm[kEvalThreads / 32][kMaxNWarp + 2];
  const int lane = threadIdx.x & 31;
  const int n = c.n, m = pc.m, kmax = pc.kmax, np1 = n + 1;
  const bool isp = lane < m;
  const int aj = pc.aj;
  const int Nj = base.N;
  int* sm = ord_sm[threadIdx.x >> 5];

  // ---------------- coarse init + forward OptimizeSchedule -------------
  int cj = Nj, kf = 0;
  int64_t dv = base.dvF;
  int cnt = base.cnt, H = base.H;
  unsigned B = level_mask(H, cnt);
  int sumc = n, Qc = 0;
  int64_t dep = dep_fwd(n, B, Qc, sumc, G, pc.preEF);
  int64_t Delta;
  int itf = 0, atf = 0, itb = 0, atb = 0;
  for (;;) {
    ++itf;
    const bool valid = isp && cj > 0;
    const int64_t dvv = valid ? dv : kNegInf;
    const int64_t dev = warp_max64(dvv);
    Delta = max((int64_t)0, max(dev, dep));
    if (Delta == 0 || sumc == 0) break;
    const int js = __ffs(__ballot_sync(FULL, valid && dvv == dev)) - 1;  // findCritical, ties -> lowest j (R11)
    const int kfj = __shfl_sync(FULL, kf, js), cjs = __shfl_sync(FULL, cj, js);
    const int as = __shfl_sync(FULL, aj, js);
    if (kfj >= (int)__ldg(&pc.lenF[as])) break;  // ScheduleKernels fails (R12)
    const int64_t EF = __ldg(&pc.inbF[as * kmax + kfj]);
    ++atf;
    const int H2 = H - (lane + 1 >= cjs ? 1 : 0);
    const int cnt2 = cnt - (lane + 1 == cjs ? 1 : 0);
    const unsigned B2 = level_mask(H2, cnt2);
    const int Qc2 = Qc + (EF <= G ? 1 : 0);
    const int64_t dep2 = dep_fwd(n, B2, Qc2, sumc - 1, G, pc.preEF);
    if (dep2 > Delta) break;  // checkEncLLMDep (R13)
    H = H2;
    cnt = cnt2;
    B = B2;
    Qc = Qc2;
    dep = dep2;
    --sumc;
    if (lane == js) {
      --cj;
      ++kf;
      dv = cj > 0 ? __ldg(&pc.devF[aj * np1 + cj]) : kNegInf;
    }
  }
  const int64_t Df = Delta;

  // ---------------- global ordering (R14) -------------------------------
  // owner[i] and r[i] = rank of slot i's deadline within its owner's sorted
  // deadlines = #{later slots of the same owner} + 1
  int owner, r;
  if (sumc == n && pc.strict) {
    // no chain moved: entries are the pre levels, ordered by (t, j)
    const int maxc = __reduce_max_sync(FULL, cj);
    for (int t = 1; t <= maxc; ++t) {
      const unsigned mk = __ballot_sync(FULL, isp && cj >= t);
      const int Hp = t == 1 ? 0 : __shfl_sync(FULL, H, t - 2);
      if (isp && cj >= t) sm[Hp + __popc(mk & (lane ? (0xffffffffu >> (32 - lane)) : 0u))] = lane | ((cj - t + 1) << 8);
    }
    __syncwarp();
    const int vv = sm[lane];
    __syncwarp();
    owner = lane < n ? (vv & 0xff) : 64 + lane;
    r = vv >> 8;
  } else {
    int incl = isp ? Nj : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int off = incl - (isp ? Nj : 0);
    const unsigned segs = __reduce_or_sync(FULL, isp ? (1u << off) : 0u);
    int64_t key = INT64_MAX;
    {
      const int jj = max(__popc(segs & lanemask_le(lane)) - 1, 0);
      const int offj = __shfl_sync(FULL, off, jj);
      const int cjj = __shfl_sync(FULL, cj, jj);
      const int ajj = __shfl_sync(FULL, aj, jj);
      const int local = lane - offj;
      const int64_t pre = __shfl_sync(FULL, pc.preEF, max(local, 0) & 31);  // PRE_EF(local+1)
      if (lane < n) {
        const int64_t val = local < cjj ? pre - Df : __ldg(&pc.inbF[ajj * kmax + (local - cjj)]);
        key = val * 65536 + (int64_t)(jj << 8) + local;
      }
    }
    // bitonic sort of the 32 keys, ascending
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const int64_t other = __shfl_xor_sync(FULL, key, j);
        const bool up = ((lane & j) == 0) == ((lane & k) == 0);  // keep the smaller key
        if ((other < key) == up) key = other;
      }
    owner = lane < n ? (int)((key >> 8) & 0xff) : 64 + lane;
    const unsigned same = __match_any_sync(FULL, owner);
    r = __popc(same & lanemask_gt(lane)) + 1;
  }

  // ---------------- backward OptimizeSchedule (R15) ----------------------
  int cb = Nj, kb = 0;
  int64_t dvb = base.dvB;
  int Qcb = 0, sumcb = n;
  int cbo = __shfl_sync(FULL, cb, owner & 31);
  int64_t depb = dep_bwd(n, r, Qcb, cbo, D, pc.preBEF);
  for (;;) {
    ++itb;
    const bool valid = isp && cb > 0;
    const int64_t dvv = valid ? dvb : kNegInf;
    const int64_t dev = warp_max64(dvv);
    Delta = max((int64_t)0, max(dev, depb));
    if (Delta == 0 || sumcb == 0) break;
    const int js = __ffs(__ballot_sync(FULL, valid && dvv == dev)) - 1;
    const int kfj = __shfl_sync(FULL, kf, js), kbj = __shfl_sync(FULL, kb, js);
    const int as = __shfl_sync(FULL, aj, js);
    const int64_t rowoff = (int64_t)as * (kmax + 1) + kfj;
    if (kbj >= (int)__ldg(&pc.lenB[rowoff])) break;
    const int64_t EFb = __ldg(&pc.inbB[rowoff * kmax + kbj]);
    ++atb;
    const bool mine = owner == js;
    const int Qcb2 = Qcb + (mine && EFb <= D ? 1 : 0);
    const int cbo2 = cbo - (mine ? 1 : 0);
    const int64_t dep2 = dep_bwd(n, r, Qcb2, cbo2, D, pc.preBEF);
    if (dep2 > Delta) break;
    Qcb = Qcb2;
    cbo = cbo2;
    depb = dep2;
    --sumcb;
    if (lane == js) {
      --cb;
      ++kb;
      dvb = cb > 0 ? __ldg(&pc.devB[aj * np1 + cb]) : kNegInf;
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
  return T_end + Df + Delta;  // R16
}

__device__ __forceinline__ void better(int64_t lat, uint64_t g, int64_t& bl, uint64_t& bg) {
  if (lat < bl || (lat == bl && g < bg)) { bl = lat; bg = g; }
}

template <bool EXPLICIT>
__global__ void __launch_bounds__(kEvalThreads) k2_eval(Cfg c, EvalArgs A) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = c.n;
  const int64_t T_end = c.scal[1];
  const int64_t G = lane < n ? c.F[lane] - c.L : 0;          // EF_i + L <= F_i
  const int64_t D = lane < n ? T_end - c.B[lane] - c.L : 0;  // EB_i >= B_i + L (mirrored)
  int64_t bl = INT64_MAX;
  uint64_t bg = UINT64_MAX;
  PlanCache pc;
  pc.e = -1;
  Stats st = {{0, 0, 0, 0, 0, 0, 0, 0}};
  Comp cs;
  const uint64_t nchunks = (A.count + kChunk - 1) / kChunk;
  for (;;) {
    unsigned long long ch = 0;
    if (lane == 0) ch = atomicAdd(A.counter, 1ull);
    ch = __shfl_sync(FULL, ch, 0);
    if (ch >= nchunks) break;
    if (EXPLICIT) {
      const uint64_t i0 = ch * kChunk;
      for (uint64_t i = i0; i < min(i0 + kChunk, A.count); ++i) {
        const uint64_t g = A.index[i];
        const int e = find_plan(c, g);
        if (e < 0) continue;
        if (e != pc.e) load_plan(c, e, pc);
        comp_init(c, pc, unrank_lane(c, n, pc.m, g - pc.first), cs);
        const int64_t lat = eval_one(c, pc, cs, G, D, T_end, st);
        if (A.lat_out && lane == 0) A.lat_out[i] = lat;
        better(lat, g, bl, bg);
      }
    } else {
      // this rank's chunk -> global indices (block-cyclic over ranks)
      const uint64_t pos = ch * kChunk;
      const uint64_t rb = pos / A.block, offb = pos % A.block;
      uint64_t g = A.begin + (rb * A.world + A.rank) * (uint64_t)A.block + offb;
      uint64_t gend = min(g + kChunk, A.end);
      if (g >= gend) continue;
      int e = find_plan(c, g);
      if (e != pc.e) load_plan(c, e, pc);
      comp_init(c, pc, unrank_lane(c, n, pc.m, g - pc.first), cs);
      for (;;) {
        const int64_t lat = eval_one(c, pc, cs, G, D, T_end, st);
        if (A.lat_out && lane == 0) A.lat_out[g - A.begin] = lat;
        better(lat, g, bl, bg);
        if (++g >= gend) break;
        if (g >= pc.first + pc.count) {  // next plan with candidates
          e = find_plan(c, g);
          load_plan(c, e, pc);
          comp_init(c, pc, unrank_lane(c, n, pc.m, 0), cs);
        } else {
          comp_next(c, pc, cs);
        }
      }
    }
  }
  if (lane == 0 && A.stats) {
#pragma unroll
    for (int i = 0; i < 8; ++i) atomicAdd(&A.stats[i], (unsigned long long)st.v[i]);
  }
  // block argmin -> partials
  __shared__ long long bl_sm[kEvalThreads / 32];
  __shared__ unsigned long long bg_sm[kEvalThreads / 32];
  if (lane == 0) { bl_sm[warp] = bl; bg_sm[warp] = bg; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t l = INT64_MAX;
    uint64_t gg = UINT64_MAX;
    for (int w = 0; w < kEvalThreads / 32; ++w) better(bl_sm[w], bg_sm[w], l, gg);
    A.partials[2 * blockIdx.x] = l;
    A.partials[2 * blockIdx.x + 1] = (int64_t)gg;
  }
}

__global__ void k3_reduce(EvalArgs A) {
  __shared__ long long l_sm[256];
  __shared__ unsigned long long g_sm[256];
  int64_t l = INT64_MAX;
  uint64_t g = UINT64_MAX;
  for (int i = threadIdx.x; i < A.grid; i += blockDim.x) better(A.partials[2 * i], (uint64_t)A.partials[2 * i + 1], l, g);
  for (int i = threadIdx.x; i < A.grid2; i += blockDim.x)  // K2 mode 1's general kernel
    better(A.partials2[2 * i], (uint64_t)A.partials2[2 * i + 1], l, g);
  l_sm[threadIdx.x] = l;
  g_sm[threadIdx.x] = g;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      int64_t a = l_sm[threadIdx.x];
      uint64_t b = g_sm[threadIdx.x];
      better(l_sm[threadIdx.x + s], g_sm[threadIdx.x + s], a, b);
      l_sm[threadIdx.x] = a;
      g_sm[threadIdx.x] = b;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    A.best2[0] = l_sm[0];
    A.best2[1] = l_sm[0] == INT64_MAX ? -1 : (int64_t)g_sm[0];
    *A.counter = 0;  // ready for the next eval on this stream
  }
  for (int e = threadIdx.x; e < A.nplans; e += blockDim.x) A.pclaim[e] = 0;
}

}  // namespace

int eval_grid(int sms) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k2_eval<false>, kEvalThreads, 0);
  return max(1, per) * sms;
}

cudaError_t launch_eval(const Cfg& c, const EvalArgs& a, cudaStream_t st, int* launches) {
  if (a.ev0) cudaEventRecord(a.ev0, st);
  if (a.mode == 1) {
    const cudaError_t e = launch_eval_thread(c, a, st);
    if (e != cudaSuccess) return e;
  } else if (a.index) {
    k2_eval<true><<<a.grid, kEvalThreads, 0, st>>>(c, a);
  } else {
    k2_eval<false><<<a.grid, kEvalThreads, 0, st>>>(c, a);
  }
  if (a.ev1) cudaEventRecord(a.ev1, st);
  k3_reduce<<<1, 256, 0, st>>>(a);
  if (launches) *launches += a.mode == 1 ? 1 + 2 * eval_thread_chunks(a) : 2;
  return cudaGetLastError();
}

}  // namespace optimus
