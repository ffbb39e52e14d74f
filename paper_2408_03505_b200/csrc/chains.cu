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
// k_plan_tables: one block per plan — stage sums, coarse GPipe fill tables
//   PRE_F / PRE_B (R9) and the critical-path tables DEV_F / DEV_B (R11).
// k1_forward:  one warp per (plan, row): successive forward chains until the
//   first failure; snapshots the fill state after each chain.
// k1_backward: one warp per (plan, row, kf): mirrored backward chains on top
//   of forward snapshot kf.
// First fit is warp-cooperative: a window of 32 consecutive intervals lives
// in registers (lane i = interval base+i), one ballot tests all 32.
#include <algorithm>

#include "optimus_dev.cuh"

namespace optimus {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// ------------------------------------------------------------ plan tables
__global__ void k_plan_tables(Cfg c) {
  const int e = blockIdx.x;
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
  // rank << 5 | 31 - j): rank = #{entries < v}, >= rp for cnt > 0, 0 at cnt 0
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
}

// ------------------------------------------------------ first-fit machinery
// Register view of one (LLM stage, resource) interval list of one unit.
// Forward (M = false): intervals as in the template; fill = this unit's fill
// pointers, valid below hw.  Mirrored (M = true, R15): interval i' is real
// interval count-1-i' in time t -> T_end - t; its end is T_end minus the
// forward fill pointer of forward snapshot kf (valid below hwf).
template <bool M>
struct VR {
  int count, hw, hwf;
  const int64_t* S;
  const int64_t* H;
  int64_t* fill;
  const int64_t* snapf;
  int64_t T_end;
  __device__ __forceinline__ int64_t hi_at(int i) const {
    if (!M) return H[i];
    const int r = count - 1 - i;
    return T_end - (r < hwf ? snapf[r] : S[r]);
  }
  __device__ __forceinline__ int64_t start_at(int i) const { return M ? T_end - H[count - 1 - i] : S[i]; }
  __device__ __forceinline__ int64_t lo_at(int i) const { return i < hw ? fill[i] : start_at(i); }
};

// A window of 32 consecutive intervals in registers (lane l = interval
// base+l) plus the prefetched next window, and the "current" interval of
// the chain-stage as warp-uniform scalars (cur = -1: none): the interval
// the last kernel of this resource went into; every earlier interval ends
// at or before `ready` from then on, so first fit can start there.
struct Win {
  int base, cur;
  bool dirty;
  int64_t lo, hi, nlo, nhi;
  int64_t clo, chi;  // fill pointer / end of interval cur (clo authoritative)
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

template <bool M>
__device__ __forceinline__ void win_open(const VR<M>& V, Win& w, int b) {
  w.base = b;
  w.cur = -1;
  w.dirty = false;
  win_fetch(V, b, w.lo, w.hi);
  win_fetch(V, b + 32, w.nlo, w.nhi);
}

__device__ __forceinline__ void win_sync_cur(Win& w) {
  if (w.cur >= 0 && (threadIdx.x & 31) == w.cur - w.base) w.lo = w.clo;
  w.cur = -1;
}

template <bool M>
__device__ __forceinline__ void win_flush(VR<M>& V, Win& w) {
  win_sync_cur(w);
  if (!w.dirty) return;
  const int lane = threadIdx.x & 31;
  for (int i = V.hw + lane; i < w.base; i += 32) V.fill[i] = V.start_at(i);  // gap fill
  const int i = w.base + lane;
  if (i < V.count) V.fill[i] = w.lo;
  V.hw = max(V.hw, min(V.count, w.base + 32));
  w.dirty = false;
  __syncwarp();
}

// Place one kernel of duration d at or after `ready` (R12): the first
// interval (time order) with end > ready and max(ready, lo) + d <= end.
// Fast path: the current interval (uniform scalars); else a ballot over the
// 32-interval window, then the following windows.
template <bool M>
__device__ __forceinline__ bool place(VR<M>& V, Win& w, int64_t d, int64_t& ready) {
  if (w.cur >= 0) {
    const int64_t x = max(ready, w.clo);
    if (x + d <= w.chi) {
      w.clo = x + d;
      ready = x + d;
      return true;
    }
    win_sync_cur(w);
  }
  for (;;) {
    const int64_t x = max(ready, w.lo);
    const unsigned b = __ballot_sync(FULL, w.hi > ready && x + d <= w.hi);
    if (b) {
      const int f = __ffs(b) - 1;
      const int64_t xf = __shfl_sync(FULL, x, f);
      w.chi = __shfl_sync(FULL, w.hi, f);
      w.cur = w.base + f;
      w.clo = xf + d;
      w.dirty = true;
      ready = xf + d;
      return true;
    }
    win_flush(V, w);
    if (w.base + 32 >= V.count) return false;
    w.base += 32;
    w.lo = w.nlo;
    w.hi = w.nhi;
    win_fetch(V, w.base + 32, w.nlo, w.nhi);
  }
}

// Per-warp shared memory of a K1 unit.
struct UnitSm {
  int64_t* seq_d;     // [NK] flattened kernel durations of the whole encoder, stage-major
  uint8_t* seq_k;     // [NK] kinds
  int* soff;          // [P+1] stage offsets into seq
  int* hw;            // [2P] valid fill prefix per (stage, resource)
  int64_t* ci;        // [P][2][CI] coarse index: end of the last interval of each 32-block
  int CI;
};

__host__ __device__ inline size_t unit_smem_bytes(int NK, int P, int CI) {
  return ((size_t)NK * 8 + 15) / 16 * 16 + ((size_t)NK + 15) / 16 * 16 + ((size_t)(P + 1) * 4 + 15) / 16 * 16 +
         ((size_t)2 * P * 4 + 15) / 16 * 16 + (size_t)P * 2 * CI * 8;
}

__device__ UnitSm carve(unsigned char* p, int NK, int P, int CI) {
  UnitSm u;
  u.seq_d = (int64_t*)p;
  p += ((size_t)NK * 8 + 15) / 16 * 16;
  u.seq_k = p;
  p += ((size_t)NK + 15) / 16 * 16;
  u.soff = (int*)p;
  p += ((size_t)(P + 1) * 4 + 15) / 16 * 16;
  u.hw = (int*)p;
  p += ((size_t)2 * P * 4 + 15) / 16 * 16;
  u.ci = (int64_t*)p;
  u.CI = CI;
  return u;
}

// Flatten the encoder's stage kernel lists (R8; §4.4 branches in order,
// P:478) for plan pd: stage s = for each branch its layers
// [floor(sL/P), floor((s+1)L/P)); mirrored time runs each layer's backward
// list in reverse (R15).
__device__ void build_seq(const Cfg& c, const PlanDesc& pd, bool mirror, UnitSm& U) {
  const int lane = threadIdx.x & 31, P = pd.P;
  int pos = 0;
  for (int s = 0; s < P; ++s) {
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
        U.seq_d[pos + x] = c.lns[kk];
        U.seq_k[pos + x] = (uint8_t)c.lkind[kk];
      }
      pos += cnt;
    }
  }
  if (lane == 0) U.soff[P] = pos;
  __syncwarp();
}

template <bool M>
__device__ VR<M> make_view(const Cfg& c, const PlanDesc& pd, int a, int s, int r, int64_t* fill,
                           const int64_t* snapf, int hwf, int hw) {
  const int q = a * pd.P + s;
  VR<M> V;
  V.count = r == 0 ? c.ncomp[q] : c.ncomm[q];
  V.S = r == 0 ? c.comp_lo + (int64_t)q * c.icapc : c.comm_lo + (int64_t)q * c.icapm;
  V.H = r == 0 ? c.comp_hi + (int64_t)q * c.icapc : c.comm_hi + (int64_t)q * c.icapm;
  V.fill = fill;
  V.snapf = snapf;
  V.hwf = hwf;
  V.hw = hw;
  V.T_end = c.scal[1];
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
  int64_t* fill;        // this unit's fill state, slot-major: [P][icapc + icapm]
  const int64_t* snap;  // mirror: forward snapshot kf, same layout
  const int* snap_hw;   // mirror: [P][2] (nullptr -> all 0)
};

// Place stage s of one chain starting at `ready` (R12; mirrored lists and
// w' = T_end - z for backward, R15).  On success *end = the stage's last
// kernel end.  On failure the stage's fill state may be partly modified
// (the unit stops).
template <bool M>
__device__ bool place_stage(const Cfg& c, const PlanDesc& pd, const UnitCtx& X, UnitSm& U, int s, int64_t ready,
                            int64_t* end) {
  const int icap = c.icapc + c.icapm;
  int64_t* f0 = X.fill + (int64_t)s * icap;
  const int64_t* s0 = M ? X.snap + (int64_t)s * icap : nullptr;
  VR<M> V0 = make_view<M>(c, pd, X.a, s, 0, f0, s0, X.snap_hw ? X.snap_hw[2 * s] : 0, U.hw[2 * s]);
  VR<M> V1 = make_view<M>(c, pd, X.a, s, 1, f0 + c.icapc, M ? s0 + c.icapc : nullptr,
                          X.snap_hw ? X.snap_hw[2 * s + 1] : 0, U.hw[2 * s + 1]);
  Win w0, w1;  // compute-free / comm-free windows of this stage
  win_open(V0, w0, ci_search(U.ci + (2 * s) * U.CI, U.CI, ready));
  win_open(V1, w1, ci_search(U.ci + (2 * s + 1) * U.CI, U.CI, ready));
  const int i0 = U.soff[s], i1 = U.soff[s + 1];
  bool ok = true;
  int64_t d = i0 < i1 ? U.seq_d[i0] : 0;
  int kind = i0 < i1 ? U.seq_k[i0] : 0;
  for (int i = i0; i < i1 && ok; ++i) {
    const int64_t dn = U.seq_d[min(i + 1, i1 - 1)];  // prefetch the next kernel
    const int kn = U.seq_k[min(i + 1, i1 - 1)];
    ok = kind == 0 ? place(V0, w0, d, ready) : place(V1, w1, d, ready);
    d = dn;
    kind = kn;
  }
  if (!ok) return false;
  win_flush(V0, w0);
  win_flush(V1, w1);
  if ((threadIdx.x & 31) == 0) { U.hw[2 * s] = V0.hw; U.hw[2 * s + 1] = V1.hw; }
  __syncwarp();
  *end = ready;
  return true;
}

__device__ bool decode_row_unit(const Cfg& c, int64_t u, bool with_kf, int& e, int& a, int& kf) {
  for (e = 0; e < c.E; ++e) {
    const PlanDesc& pd = c.plans[e];
    if (pd.count == 0) continue;
    const int64_t nu = (int64_t)pd.rp * (with_kf ? pd.kmax + 1 : 1);
    if (u < nu) {
      if (with_kf) { a = (int)(u / (pd.kmax + 1)); kf = (int)(u % (pd.kmax + 1)); }
      else { a = (int)u; kf = 0; }
      return true;
    }
    u -= nu;
  }
  return false;
}

struct K1Launch {
  int NK, Pmax, CI, KM;  // KM = max kmax
};

__host__ __device__ inline size_t k1_smem_bytes(const K1Launch& L) {
  return unit_smem_bytes(L.NK, L.Pmax, L.CI) + (size_t)L.Pmax * L.KM * (8 + 4) + 16;
}

// One K1 unit per block, one warp per encoder stage s (a wavefront over
// chains): chain k of stage s starts when chain k of stage s-1 has ended
// (shared-memory flags) and chain k-1 of stage s is done (program order).
// Forward (M = false): successive chains on fresh instances, fill state of
// every stage snapshotted after every chain.  Backward (M = true): mirrored
// chains on top of forward snapshot kf.  Both stop at the first failure.
template <bool M>
__global__ void k1_chains(Cfg c, int64_t units, K1Launch L) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ int stop_at;  // first chain index known to fail (chains >= it are void)
  const int s = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int e, a, kf;
  if (!decode_row_unit(c, blockIdx.x, M, e, a, kf)) return;  // uniform over the block
  const PlanDesc pd = c.plans[e];
  const int P = pd.P, icap = c.icapc + c.icapm;
  if (M && kf > (int)c.tables[pd.lenF + a]) return;  // uniform: no pipeline of this row has kf forward chains
  const bool active = s < P;  // warps beyond this plan's P only join the barriers
  UnitSm U = carve(dsm, L.NK, L.Pmax, L.CI);
  const size_t ub = unit_smem_bytes(L.NK, L.Pmax, L.CI);
  volatile int* status = (volatile int*)(dsm + ub);  // [P][KM]: 0 pending, 1 done, 2 failed
  volatile int64_t* endv = (volatile int64_t*)(dsm + ub + (((size_t)L.Pmax * L.KM * 4 + 15) & ~size_t(15)));
  volatile int* stop = &stop_at;
  auto slot = [&](int k, int st) { return pd.slot_base + ((int64_t)k * pd.rp + a) * P + st; };
  if (s == 0) build_seq(c, pd, M, U);
  for (int i = threadIdx.x; i < P * L.KM; i += blockDim.x) status[i] = 0;
  if (threadIdx.x == 0) stop_at = pd.kmax;
  const int64_t* snap = M ? c.snap + slot(kf, 0) * icap : nullptr;
  const int* snap_hw = (M && kf > 0) ? c.snap_hw + slot(kf, 0) * 2 : nullptr;
  if (active) {
    if (lane < 2) U.hw[2 * s + lane] = 0;
    for (int r = 0; r < 2; ++r) {
      VR<M> V = make_view<M>(c, pd, a, s, r, nullptr, M ? snap + (int64_t)s * icap + (r ? c.icapc : 0) : nullptr,
                             snap_hw ? snap_hw[2 * s + r] : 0, 0);
      build_ci(V, U.ci + (2 * s + r) * U.CI, U.CI);
    }
  }
  __syncthreads();
  if (active) {
    const UnitCtx X{P, a, (M ? c.bfill : c.snap) + slot(M ? kf : 0, 0) * icap, snap, snap_hw};
    const int64_t T_end = c.scal[1];
    const int q = a * P + s;
    const int64_t ws = M ? T_end - c.z[q] : c.w[q];
    for (int k = 0; k < pd.kmax; ++k) {
      if (k >= *stop) break;
      int64_t ready = ws;
      if (s > 0) {  // wait for chain k of the upstream stage
        int st;
        bool quit = false;
        while ((st = status[(s - 1) * L.KM + k]) == 0) {
          if (k >= *stop) { quit = true; break; }
          __nanosleep(20);
        }
        if (quit || st == 2) break;
        ready = max(endv[(s - 1) * L.KM + k] + c.enc_p2p, ws);
      }
      int64_t end;
      if (!place_stage<M>(c, pd, X, U, s, ready, &end)) {
        if (lane == 0) {
          atomicMin(&stop_at, k);
          status[s * L.KM + k] = 2;
        }
        break;
      }
      if (!M) {  // snapshot this stage after k+1 chains
        for (int r = 0; r < 2; ++r) {
          const int h = U.hw[2 * s + r];
          const int64_t* src = X.fill + (int64_t)s * icap + (r ? c.icapc : 0);
          int64_t* dst = c.snap + slot(k + 1, s) * icap + (r ? c.icapc : 0);
          for (int i = lane; i < h; i += 32) dst[i] = src[i];
          if (lane == 0) c.snap_hw[slot(k + 1, s) * 2 + r] = h;
        }
      }
      if (lane == 0) {
        endv[s * L.KM + k] = end;
        __threadfence_block();
        status[s * L.KM + k] = 1;
        if (s == P - 1) {
          if (M) c.tables[pd.inbB + ((int64_t)a * (pd.kmax + 1) + kf) * pd.kmax + k] = end;
          else c.tables[pd.inbF + (int64_t)a * pd.kmax + k] = end;
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // chains completed by every stage
    int k = 0;
    while (k < pd.kmax && status[(P - 1) * L.KM + k] == 1) ++k;
    if (M) c.tables[pd.lenB + (int64_t)a * (pd.kmax + 1) + kf] = k;
    else c.tables[pd.lenF + a] = k;
  }
}

}  // namespace

cudaError_t launch_plan_tables(const Cfg& c, cudaStream_t st, int* launches) {
  k_plan_tables<<<c.E, 128, 0, st>>>(c);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_chain_tables(const Cfg& c, int64_t fwd_units, int64_t bwd_units, cudaStream_t st,
                                int* launches) {
  K1Launch L;
  L.NK = c.nk_max;
  L.Pmax = c.p;
  L.CI = (std::max(c.icapc, c.icapm) + 31) / 32;
  L.KM = std::max(1, c.kmax_all);
  const size_t smem = k1_smem_bytes(L);
  if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
  static bool attrs = false;  // opt in to large dynamic shared memory once per process
  if (!attrs) {
    cudaFuncSetAttribute(k1_chains<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k1_chains<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attrs = true;
  }
  // one block per unit, one warp per stage of the widest plan
  if (fwd_units > 0) k1_chains<false><<<(unsigned)fwd_units, 32 * c.p, smem, st>>>(c, fwd_units, L);
  if (bwd_units > 0) k1_chains<true><<<(unsigned)bwd_units, 32 * c.p, smem, st>>>(c, bwd_units, L);
  if (launches) *launches += (fwd_units > 0) + (bwd_units > 0);
  return cudaGetLastError();
}

}  // namespace optimus
