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
}

// ------------------------------------------------------ first-fit machinery
// View of one (LLM stage, resource) interval list for one unit.
struct View {
  int count;
  bool mirror;
  const int64_t* S;   // template interval starts
  const int64_t* H;   // template interval ends
  int64_t* fill;      // this unit's fill pointers (own direction)
  int* hw;            // valid prefix of `fill` (lives in shared memory)
  const int64_t* snapf;  // mirror only: forward fill snapshot
  int hwf;               // mirror only: valid prefix of the snapshot
  int64_t T_end;
};

// forward fill pointer of REAL interval r (mirror view)
__device__ __forceinline__ int64_t fwd_lo(const View& V, int r) { return r < V.hwf ? V.snapf[r] : V.S[r]; }

__device__ __forceinline__ int64_t view_hi(const View& V, int i) {
  if (!V.mirror) return V.H[i];
  return V.T_end - fwd_lo(V, V.count - 1 - i);  // mirrored end = T_end - forward fill pointer (R15)
}
__device__ __forceinline__ int64_t view_start(const View& V, int i) {
  if (!V.mirror) return V.S[i];
  return V.T_end - V.H[V.count - 1 - i];
}

struct Window {
  int base;
  bool loaded, dirty;
  int64_t lo, hi;  // interval base+lane
};

__device__ __forceinline__ void win_load(const View& V, Window& w) {
  const int i = w.base + (threadIdx.x & 31);
  if (i < V.count) {
    w.hi = view_hi(V, i);
    w.lo = i < *V.hw ? V.fill[i] : view_start(V, i);
  } else {
    w.hi = kNegInf;
    w.lo = 0;
  }
  w.loaded = true;
  w.dirty = false;
}

__device__ __forceinline__ void win_writeback(const View& V, Window& w) {
  if (!w.loaded || !w.dirty) return;
  const int lane = threadIdx.x & 31;
  const int hw = *V.hw;
  for (int i = hw + lane; i < w.base; i += 32) V.fill[i] = view_start(V, i);  // gap fill
  const int i = w.base + lane;
  if (i < V.count) V.fill[i] = w.lo;
  __syncwarp();
  if (lane == 0) *V.hw = max(hw, min(V.count, w.base + 32));
  __syncwarp();
  w.dirty = false;
}

// first interval index with end > ready (ends are non-decreasing)
__device__ int first_end_after(const View& V, int64_t ready) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = V.count;
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int i = lo + lane * step;
    const bool le = i < hi && view_hi(V, i) <= ready;
    const int cnt = __popc(__ballot_sync(FULL, le));
    if (cnt == 0) return lo;
    const int nlo = lo + (cnt - 1) * step + 1;
    hi = min(hi, lo + cnt * step);
    lo = nlo;
  }
  const int i = lo + lane;
  const unsigned b = __ballot_sync(FULL, i < hi && view_hi(V, i) > ready);
  return b ? lo + __ffs(b) - 1 : hi;
}

// Place one kernel of duration d at or after `ready` (R12): scan intervals
// in time order from the first with end > ready, take the first where
// max(ready, lo) + d <= end; lo <- x + d.
__device__ __forceinline__ bool place_kernel(const View& V, Window& w, int64_t d, int64_t& ready) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (!w.loaded) {
      if (w.base >= V.count) return false;
      win_load(V, w);
    }
    const int64_t x = max(ready, w.lo);
    const bool ok = w.hi > ready && x + d <= w.hi;
    const unsigned b = __ballot_sync(FULL, ok);
    if (b) {
      const int f = __ffs(b) - 1;
      const int64_t xf = __shfl_sync(FULL, x, f);
      if (lane == f) w.lo = xf + d;
      w.dirty = true;
      ready = xf + d;
      return true;
    }
    win_writeback(V, w);
    w.base += 32;
    w.loaded = false;
  }
}

struct Row {
  int P, ti, a;
};

// One chain over stages 0..P-1 (R12; mirrored lists and w' for backward, R15).
// views[2*s + r]; returns false on failure (caller stops the unit).
__device__ bool place_chain(const Cfg& c, const Row& R, View* views, bool mirror, int64_t& EF) {
  const int64_t T_end = c.scal[1];
  int64_t ready = 0, prev = 0;
  for (int s = 0; s < R.P; ++s) {
    const int q = R.a * R.P + s;
    const int64_t ws = mirror ? T_end - c.z[q] : c.w[q];
    ready = (s == 0) ? ws : max(prev + c.enc_p2p, ws);
    Window w0, w1;  // compute-free / comm-free windows of this stage
    w0.base = first_end_after(views[2 * s + 0], ready);
    w1.base = first_end_after(views[2 * s + 1], ready);
    w0.loaded = w0.dirty = w1.loaded = w1.dirty = false;
    for (int b = 0; b < c.nb; ++b) {
      const int L = c.blayers[b];
      const int l0 = s * L / R.P, l1 = (s + 1) * L / R.P;
      const int id = enc_list_id(b, R.ti, c.ntp, mirror ? 1 : 0);
      const int off = c.loff[id], len = c.loff[id + 1] - off;
      for (int l = l0; l < l1; ++l)
        for (int k = 0; k < len; ++k) {
          // mirrored time runs each layer's backward list in reverse (R15)
          const int kk = mirror ? off + len - 1 - k : off + k;
          const int kind = __ldg(&c.lkind[kk]);
          const int64_t d = __ldg(&c.lns[kk]);
          const bool ok = kind == 0 ? place_kernel(views[2 * s + 0], w0, d, ready)
                                    : place_kernel(views[2 * s + 1], w1, d, ready);
          if (!ok) return false;
        }
    }
    win_writeback(views[2 * s + 0], w0);
    win_writeback(views[2 * s + 1], w1);
    prev = ready;
  }
  EF = ready;
  return true;
}

constexpr int kK1Warps = 4;

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

__global__ void __launch_bounds__(kK1Warps * 32) k1_forward(Cfg c, int64_t units) {
  __shared__ int hw_sm[kK1Warps][2 * kMaxP];
  __shared__ View views_sm[kK1Warps][2 * kMaxP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * kK1Warps + warp;
  if (u >= units) return;
  int e, a, kf;
  if (!decode_row_unit(c, u, false, e, a, kf)) return;
  const PlanDesc pd = c.plans[e];
  const int P = pd.P, icap = c.icapc + c.icapm;
  View* V = views_sm[warp];
  int* hw = hw_sm[warp];
  auto slot = [&](int k, int s) { return pd.slot_base + ((int64_t)k * pd.rp + a) * P + s; };
  if (lane < 2 * P) {
    const int s = lane >> 1, r = lane & 1, q = a * P + s;
    View& v = V[lane];
    v.count = r == 0 ? c.ncomp[q] : c.ncomm[q];
    v.mirror = false;
    v.S = r == 0 ? c.comp_lo + (int64_t)q * c.icapc : c.comm_lo + (int64_t)q * c.icapm;
    v.H = r == 0 ? c.comp_hi + (int64_t)q * c.icapc : c.comm_hi + (int64_t)q * c.icapm;
    v.fill = c.snap + slot(0, s) * icap + (r == 0 ? 0 : c.icapc);
    v.hw = &hw[lane];
    v.snapf = nullptr;
    v.hwf = 0;
    v.T_end = c.scal[1];
    hw[lane] = 0;
  }
  __syncwarp();
  int k = 0;
  for (; k < pd.kmax; ++k) {
    int64_t EF;
    if (!place_chain(c, Row{P, pd.ti, a}, V, false, EF)) break;
    if (lane == 0) c.tables[pd.inbF + (int64_t)a * pd.kmax + k] = EF;
    // snapshot the fill state after k+1 chains for the backward units
    if (k + 1 <= pd.kmax) {
      for (int sr = 0; sr < 2 * P; ++sr) {
        const int s = sr >> 1, r = sr & 1;
        const int h = hw[sr];
        const int64_t* src = V[sr].fill;
        int64_t* dst = c.snap + slot(k + 1, s) * icap + (r == 0 ? 0 : c.icapc);
        for (int i = lane; i < h; i += 32) dst[i] = src[i];
        if (lane == 0) c.snap_hw[slot(k + 1, s) * 2 + r] = h;
      }
    }
    __syncwarp();
  }
  if (lane == 0) c.tables[pd.lenF + a] = k;
}

__global__ void __launch_bounds__(kK1Warps * 32) k1_backward(Cfg c, int64_t units) {
  __shared__ int hw_sm[kK1Warps][2 * kMaxP];
  __shared__ View views_sm[kK1Warps][2 * kMaxP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t u = (int64_t)blockIdx.x * kK1Warps + warp;
  if (u >= units) return;
  int e, a, kf;
  if (!decode_row_unit(c, u, true, e, a, kf)) return;
  const PlanDesc pd = c.plans[e];
  const int lenF = (int)c.tables[pd.lenF + a];
  if (kf > lenF) return;  // no pipeline of this row can have kf forward chains
  const int P = pd.P, icap = c.icapc + c.icapm;
  View* V = views_sm[warp];
  int* hw = hw_sm[warp];
  auto slot = [&](int k, int s) { return pd.slot_base + ((int64_t)k * pd.rp + a) * P + s; };
  if (lane < 2 * P) {
    const int s = lane >> 1, r = lane & 1, q = a * P + s;
    View& v = V[lane];
    v.count = r == 0 ? c.ncomp[q] : c.ncomm[q];
    v.mirror = true;
    v.S = r == 0 ? c.comp_lo + (int64_t)q * c.icapc : c.comm_lo + (int64_t)q * c.icapm;
    v.H = r == 0 ? c.comp_hi + (int64_t)q * c.icapc : c.comm_hi + (int64_t)q * c.icapm;
    v.fill = c.bfill + slot(kf, s) * icap + (r == 0 ? 0 : c.icapc);
    v.hw = &hw[lane];
    v.snapf = c.snap + slot(kf, s) * icap + (r == 0 ? 0 : c.icapc);
    v.hwf = kf == 0 ? 0 : c.snap_hw[slot(kf, s) * 2 + r];
    v.T_end = c.scal[1];
    hw[lane] = 0;
  }
  __syncwarp();
  int k = 0;
  for (; k < pd.kmax; ++k) {
    int64_t EF;
    if (!place_chain(c, Row{P, pd.ti, a}, V, true, EF)) break;
    if (lane == 0) c.tables[pd.inbB + ((int64_t)a * (pd.kmax + 1) + kf) * pd.kmax + k] = EF;
  }
  if (lane == 0) c.tables[pd.lenB + (int64_t)a * (pd.kmax + 1) + kf] = k;
}

}  // namespace

cudaError_t launch_plan_tables(const Cfg& c, cudaStream_t st, int* launches) {
  k_plan_tables<<<c.E, 128, 0, st>>>(c);
  if (launches) *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_chain_tables(const Cfg& c, int64_t fwd_units, int64_t bwd_units, cudaStream_t st,
                                int* launches) {
  if (fwd_units > 0) k1_forward<<<(unsigned)((fwd_units + kK1Warps - 1) / kK1Warps), kK1Warps * 32, 0, st>>>(c, fwd_units);
  if (bwd_units > 0) k1_backward<<<(unsigned)((bwd_units + kK1Warps - 1) / kK1Warps), kK1Warps * 32, 0, st>>>(c, bwd_units);
  if (launches) *launches += (fwd_units > 0) + (bwd_units > 0);
  return cudaGetLastError();
}

}  // namespace optimus
