// template.cu — K0: the LLM template (GetEncLLMDep + bubble timeline).
//
// PAPER.md §4.3: interleaved 1F1B schedule of the LLM, adjusted
// warm-up counts, dependency points F_i / B_i; §4.2: the bubble
// pattern of 3D parallelism (DP all-gather / reduce-scatter bubbles, PP
// bubbles, TP bubbles); Design decision 3: encoder compute
// goes into compute-free time, encoder comm into comm-free time.
// Readings R2-R6.
//
// k0_template: one block of 32 warps.  A warp simulates the whole LLM
//   pipeline (lane = stage) as an ASAP list schedule in the fixed per-stage
//   Megatron order; the reverse-stage warm-up search (R5) tests up to 32
//   warm-up values of one stage at once, one warp each.
// k0_intervals: one block per LLM stage.  Threads expand the stage's ops
//   into kernels (lane-parallel over the kernel index), emit the gap after
//   each compute kernel (compute-free interval) and after each comm kernel
//   clipped to [w, z] (comm-free interval), and compact them in time order
//   with a block scan.
#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "optimus_dev.cuh"

namespace optimus {
namespace {

// K0 dynamic shared memory (declared at namespace scope so that every access
// compiles to LDS/STS, not to generic strong loads/stores)
extern __shared__ __align__(16) unsigned char k0_dsm[];

__device__ int64_t list_sum(const Cfg& c, int id) {
  int64_t s = 0;
  for (int i = c.loff[id]; i < c.loff[id + 1]; ++i) s += c.lns[i];
  return s;
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// K0 per-warp shared memory: [optab: p*nops int64][done: p*2*v*n int64].
// optab[s][pos] packs the op at position pos of stage s for the warp's
// current warm-up vector: bits 0-23 its own slot in done, 24-47 the slot of
// its dependency (0xFFFFFF = none), 48 forward, 49 cross-stage dependency.
constexpr uint64_t kNoDep = 0xFFFFFF;
constexpr int kFinalWarps = 8;

__host__ __device__ __forceinline__ size_t k0_warp_bytes(int p, int nops, int v, int n) {
  return (size_t)p * nops * 8 + (size_t)p * 2 * v * n * 8;
}

// Fill the warp's optab for the warm-up vector W (lane-parallel).
__device__ void build_optab(const Cfg& c, const int* W, size_t base) {
  uint64_t* tab = reinterpret_cast<uint64_t*>(k0_dsm + base);
  const int p = c.p, v = c.v, n = c.n, nops = c.nops;
  for (int i = threadIdx.x & 31; i < p * nops; i += 32) {
    const int s = i / nops, pos = i % nops;
    const OpRef op = op_at(p, v, n, W[s], pos);  // Megatron interleaved order (R2)
    int ds = -1, df = 0, dc = 0;                 // dependency (R2)
    if (op.fwd) {
      if (s > 0) { ds = s - 1; df = 1; dc = op.chunk; }
      else if (op.chunk > 0) { ds = p - 1; df = 1; dc = op.chunk - 1; }
    } else {
      if (s < p - 1) { ds = s + 1; df = 0; dc = op.chunk; }
      else if (op.chunk < v - 1) { ds = 0; df = 0; dc = op.chunk + 1; }
      else { ds = p - 1; df = 1; dc = v - 1; }
    }
    const uint64_t self = ((s * 2 + op.fwd) * v + op.chunk) * n + op.mb;
    const uint64_t dep = ds < 0 ? kNoDep : (uint64_t)(((ds * 2 + df) * v + dc) * n + op.mb);
    tab[i] = self | (dep << 24) | ((uint64_t)op.fwd << 48) | ((uint64_t)(ds >= 0 && ds != s) << 49);
  }
  __syncwarp();
}

// ASAP list schedule of the pipeline in optab's fixed per-stage order (R2,
// R3), one warp, lane = stage.  A trial stops as soon as an op ends after
// span_limit.  record: also write op starts, F, B.  Returns ok
// (deadlock-free and within the limit) and the span (max last-op end).
__device__ void warp_simulate(const Cfg& c, size_t base, bool record, int64_t dur_f, int64_t dur_b,
                              int64_t span_limit, int64_t* span, int* ok) {
  const uint64_t* tab = reinterpret_cast<const uint64_t*>(k0_dsm + base);
  volatile int64_t* done = reinterpret_cast<volatile int64_t*>(k0_dsm + base + (size_t)c.p * c.nops * 8);
  const int lane = threadIdx.x & 31;
  const int p = c.p, v = c.v, n = c.n, nops = c.nops;
  const int sz = p * 2 * v * n;
  for (int i = lane; i < sz; i += 32) done[i] = -1;
  __syncwarp();
  int pos = 0;
  int64_t fr = max((int64_t)0, c.T_ag);  // every op starts after the DP all-gather (R3)
  const int64_t pp2p = c.pp_p2p;
  bool over = false;
  const uint64_t* row = tab + (size_t)min(lane, p - 1) * nops;
  for (;;) {
    bool prog = false;
    if (lane < p) {
      while (pos < nops) {
        const uint64_t e = row[pos];
        const int dep = (int)((e >> 24) & kNoDep);
        int64_t t = fr;
        if (dep != (int)kNoDep) {
          const int64_t de = done[dep];
          if (de < 0) break;
          t = max(t, de + ((e >> 49) & 1 ? pp2p : 0));
        }
        const bool fwd = (e >> 48) & 1;
        const int64_t fin = t + (fwd ? dur_f : dur_b);
        if (fin > span_limit) { over = true; break; }
        const int self = (int)(e & kNoDep);
        done[self] = fin;
        if (record) {
          c.opstart[(int64_t)lane * nops + pos] = t;
          const int mb = self % n, ch = (self / n) % v;
          if (lane == 0 && ch == 0) {
            if (fwd) c.F[mb] = t;    // F_i: start of F(stage 0, chunk 0, i) (R4)
            else c.B[mb] = fin;      // B_i: end of B(stage 0, chunk 0, i)
          }
        }
        fr = fin;
        ++pos;
        prog = true;
      }
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, over) || !__any_sync(0xffffffffu, prog)) break;
  }
  *ok = __all_sync(0xffffffffu, lane >= p || pos == nops) && !__any_sync(0xffffffffu, over);
  *span = warp_max64(lane < p ? fr : 0);
}

__device__ __forceinline__ int default_w(int p, int v, int n, int s) {  // Megatron default warm-up (R2)
  if (v == 1) return min(n, p - 1 - s);
  if (n == p) return n * v;
  return min(n * v, 2 * (p - 1 - s) + (v - 1) * p);
}

// Speculative guess for the adjusted warm-up of stage s (only used to run
// the stage phases of R5 in parallel; every guess is verified).
__device__ __forceinline__ int guess_w(int p, int v, int n, int s) {
  return v == 1 ? default_w(p, v, n, s) : min(n * v, (v - 1) * p + (p - 1 - s));
}

__device__ __forceinline__ void dur_fb(const Cfg& c, int64_t& f, int64_t& b) {
  f = (int64_t)c.lc * list_sum(c, 0);
  b = (int64_t)c.lc * list_sum(c, 1);
}

// K0a: default warm-up, default schedule (span to preserve), reset of the search.
__global__ void __launch_bounds__(32) k0_default(Cfg c) {
  __shared__ int Wsm[kMaxP];
  const int lane = threadIdx.x;
  int64_t df, db;
  dur_fb(c, df, db);
  if (lane < c.p) {
    const int w = default_w(c.p, c.v, c.n, lane);
    c.Wdef[lane] = w;
    c.W[lane] = w;
    c.bestw[lane] = INT32_MAX;
    Wsm[lane] = w;
  }
  __syncwarp();
  build_optab(c, Wsm, 0);
  int64_t sp;
  int ok;
  warp_simulate(c, 0, false, df, db, INT64_MAX, &sp, &ok);
  if (lane == 0) { c.scal[0] = sp; c.scal[2] = ok; }
}

// K0b: GetEncLLMDep's warm-up adjustment (R5) is, for s = p-1 .. 0,
// the smallest w in [0, Wdef_s] keeping the schedule deadlock-free with the
// default span.  All stage phases run here at once, one trial (s, w) per
// block, each assuming the later stages take their guessed value; K0c
// verifies (a stage's result is exact when every later guess was right).
__global__ void __launch_bounds__(32) k0_wave(Cfg c) {
  __shared__ int Wsm[kMaxP];
  const int lane = threadIdx.x, p = c.p, v = c.v, n = c.n;
  if (c.policy != 1 || c.scal[2] == 0) return;
  int s = 0, w = blockIdx.x;
  while (s < p && w > default_w(p, v, n, s)) { w -= default_w(p, v, n, s) + 1; ++s; }
  if (s >= p) return;
  int64_t df, db;
  dur_fb(c, df, db);
  if (lane < p) Wsm[lane] = lane < s ? default_w(p, v, n, lane) : lane == s ? w : guess_w(p, v, n, lane);
  __syncwarp();
  build_optab(c, Wsm, 0);
  int64_t sp;
  int ok;
  warp_simulate(c, 0, false, df, db, c.scal[0], &sp, &ok);
  if (lane == 0 && ok && sp == c.scal[0]) atomicMin(&c.bestw[s], w);
}

// K0c: verify the wave from the last stage down, redo the phases below the
// first wrong guess exactly (kFinalWarps trials at a time), then the final
// schedule with its op starts, F_i, B_i and T_end.
__global__ void __launch_bounds__(kFinalWarps * 32) k0_final(Cfg c) {
  __shared__ int Wcur[kMaxP];
  __shared__ int Wsm[kFinalWarps][kMaxP];
  __shared__ int best_sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, p = c.p, v = c.v, n = c.n;
  const int nwarps = blockDim.x >> 5;
  if (c.scal[2] == 0) return;  // default schedule deadlocks: template fails
  const size_t base = (size_t)warp * k0_warp_bytes(p, c.nops, v, n);
  int64_t df, db;
  dur_fb(c, df, db);
  const int64_t span_def = c.scal[0];
  int s0 = -1;
  if (c.policy == 1) {
    int s = p - 1;
    while (s >= 0 && c.bestw[s] == guess_w(p, v, n, s)) --s;
    s0 = s;  // stages > s0 verified; stage s0 exact (its later stages were right)
  }
  if (threadIdx.x < p) {
    const int t = threadIdx.x;
    Wcur[t] = c.policy != 1 ? default_w(p, v, n, t)
                            : t > s0 ? guess_w(p, v, n, t) : t == s0 ? c.bestw[t] : default_w(p, v, n, t);
  }
  __syncthreads();
  for (int s = s0 - 1; s >= 0; --s) {  // exact sequential phases (rarely needed)
    const int wd = default_w(p, v, n, s);
    for (int b = 0; b <= wd; b += nwarps) {
      if (threadIdx.x == 0) best_sm = INT32_MAX;
      __syncthreads();
      const int w = b + warp;
      if (w <= wd) {
        if (lane < p) Wsm[warp][lane] = lane == s ? w : Wcur[lane];
        __syncwarp();
        build_optab(c, Wsm[warp], base);
        int64_t sp;
        int ok;
        warp_simulate(c, base, false, df, db, span_def, &sp, &ok);
        if (lane == 0 && ok && sp == span_def) atomicMin(&best_sm, w);
      }
      __syncthreads();
      const int bw = best_sm;
      __syncthreads();
      if (bw != INT32_MAX) {
        if (threadIdx.x == 0) Wcur[s] = bw;
        __syncthreads();
        break;
      }
    }
  }
  if (warp == 0) {
    build_optab(c, Wcur, 0);
    int64_t sp;
    int ok;
    warp_simulate(c, 0, true, df, db, INT64_MAX, &sp, &ok);
    if (lane < p) c.W[lane] = Wcur[lane];
    if (lane == 0) {
      c.scal[1] = sp + c.T_rs;  // T_end = max_p(last op end_p + T_rs) (R3)
      c.scal[2] = ok;
    }
  }
}

// ------------------------------------------------------------ intervals
constexpr int kIvThreads = 512;

struct ListInfo {
  int off, len;
  int64_t sum;
  int firstc, lastc, firstm;  // first compute, last compute, first comm index (-1 if none)
};

__device__ ListInfo list_info(const Cfg& c, int id) {
  ListInfo L;
  L.off = c.loff[id];
  L.len = c.loff[id + 1] - L.off;
  L.sum = 0;
  L.firstc = L.lastc = L.firstm = -1;
  for (int i = 0; i < L.len; ++i) {
    L.sum += c.lns[L.off + i];
    if (c.lkind[L.off + i] == 0) {
      if (L.firstc < 0) L.firstc = i;
      L.lastc = i;
    } else if (L.firstm < 0) {
      L.firstm = i;
    }
  }
  return L;
}

__global__ void __launch_bounds__(kIvThreads) k0_intervals(Cfg c) {
  using Scan = cub::BlockScan<int, kIvThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int run_c, run_m;
  extern __shared__ int opoff[];  // [nops + 1] kernel offset of each op
  if (c.scal[2] == 0) return;     // template failed (deadlock): nothing to emit
  const int s = blockIdx.x;
  const int p = c.p, v = c.v, n = c.n, nops = c.nops, lc = c.lc;
  const int Ws = c.W[s];
  const ListInfo Lf = list_info(c, 0), Lb = list_info(c, 1);
  const int64_t* ost = c.opstart + (int64_t)s * nops;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < nops; ++q) {
      opoff[q] = acc;
      acc += lc * (op_at(p, v, n, Ws, q).fwd ? Lf.len : Lb.len);
    }
    opoff[nops] = acc;
    run_c = run_m = 0;
  }
  __syncthreads();
  const int K = opoff[nops];
  // first op is always a forward, last always a backward
  const int64_t w = ost[0] + [&] { int64_t a = 0; for (int i = 0; i < Lf.firstc; ++i) a += c.lns[Lf.off + i]; return a; }();
  const int64_t z = ost[nops - 1] + (int64_t)(lc - 1) * Lb.sum +
                    [&] { int64_t a = 0; for (int i = 0; i <= Lb.lastc; ++i) a += c.lns[Lb.off + i]; return a; }();
  if (threadIdx.x == 0) { c.w[s] = w; c.z[s] = z; }
  int64_t* clo = c.comp_lo + (int64_t)s * c.icapc;
  int64_t* chi = c.comp_hi + (int64_t)s * c.icapc;
  int64_t* mlo = c.comm_lo + (int64_t)s * c.icapm;
  int64_t* mhi = c.comm_hi + (int64_t)s * c.icapm;
  // head comm-free piece [w, first comm start) (R6), emitted first
  if (threadIdx.x == 0) {
    int64_t first_comm = kInf;
    if (Lf.firstm >= 0) {
      int64_t a = 0;
      for (int i = 0; i < Lf.firstm; ++i) a += c.lns[Lf.off + i];
      first_comm = ost[0] + a;
    } else if (Lb.firstm >= 0) {
      first_comm = -1;  // unreachable: validated (both lists have comm or neither)
    }
    int64_t hi = min(first_comm, z);
    if (hi > w) { mlo[0] = w; mhi[0] = hi; run_m = 1; }
  }
  __syncthreads();
  // offset of kernel i of list L within a layer pass
  auto koff = [&](const ListInfo& L, int i) {
    int64_t a = 0;
    for (int q = 0; q < i; ++q) a += c.lns[L.off + q];
    return a;
  };
  for (int base = 0; base < K; base += kIvThreads) {
    const int kk = base + threadIdx.x;
    int ec = 0, em = 0;
    int64_t clo_v = 0, chi_v = 0, mlo_v = 0, mhi_v = 0;
    if (kk < K) {
      // locate the op (binary search on opoff)
      int lo = 0, hi = nops - 1;
      while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (opoff[mid] <= kk) lo = mid; else hi = mid - 1;
      }
      const int q = lo;
      const bool fwd = op_at(p, v, n, Ws, q).fwd;
      const ListInfo& L = fwd ? Lf : Lb;
      const int r = kk - opoff[q], rep = r / L.len, i = r % L.len;
      const int kind = c.lkind[L.off + i];
      const int64_t st = ost[q] + (int64_t)rep * L.sum + koff(L, i);
      const int64_t en = st + c.lns[L.off + i];
      // start of the next kernel of the same kind
      int64_t nxt = kInf;
      int j = -1;
      for (int t = i + 1; t < L.len; ++t)
        if (c.lkind[L.off + t] == kind) { j = t; break; }
      if (j >= 0) {
        nxt = ost[q] + (int64_t)rep * L.sum + koff(L, j);
      } else if (rep < lc - 1) {
        int f = kind == 0 ? L.firstc : L.firstm;
        nxt = ost[q] + (int64_t)(rep + 1) * L.sum + koff(L, f);
      } else if (q < nops - 1) {
        const ListInfo& L2 = op_at(p, v, n, Ws, q + 1).fwd ? Lf : Lb;
        int f = kind == 0 ? L2.firstc : L2.firstm;
        if (f >= 0) nxt = ost[q + 1] + koff(L2, f);
      }
      if (kind == 0) {
        if (nxt != kInf && nxt > en) { ec = 1; clo_v = en; chi_v = nxt; }  // compute-free gap
      } else {
        int64_t a = max(en, w), b = min(nxt, z);
        if (b > a) { em = 1; mlo_v = a; mhi_v = b; }  // comm-free piece inside [w, z]
      }
    }
    int pc, pm, tc, tm;
    Scan(tmp).ExclusiveSum(ec, pc, tc);
    __syncthreads();
    Scan(tmp).ExclusiveSum(em, pm, tm);
    const int bc = run_c, bm = run_m;
    if (ec) { clo[bc + pc] = clo_v; chi[bc + pc] = chi_v; }
    if (em) { mlo[bm + pm] = mlo_v; mhi[bm + pm] = mhi_v; }
    __syncthreads();
    if (threadIdx.x == 0) { run_c = bc + tc; run_m = bm + tm; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { c.ncomp[s] = run_c; c.ncomm[s] = run_m; }
}

}  // namespace

cudaError_t launch_template(const Cfg& c, cudaStream_t st, int* launches) {
  const size_t per = k0_warp_bytes(c.p, c.nops, c.v, c.n);
  if (per > 200 * 1024) return cudaErrorInvalidConfiguration;
  const int fw = (int)std::max<size_t>(1, std::min<size_t>(kFinalWarps, (200 * 1024) / per));
  cudaFuncSetAttribute(k0_default, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  cudaFuncSetAttribute(k0_wave, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
  cudaFuncSetAttribute(k0_final, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(per * fw));
  int trials = 0;
  for (int s = 0; s < c.p; ++s) {
    const int p = c.p, v = c.v, n = c.n;
    trials += (v == 1 ? std::min(n, p - 1 - s) : n == p ? n * v : std::min(n * v, 2 * (p - 1 - s) + (v - 1) * p)) + 1;
  }
  k0_default<<<1, 32, per, st>>>(c);
  k0_wave<<<std::max(1, trials), 32, per, st>>>(c);
  k0_final<<<1, 32 * fw, per * fw, st>>>(c);
  k0_intervals<<<c.p, kIvThreads, (c.nops + 1) * sizeof(int), st>>>(c);
  if (launches) *launches += 4;
  return cudaGetLastError();
}

}  // namespace optimus
