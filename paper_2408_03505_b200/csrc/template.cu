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
#include <cub/block/block_scan.cuh>

#include "optimus_dev.cuh"

namespace optimus {
namespace {

__device__ __forceinline__ int64_t ldv(const int64_t* p) { return *(volatile const int64_t*)p; }
__device__ __forceinline__ void stv(int64_t* p, int64_t v) { *(volatile int64_t*)p = v; }

__device__ int64_t list_sum(const Cfg& c, int id) {
  int64_t s = 0;
  for (int i = c.loff[id]; i < c.loff[id + 1]; ++i) s += c.lns[i];
  return s;
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Simulate the interleaved 1F1B pipeline with per-stage warm-up counts W
// (lane s reads W[s]).  done: this warp's scratch [p][2][v][n] of op end
// times.  record: also write op starts, F, B.  Returns ok (deadlock-free)
// and the span (max last-op end).
__device__ void warp_simulate(const Cfg& c, const int* W, int64_t* done, bool record, int64_t dur_f,
                              int64_t dur_b, int64_t* span, int* ok) {
  const int lane = threadIdx.x & 31;
  const int p = c.p, v = c.v, n = c.n, nops = c.nops;
  const int sz = p * 2 * v * n;
  for (int i = lane; i < sz; i += 32) stv(&done[i], -1);
  __syncwarp();
  auto idx = [&](int s, int f, int ch, int mb) { return ((s * 2 + f) * v + ch) * n + mb; };
  int pos = 0;
  int64_t fr = 0;
  const int Ws = lane < p ? W[lane] : 0;
  for (;;) {
    bool prog = false;
    if (lane < p) {
      while (pos < nops) {
        OpRef op = op_at(p, v, n, Ws, pos);
        int ds = -1, df = 0, dc = 0;  // dependency (R2)
        if (op.fwd) {
          if (lane > 0) { ds = lane - 1; df = 1; dc = op.chunk; }
          else if (op.chunk > 0) { ds = p - 1; df = 1; dc = op.chunk - 1; }
        } else {
          if (lane < p - 1) { ds = lane + 1; df = 0; dc = op.chunk; }
          else if (op.chunk < v - 1) { ds = 0; df = 0; dc = op.chunk + 1; }
          else { ds = p - 1; df = 1; dc = v - 1; }
        }
        int64_t t = max(fr, c.T_ag);  // every op starts after the DP all-gather (R3)
        if (ds >= 0) {
          int64_t e = ldv(&done[idx(ds, df, dc, op.mb)]);
          if (e < 0) break;
          t = max(t, e + (ds != lane ? c.pp_p2p : 0));
        }
        const int64_t d = op.fwd ? dur_f : dur_b;
        stv(&done[idx(lane, op.fwd, op.chunk, op.mb)], t + d);
        if (record) {
          c.opstart[(int64_t)lane * nops + pos] = t;
          if (lane == 0 && op.chunk == 0) {
            if (op.fwd) c.F[op.mb] = t;       // F_i: start of F(stage 0, chunk 0, i) (R4)
            else c.B[op.mb] = t + d;          // B_i: end of B(stage 0, chunk 0, i)
          }
        }
        fr = t + d;
        ++pos;
        prog = true;
      }
    }
    __syncwarp();
    if (!__any_sync(0xffffffffu, prog)) break;
  }
  *ok = __all_sync(0xffffffffu, lane >= p || pos == nops);
  *span = warp_max64(lane < p ? fr : 0);
}

__global__ void __launch_bounds__(kSimWarps * 32) k0_template(Cfg c) {
  __shared__ int Wsm[kSimWarps][kMaxP];
  __shared__ int Wcur[kMaxP];
  __shared__ int Wd[kMaxP];
  __shared__ long long span_def;
  __shared__ int ok_def, best_w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = c.p, v = c.v, n = c.n;
  const int64_t dur_f = (int64_t)c.lc * list_sum(c, 0);
  const int64_t dur_b = (int64_t)c.lc * list_sum(c, 1);
  int64_t* scratch = c.sim + (int64_t)warp * p * 2 * v * n;
  if (threadIdx.x < p) {  // Megatron default warm-up (R2)
    int s = threadIdx.x, w;
    if (v == 1) w = min(n, p - 1 - s);
    else if (n == p) w = n * v;
    else w = min(n * v, 2 * (p - 1 - s) + (v - 1) * p);
    Wd[s] = w;
    Wcur[s] = w;
  }
  __syncthreads();
  if (warp == 0) {
    int64_t sp;
    int ok;
    warp_simulate(c, Wd, scratch, false, dur_f, dur_b, &sp, &ok);
    if (lane == 0) { span_def = sp; ok_def = ok; }
  }
  __syncthreads();
  if (!ok_def) {
    if (threadIdx.x == 0) c.scal[2] = 0;
    return;
  }
  if (c.policy == 1) {
    // R5: for s = p-1 .. 0, the smallest w in [0, Wdef_s] keeping the
    // schedule deadlock-free with the default span
    for (int s = p - 1; s >= 0; --s) {
      for (int base = 0; base <= Wd[s]; base += kSimWarps) {
        if (threadIdx.x == 0) best_w = INT32_MAX;
        const int w = base + warp;
        if (lane < p) Wsm[warp][lane] = (lane == s) ? w : Wcur[lane];
        __syncthreads();
        if (w <= Wd[s]) {
          int64_t sp;
          int ok;
          warp_simulate(c, Wsm[warp], scratch, false, dur_f, dur_b, &sp, &ok);
          if (lane == 0 && ok && sp == span_def) atomicMin(&best_w, w);
        }
        __syncthreads();
        const int bw = best_w;
        __syncthreads();
        if (bw != INT32_MAX) {
          if (threadIdx.x == 0) Wcur[s] = bw;
          __syncthreads();
          break;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 0) {
    int64_t sp;
    int ok;
    warp_simulate(c, Wcur, scratch, true, dur_f, dur_b, &sp, &ok);
    if (lane < p) { c.W[lane] = Wcur[lane]; c.Wdef[lane] = Wd[lane]; }
    if (lane == 0) {
      c.scal[0] = span_def;
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
  k0_template<<<1, kSimWarps * 32, 0, st>>>(c);
  k0_intervals<<<c.p, kIvThreads, (c.nops + 1) * sizeof(int), st>>>(c);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

}  // namespace optimus
