// template.cu — K0: the LLM template (GetEncLLMDep + bubble timeline).
//
// PAPER.md §4.3: interleaved 1F1B schedule of the LLM, adjusted
// warm-up counts, dependency points F_i / B_i; §4.2: the bubble
// pattern of 3D parallelism (DP all-gather / reduce-scatter bubbles, PP
// bubbles, TP bubbles); Design decision 3: encoder compute
// goes into compute-free time, encoder comm into comm-free time.
// Readings R2-R6.
//
// k0_wave: one warp per simulation (lane = stage): the ASAP list schedule
//   of the LLM pipeline in the fixed per-stage Megatron order, in lockstep
//   rounds; the default warm-up vector and every (stage, w) trial of the
//   reverse-stage warm-up search (R5) run at once, speculatively.
// k0_final: verifies the speculation (exact fallback on all warps of one
//   block), fixes W and T_end.
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

// sum of list `id`'s durations (called by a whole warp)
__device__ int64_t list_sum(const Cfg& c, int id) {
  const int lane = threadIdx.x & 31, off = c.loff[id], len = c.loff[id + 1] - off;
  int64_t a = 0;
  for (int i = lane; i < len; i += 32) a += c.lns[off + i];
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// K0 shared memory: [vtab: n*v shorts x 2] then, per simulating warp,
// [W: kMaxP ints][endv: p*(2vn+1) int64][optab: p*(nops+1) uint32].  vtab
// maps a virtual id k to its forward chunk and microbatch (R2); endv[slot]
// = end of the op in that slot (-1: not placed yet).  Per-stage strides are
// odd (2vn+1, nops+1) so that the 32 lanes (stages) hit distinct banks.
constexpr int kNone = 0xFFFF;
constexpr int kSimWarps = 8;  // simulations per block
constexpr int kIvBlocks = 8;  // k0_intervals blocks per LLM stage (capi sizes the exchange for 8)

__host__ __device__ __forceinline__ size_t k0_vtab_bytes(int n, int v) { return ((size_t)4 * n * v + 15) & ~size_t(15); }
__host__ __device__ __forceinline__ size_t k0_warp_bytes(int p, int v, int n) {
  return ((size_t)kMaxP * 4 + (size_t)p * (2 * v * n + 1) * (8 + 4) + 15) & ~size_t(15);  // W, endv, optab
}
__host__ __device__ __forceinline__ int k0_sim_warps(int p, int v, int n) {
  const size_t room = 200 * 1024 - k0_vtab_bytes(n, v);
  return (int)max((size_t)1, min((size_t)kSimWarps, room / k0_warp_bytes(p, v, n)));
}

// op at position pos of stage s under warm-up count Ws (R2): its endv slot,
// dependency slot and whether the dependency is on another stage
__device__ __forceinline__ void op_slots(int p, int v, int n, int s, int pos, int Ws, const short* vch,
                                         const short* vmb, int& self, int& dep, int& fwd, int& cross, int& dstage) {
  const int nv = n * v, r = pos - Ws;
  int k;
  if (r < 0) { k = pos; fwd = 1; }
  else if (r < 2 * (nv - Ws)) { fwd = (r & 1) ? 0 : 1; k = fwd ? Ws + r / 2 : r / 2; }
  else { fwd = 0; k = (nv - Ws) + (r - 2 * (nv - Ws)); }
  const int chf = vch[k], mb = vmb[k], ch = fwd ? chf : v - 1 - chf;
  int ds = -1, df = 0, dc = 0;
  if (fwd) {
    if (s > 0) { ds = s - 1; df = 1; dc = ch; }
    else if (ch > 0) { ds = p - 1; df = 1; dc = ch - 1; }
  } else {
    if (s < p - 1) { ds = s + 1; df = 0; dc = ch; }
    else if (ch < v - 1) { ds = 0; df = 0; dc = ch + 1; }
    else { ds = p - 1; df = 1; dc = v - 1; }
  }
  self = ((s * 2 + fwd) * v + ch) * n + mb;
  dep = ds < 0 ? (int)kNone : ((ds * 2 + df) * v + dc) * n + mb;
  cross = ds >= 0 && ds != s;
  dstage = ds;
}

__device__ void build_vtab(const Cfg& c) {
  const int p = c.p, v = c.v, n = c.n, nv = n * v;
  short* vch = reinterpret_cast<short*>(k0_dsm);
  short* vmb = vch + nv;
  for (int k = threadIdx.x; k < nv; k += blockDim.x) {
    vch[k] = (short)((k % (p * v)) / p);
    vmb[k] = (short)((k / (p * v)) * p + (k % p));
  }
  __syncthreads();
}

// One simulation per warp, lane = stage: the ASAP list schedule of the
// pipeline in the fixed per-stage order for warm-up vector W (R2, R3).
// Each stage places its ops in order; an op starts at max(previous op's
// end, dependency end (+ pp_p2p across stages), T_ag) once its dependency
// has ended, one op per stage per round between warp barriers.  No
// progress in a whole check period (8 rounds) before every op is placed means the
// order deadlocks.  record: also write op starts, F, B.  Returns the span
// (max last-op end), or -1 on deadlock.  A trial of R5 that must keep the
// default span returns -3 as soon as an op ends after `bound` (the default
// span when known; poll: read it from scal[3] once the default simulation
// has published it).
__device__ int64_t warp_simulate(const Cfg& c, const int* W, int64_t* endv_, uint32_t* optab, bool record,
                                 int64_t dur_f, int64_t dur_b, int64_t bound = INT64_MAX, bool poll = false) {
  const int lane = threadIdx.x & 31, p = c.p, v = c.v, n = c.n, nops = c.nops, nv = n * v;
  const short* vch = reinterpret_cast<const short*>(k0_dsm);
  const short* vmb = vch + nv;
  volatile int64_t* endv = endv_;
  const int S = 2 * v * n;  // slots per stage; padded stride S + 1
  for (int i = lane; i < p * (S + 1); i += 32) endv[i] = -1;
  const int s = lane;
  // op tables, built by the whole warp: self slot | dep slot << 15 (0x7FFF
  // none) | fwd << 30 | cross << 31 (padded slots)
  // (no integer division: slot / S is the slot's stage, so the padded slot
  // of stage t's slot x is x + t; the op tables used to spend most of a
  // simulation's time in divisions)
  for (int st = 0; st < p; ++st) {
    const int Ws = W[st];
    for (int pos = lane; pos < nops; pos += 32) {
      int self, dep, fwd, cross, ds;
      op_slots(p, v, n, st, pos, Ws, vch, vmb, self, dep, fwd, cross, ds);
      const int ps = self + st, pd = dep == kNone ? 0x7FFF : dep + ds;
      optab[(size_t)st * (nops + 1) + pos] = (uint32_t)ps | (uint32_t)pd << 15 | (uint32_t)fwd << 30 | (uint32_t)cross << 31;
    }
  }
  const uint32_t* tab = optab + (size_t)s * (nops + 1);
  __syncwarp();
  const int64_t T_ag = max((int64_t)0, c.T_ag), pp2p = c.pp_p2p;
  int pos = s < p ? 0 : nops;
  int64_t tprev = T_ag;  // every op starts after the DP all-gather (R3)
  bool prog = false;
  uint32_t op = pos < nops ? tab[pos] : 0;
  int64_t polled = 0;
  for (int round = 0;; ++round) {
    if (poll && (round & 7) == 0 && lane == 0)  // used 8 rounds later
      asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(polled) : "l"(&c.scal[3]));
    const int dep = (op >> 15) & 0x7FFF;
    const int64_t de = pos >= nops ? -1 : dep == 0x7FFF ? 0 : endv[dep];
    if (de >= 0) {  // one op per stage per round (running ahead serialises the warp)
      const uint32_t nxt = tab[min(pos + 1, nops - 1)];
      const int self = op & 0x7FFF;
      const bool fwd = (op >> 30) & 1;
      const int64_t t = dep == 0x7FFF ? tprev : max(tprev, de + ((op >> 31) ? pp2p : 0));
      const int64_t e = t + (fwd ? dur_f : dur_b);
      endv[self] = e;
      tprev = e;
      ++pos;
      op = nxt;
      prog = true;
    }
    __syncwarp();
    if ((round & 7) == 7) {  // periodic checks: done, deadlock, default span exceeded
      const unsigned left = __ballot_sync(0xffffffffu, pos < nops), any = __ballot_sync(0xffffffffu, prog);
#ifdef K0_STATS
      if (!left && lane == 0) printf("K0ROUNDS %d rec=%d\n", round, (int)record);
#endif
      if (!left) break;
      if (!any) return -1;  // no progress in 8 rounds: deadlock
      prog = false;
      if (poll && bound == INT64_MAX) {
        const int64_t b = __shfl_sync(0xffffffffu, polled, 0);
        if (b > 0) bound = b - 1;
      }
      if (__any_sync(0xffffffffu, tprev > bound)) return -3;
    }
  }
  if (record) {  // op starts from the ends; F_i / B_i (R4): start of F / end of B of (stage 0, chunk 0, i)
    __syncwarp();
    for (int idx = lane; idx < p * nops; idx += 32) {
      const int st = idx / nops, pos = idx - st * nops;
      const uint32_t op = optab[(size_t)st * (nops + 1) + pos];
      const bool fwd = (op >> 30) & 1;
      const int64_t e = endv[op & 0x7FFF], t = e - (fwd ? dur_f : dur_b);
      c.opstart[idx] = t;
      if (st == 0) {
        const int us = (int)(op & 0x7FFF) - (int)(op & 0x7FFF) / (S + 1);  // unpadded slot
        const int mb = us % n, ch = (us / n) % v;
        if (ch == 0) {
          if (fwd) c.F[mb] = t;
          else c.B[mb] = e;
        }
      }
    }
  }
  return warp_max64(tprev);  // lanes >= p hold T_ag <= every end
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

// K0a, one warp per simulation: simulation 0 the default warm-up (its span
// must be preserved; it is the final schedule under policy 0), simulation
// 1 + t trial t = (s, w) of GetEncLLMDep's warm-up adjustment (R5, P:444:
// for s = p-1 .. 0 the smallest w in [0, Wdef_s] keeping the schedule
// deadlock-free with the default span).  All stage phases run at once, each
// assuming the later stages take their guessed value; the trial with every
// stage at its guess records its schedule (it is the final one when K0b
// verifies every guess).  res[b] = span, or -1 if the schedule deadlocks.
#ifdef K0_CYC
__device__ long long g_k0cyc[1024][4];
#endif
__global__ void __launch_bounds__(32 * kSimWarps) k0_wave(Cfg c, int nsim, int wpb) {
  const int p = c.p, v = c.v, n = c.n, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef K0_CYC
  const long long tc0 = clock64();
  long long tg0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg0));
#endif
  build_vtab(c);
  const int b = blockIdx.x * wpb + warp;
  if (warp >= wpb || b >= nsim) return;
  int* Wsm = reinterpret_cast<int*>(k0_dsm + k0_vtab_bytes(n, v) + (size_t)warp * k0_warp_bytes(p, v, n));
  int64_t* endv = reinterpret_cast<int64_t*>(Wsm + kMaxP);
  uint32_t* optab = reinterpret_cast<uint32_t*>(endv + (size_t)p * (2 * v * n + 1));
  int s = -1, w = 0;
  if (b > 0) {
    if (c.policy != 1) return;
    s = 0;
    w = b - 1;
    while (s < p && w > default_w(p, v, n, s)) { w -= default_w(p, v, n, s) + 1; ++s; }
    if (s >= p) return;
  }
  int64_t df, db;
  dur_fb(c, df, db);
  if (lane < p) {
    const int d = default_w(p, v, n, lane);
    Wsm[lane] = s < 0 || lane < s ? d : lane == s ? w : guess_w(p, v, n, lane);
    if (b == 0) c.Wdef[lane] = d;
  }
  __syncwarp();
  const bool all_guess = s == 0 && w == guess_w(p, v, n, 0);
  const bool record = c.policy == 1 ? all_guess : b == 0;
#ifdef K0_STATS
  const long long t0 = clock64();
#endif
#ifdef K0_CYC
  const long long tc1 = clock64();
#endif
  const int64_t sp = warp_simulate(c, Wsm, endv, optab, record, df, db, INT64_MAX, b > 0 && !record);
#ifdef K0_CYC
  if (lane == 0 && b < 1024) {
    long long tg1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg1));
    g_k0cyc[b][0] = tc1 - tc0;
    g_k0cyc[b][1] = clock64() - tc1;
    g_k0cyc[b][2] = tg0;
    g_k0cyc[b][3] = tg1;
  }
#endif
#ifdef K0_STATS
  if (lane == 0) printf("K0ST b=%d s=%d w=%d sp=%lld cyc=%lld blk=%d\n", b, s, w, (long long)sp, clock64() - t0, blockIdx.x);
#endif
  if (lane == 0) {
    c.k0res[b] = sp;
    if (b == 0) atomicExch((unsigned long long*)&c.scal[3], (unsigned long long)(sp + 1));  // trials may stop early
  }
}

// K0b: verify the wave from the last stage down; in the common case the
// recorded all-guess schedule is the final one.  Otherwise redo the phases
// below the first wrong guess exactly (the trials of one phase run on all
// warps at once; the smallest successful w wins) and record the final
// schedule.  Writes W, T_end and the ok flag.
__global__ void __launch_bounds__(32 * kSimWarps) k0_final(Cfg c, int wpb) {
  __shared__ int Wcur[kMaxP];
  __shared__ int s0_sm, wbest;
  const int p = c.p, v = c.v, n = c.n, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t span_def = c.k0res[0];
  if (threadIdx.x == 0) {
    c.scal[0] = span_def;
    c.scal[3] = 0;  // reset for the next build's wave
  }
  for (int i = threadIdx.x; i < c.nflags; i += blockDim.x) c.k1flags[i] = 0;  // K1 progress flags
  for (int i = threadIdx.x; i < c.E; i += blockDim.x) c.pdone[i] = 0;        // K1 -> K2 plan completion
  if (threadIdx.x == 0) *c.k1next = 0;                                         // K1 work counter
  for (int i = threadIdx.x; i < c.p * kIvBlocks; i += blockDim.x) c.ivflag[i] = 0;  // k0_intervals exchange
  for (int i = threadIdx.x; i < c.p * 4 * c.ci_n; i += blockDim.x) c.bmax[i] = kNegInf;
#ifdef PDL_PROBE
  if (threadIdx.x == 0) {
    unsigned long long* probe = reinterpret_cast<unsigned long long*>(c.k1next) + 1;
    printf("PROBE k1start %llu k1end %llu (+%llu us) k2start (+%llu us)\n", probe[0], probe[1],
           (probe[1] - probe[0]) / 1000, (probe[2] - probe[0]) / 1000);
    probe[0] = ~0ull; probe[1] = 0; probe[2] = ~0ull;
  }
#endif
  if (span_def < 0) {  // default schedule deadlocks: template fails
    if (threadIdx.x == 0) c.scal[2] = 0;
    return;
  }
  int64_t df, db;
  dur_fb(c, df, db);
  __shared__ int bestw_sm[kMaxP];
  if (threadIdx.x < p) bestw_sm[threadIdx.x] = INT32_MAX;
  __syncthreads();
  if (c.policy == 1)  // smallest successful w per stage (speculative), all trials in parallel
    for (int b = threadIdx.x; b < c.k0_trials; b += blockDim.x) {
      int s = 0, w = b;
      while (w > default_w(p, v, n, s)) { w -= default_w(p, v, n, s) + 1; ++s; }
      if (c.k0res[1 + b] == span_def) atomicMin(&bestw_sm[s], w);
    }
  __syncthreads();
  if (c.policy == 1 && threadIdx.x < p) c.bestw[threadIdx.x] = bestw_sm[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = -1;
    if (c.policy == 1) {
      s = p - 1;
      while (s >= 0 && c.bestw[s] == guess_w(p, v, n, s)) --s;
    }
    s0_sm = s;  // stages > s0 verified; stage s0 exact (its later stages were right)
  }
  __syncthreads();
  const int s0 = s0_sm;
  if (threadIdx.x < p) {
    const int t = threadIdx.x;
    Wcur[t] = c.policy != 1 ? default_w(p, v, n, t)
                            : t > s0 ? guess_w(p, v, n, t) : t == s0 ? c.bestw[t] : default_w(p, v, n, t);
  }
  __syncthreads();
  if (c.policy != 1 || s0 < 0) {  // the recorded schedule (default, or all guesses verified) is final
    if (threadIdx.x < p) c.W[threadIdx.x] = Wcur[threadIdx.x];
    if (threadIdx.x == 0) {
      c.scal[1] = span_def + c.T_rs;  // T_end = max_p(last op end_p + T_rs) (R3); span kept by R5
      c.scal[2] = 1;
    }
    return;
  }
  build_vtab(c);
  int* Wt = reinterpret_cast<int*>(k0_dsm + k0_vtab_bytes(n, v) + (size_t)warp * k0_warp_bytes(p, v, n));
  int64_t* endv = reinterpret_cast<int64_t*>(Wt + kMaxP);
  uint32_t* optab = reinterpret_cast<uint32_t*>(endv + (size_t)p * (2 * v * n + 1));
  for (int s = s0 - 1; s >= 0; --s) {  // exact sequential phases
    const int nw = default_w(p, v, n, s) + 1;
    if (threadIdx.x == 0) wbest = INT32_MAX;
    __syncthreads();
    for (int w0 = 0; w0 < nw; w0 += wpb) {
      const int w = w0 + warp;
      if (warp < wpb && w < nw) {
        if (lane < p) Wt[lane] = lane == s ? w : Wcur[lane];
        __syncwarp();
        const int64_t sp = warp_simulate(c, Wt, endv, optab, false, df, db, span_def);
        if (lane == 0 && sp == span_def) atomicMin(&wbest, w);
      }
      __syncthreads();
      if (wbest != INT32_MAX) break;  // uniform
    }
    if (threadIdx.x == 0) Wcur[s] = wbest;  // w = Wdef_s always succeeds (default schedule)
    __syncthreads();
  }
  if (warp == 0) {
    const int64_t sp = warp_simulate(c, Wcur, endv, optab, true, df, db);
    if (lane < p) c.W[lane] = Wcur[lane];
    if (lane == 0) {
      c.scal[1] = sp + c.T_rs;  // T_end = max_p(last op end_p + T_rs) (R3)
      c.scal[2] = sp >= 0;
    }
  }
}

// ------------------------------------------------------------ intervals
constexpr int kIvThreads = 512;

constexpr int kLmax = 256;  // LLM layer kernel list capacity (validated at load)

// One LLM layer kernel list in shared memory: per kernel its duration,
// kind, start offset within a layer pass and the next kernel of the same
// kind in the pass (-1 none).
struct LTab {
  int len, firstc, lastc, firstm;  // first compute, last compute, first comm index (-1 if none)
  int64_t sum;
  int64_t dur[kLmax], koff[kLmax];
  int16_t nsame[kLmax];
  uint8_t kind[kLmax];
};

// list `id` into T (one warp: parallel loads, then lane 0 scans smem)
__device__ void load_ltab(const Cfg& c, int id, LTab& T) {
  const int lane = threadIdx.x & 31, off = c.loff[id], len = c.loff[id + 1] - off;
  for (int i = lane; i < len; i += 32) {
    T.dur[i] = c.lns[off + i];
    T.kind[i] = (uint8_t)(c.lkind[off + i] != 0);
  }
  __syncwarp();
  if (lane == 0) {
    T.len = len;
    T.firstc = T.lastc = T.firstm = -1;
    int64_t a = 0;
    int lastk[2] = {-1, -1};
    for (int i = 0; i < len; ++i) {
      T.koff[i] = a;
      a += T.dur[i];
      const int k = T.kind[i];
      if (k == 0) {
        if (T.firstc < 0) T.firstc = i;
        T.lastc = i;
      } else if (T.firstm < 0) {
        T.firstm = i;
      }
      if (lastk[k] >= 0) T.nsame[lastk[k]] = (int16_t)i;
      lastk[k] = i;
      T.nsame[i] = -1;
    }
    T.sum = a;
  }
  __syncwarp();
}

// The kernels of stage s in time order: kernel kk is kernel i of layer pass
// rep of op q.  Its gap to the next kernel of the same kind (R6): after a
// compute kernel the compute-free interval (end, next compute start), after
// a comm kernel the comm-free piece clipped to [w, z].  Returns 1 / 2 for a
// compute / comm interval (lo, hi), 0 for none.
__device__ __forceinline__ int gap_after(const LTab& Lf, const LTab& Lb, const int64_t* ost, const uint8_t* opfwd,
                                         int nops, int lc, int q, int r, int64_t w, int64_t z, int64_t& lo,
                                         int64_t& hi) {
  const LTab& L = opfwd[q] ? Lf : Lb;
  const int rep = r / L.len, i = r - rep * L.len;
  const int kind = L.kind[i];
  const int64_t base = ost[q] + (int64_t)rep * L.sum;
  const int64_t en = base + L.koff[i] + L.dur[i];
  int64_t nxt = kInf;
  const int j = L.nsame[i];
  if (j >= 0) {
    nxt = base + L.koff[j];
  } else if (rep < lc - 1) {
    const int f = kind == 0 ? L.firstc : L.firstm;
    nxt = base + L.sum + L.koff[f];
  } else if (q < nops - 1) {
    const LTab& L2 = opfwd[q + 1] ? Lf : Lb;
    const int f = kind == 0 ? L2.firstc : L2.firstm;
    if (f >= 0) nxt = ost[q + 1] + L2.koff[f];
  }
  if (kind == 0) {
    if (nxt != kInf && nxt > en) { lo = en; hi = nxt; return 1; }  // compute-free gap
  } else {
    const int64_t a = max(en, w), b = min(nxt, z);
    if (b > a) { lo = a; hi = b; return 2; }  // comm-free piece inside [w, z]
  }
  return 0;
}

__host__ __device__ __forceinline__ size_t k0_iv_bmx_offset(int nops) {
  return ((size_t)(nops + 1) * 4 + nops + 15) & ~size_t(15);
}
__host__ __device__ __forceinline__ size_t k0_iv_smem_bytes(int nops, int ci) {
  return k0_iv_bmx_offset(nops) + (size_t)4 * ci * 8;
}

// k0_intervals, one block per LLM stage: every thread takes a contiguous
// run of the stage's kernels, counts its intervals, one block scan gives
// the output offsets, a second pass writes them (time order is kernel order).
__global__ void __launch_bounds__(kIvThreads) k0_intervals(Cfg c) {
  using Scan = cub::BlockScan<unsigned long long, kIvThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ LTab Lf, Lb;
  __shared__ int run_c, run_m, head_m, tot_c, tot_m;
  // dynamic: [nops + 1] kernel offset of each op, [nops] op is forward, then
  // (8-aligned) bmx[4][ci_n]: the per-block capacity maxima being built
  extern __shared__ __align__(16) int opoff[];
  if (c.scal[2] == 0) return;     // template failed (deadlock): nothing to emit
  // kIvBlocks blocks per stage, each a contiguous share of its kernels; the
  // blocks of a stage exchange their interval counts through ivagg/ivflag
  const int s = blockIdx.x / kIvBlocks, bi = blockIdx.x % kIvBlocks, warp = threadIdx.x >> 5;
  const int p = c.p, v = c.v, n = c.n, nops = c.nops, lc = c.lc;
  const int Ws = c.W[s];
  uint8_t* opfwd = reinterpret_cast<uint8_t*>(opoff + nops + 1);
  const int CI = c.ci_n;
  long long* bmx = reinterpret_cast<long long*>(reinterpret_cast<unsigned char*>(opoff) + k0_iv_bmx_offset(nops));
  for (int i = threadIdx.x; i < 4 * CI; i += blockDim.x) bmx[i] = kNegInf;
  if (warp == 0) load_ltab(c, 0, Lf);
  if (warp == 1) load_ltab(c, 1, Lb);
  for (int q = threadIdx.x; q < nops; q += blockDim.x) opfwd[q] = (uint8_t)op_at(p, v, n, Ws, q).fwd;
  __syncthreads();
  if (nops <= kIvThreads) {  // kernel offset of each op: one block scan
    const int q = threadIdx.x;
    const unsigned long long x = q < nops ? (unsigned long long)(lc * (opfwd[q] ? Lf.len : Lb.len)) : 0ull;
    unsigned long long ex, all;
    Scan(tmp).ExclusiveSum(x, ex, all);
    if (q < nops) opoff[q] = (int)ex;
    if (q == 0) opoff[nops] = (int)all;
  } else if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < nops; ++q) {
      opoff[q] = acc;
      acc += lc * (opfwd[q] ? Lf.len : Lb.len);
    }
    opoff[nops] = acc;
  }
  __syncthreads();
  const int K = opoff[nops];
  const int64_t* ost = c.opstart + (int64_t)s * nops;
  // first op is always a forward, last always a backward
  const int64_t w = ost[0] + Lf.koff[Lf.firstc];
  const int64_t z = ost[nops - 1] + (int64_t)(lc - 1) * Lb.sum + Lb.koff[Lb.lastc] + Lb.dur[Lb.lastc];
  if (threadIdx.x == 0 && bi == 0) { c.w[s] = w; c.z[s] = z; }
  int64_t* clo = c.comp_lo + (int64_t)s * c.icapc;
  int64_t* chi = c.comp_hi + (int64_t)s * c.icapc;
  int64_t* mlo = c.comm_lo + (int64_t)s * c.icapm;
  int64_t* mhi = c.comm_hi + (int64_t)s * c.icapm;
  // head comm-free piece [w, first comm start) (R6), emitted first
  if (threadIdx.x == 0) {
    int64_t first_comm = kInf;
    if (Lf.firstm >= 0) first_comm = ost[0] + Lf.koff[Lf.firstm];
    const int64_t hi = min(first_comm, z);  // (both lists have comm or neither: validated)
    head_m = hi > w;
    if (hi > w && bi == 0) { mlo[0] = w; mhi[0] = hi; }
  }
  __syncthreads();
  const int Kb0 = (int)((int64_t)K * bi / kIvBlocks), Kb1 = (int)((int64_t)K * (bi + 1) / kIvBlocks);
  const int C = (Kb1 - Kb0 + kIvThreads - 1) / kIvThreads;
  const int k0 = min(Kb1, Kb0 + (int)threadIdx.x * C), k1 = min(Kb1, k0 + C);
  int q0 = 0;
  {  // op of kernel k0
    int lo = 0, hi = nops - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (opoff[mid] <= k0) lo = mid; else hi = mid - 1;
    }
    q0 = lo;
  }
  unsigned long long cnt = 0;  // compute | comm << 32
  for (int kk = k0, q = q0; kk < k1; ++kk) {
    while (kk >= opoff[q + 1]) ++q;
    int64_t lo, hi;
    const int g = gap_after(Lf, Lb, ost, opfwd, nops, lc, q, kk - opoff[q], w, z, lo, hi);
    cnt += g == 1 ? 1ull : g == 2 ? (1ull << 32) : 0ull;
  }
  unsigned long long off, tot;
  Scan(tmp).ExclusiveSum(cnt, off, tot);
  if (threadIdx.x == 0) {  // publish this block's counts, then gather the stage's
    unsigned long long* agg = c.ivagg + (int64_t)s * kIvBlocks;
    int* flag = c.ivflag + (int64_t)s * kIvBlocks;
    agg[bi] = tot;
    __threadfence();
    atomicExch(&flag[bi], 1);
    unsigned long long pre = 0, all = 0;
    for (int b = 0; b < kIvBlocks; ++b) {
      while (*(volatile int*)&flag[b] == 0) __nanosleep(64);
      __threadfence();
      const unsigned long long x = *(volatile unsigned long long*)&agg[b];
      all += x;
      if (b < bi) pre += x;
    }
    run_c = (int)(pre & 0xffffffffu);
    run_m = head_m + (int)(pre >> 32);
    tot_c = (int)(all & 0xffffffffu);
    tot_m = head_m + (int)(all >> 32);
  }
  __syncthreads();
  int oc = run_c + (int)(off & 0xffffffffu), om = run_m + (int)(off >> 32);
  // per 32-interval block, the largest base capacity hi - lo, in time order
  // (orientation 0) and in mirrored order (1, interval i' = count-1-i): no
  // kernel longer than it fits anywhere in the block (K1 skips such blocks)
  const int nc = tot_c, nm = tot_m;
  auto note = [&](int r, int idx, int count, int64_t cap) {
    atomicMax(&bmx[(r * 2 + 0) * CI + (idx >> 5)], (long long)cap);
    atomicMax(&bmx[(r * 2 + 1) * CI + ((count - 1 - idx) >> 5)], (long long)cap);
  };
  if (threadIdx.x == 0 && bi == 0 && head_m) note(1, 0, nm, mhi[0] - mlo[0]);  // the head comm-free piece
  for (int kk = k0, q = q0; kk < k1; ++kk) {
    while (kk >= opoff[q + 1]) ++q;
    int64_t lo, hi;
    const int g = gap_after(Lf, Lb, ost, opfwd, nops, lc, q, kk - opoff[q], w, z, lo, hi);
    if (g == 1) { clo[oc] = lo; chi[oc] = hi; note(0, oc, nc, hi - lo); ++oc; }
    if (g == 2) { mlo[om] = lo; mhi[om] = hi; note(1, om, nm, hi - lo); ++om; }
  }
  __syncthreads();
  if (threadIdx.x == 0 && bi == 0) { c.ncomp[s] = nc; c.ncomm[s] = nm; }
  for (int i = threadIdx.x; i < 4 * CI; i += blockDim.x)  // (c.bmax starts at -inf: k0_final)
    if (bmx[i] != kNegInf) atomicMax(reinterpret_cast<long long*>(&c.bmax[(int64_t)s * 4 * CI + i]), bmx[i]);
}

}  // namespace

// opt in to large dynamic shared memory (per device: capi's device_info runs it once per device)
void template_attrs() {
  cudaFuncSetAttribute(k0_wave, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k0_final, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k0_intervals, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);  // + ~11 KB static
}

cudaError_t launch_template(const Cfg& c, cudaStream_t st, int* launches) {
  const int wpb = k0_sim_warps(c.p, c.v, c.n);
  const size_t smem = k0_vtab_bytes(c.n, c.v) + (size_t)wpb * k0_warp_bytes(c.p, c.v, c.n);
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;
  const int nsim = 1 + c.k0_trials;
  k0_wave<<<(nsim + wpb - 1) / wpb, 32 * kSimWarps, smem, st>>>(c, nsim, wpb);
  k0_final<<<1, 32 * kSimWarps, smem, st>>>(c, wpb);
  k0_intervals<<<c.p * kIvBlocks, kIvThreads, k0_iv_smem_bytes(c.nops, c.ci_n), st>>>(c);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

}  // namespace optimus

#ifdef K0_CYC
extern "C" int optimus_debug_k0cyc(void* out) {
  return (int)cudaMemcpyFromSymbol(out, optimus::g_k0cyc, sizeof(optimus::g_k0cyc));
}
#endif
