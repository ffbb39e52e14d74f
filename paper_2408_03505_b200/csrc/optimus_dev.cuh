// optimus_dev.cuh — device-side layout shared by the liboptimus kernels.
// (Product code.  Nothing here is shared with oracle/.)
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace optimus {

// Debug builds (OPTIMUS_NVCC_EXTRA=-DOPTIMUS_DEVICE_CHECKS): bounds and
// protocol checks in the kernels; a failed check prints its site and traps.
// (compute-sanitizer is not available on the GPU pool.)
#ifdef OPTIMUS_DEVICE_CHECKS
#define OPT_CHECK(cond)                                                                              \
  do {                                                                                               \
    if (!(cond)) {                                                                                   \
      printf("OPT_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,          \
             (int)blockIdx.x, (int)threadIdx.x);                                                     \
      __trap();                                                                                      \
    }                                                                                                \
  } while (0)
#else
#define OPT_CHECK(cond) do { } while (0)
#endif

constexpr int64_t kInf = INT64_MAX / 4;   // "no finite shift" / +infinity
constexpr int64_t kNegInf = -(INT64_MAX / 4);
constexpr int kMaxP = 32;                 // LLM pipeline stages handled (one lane per stage in K0)
constexpr int kMaxN = 128;                // microbatches per LLM pipeline (K2 mode 1; mode 0, one lane per slot, takes n <= 32)
constexpr int kMaxNWarp = 32;             // n handled by K2 mode 0 (eval.cu) and K2 mode 1's compact scratch

// List ids in the packed input: 0 = LLM layer fwd, 1 = LLM layer bwd,
// 2 + 2*(branch*ntp + ti) = encoder layer fwd at TP option ti, +1 = bwd.
__host__ __device__ inline int enc_list_id(int b, int ti, int ntp, int bwd) { return 2 + 2 * (b * ntp + ti) + bwd; }

constexpr int kMaxE = 128;  // plans (validated at load)

// Per-plan descriptor (host-built at load, copied to the workspace).
struct PlanDesc {
  int32_t P, T, ti, m, rp, rt, kmax, pad;
  uint64_t first, count;
  // offsets, in int64 elements, of this plan's tables from Cfg::tables
  int64_t preF, preB, devF, devB, inbF, lenF, inbB, lenB;
  int64_t devK;       // rp*(n+1) words: uint32 order ranks of DEV_F then DEV_B (0 at cnt 0)
  int64_t bpF;        // [rp][kmax]: first LLM slot (1-based) whose F - L >= INB_F[a][k] (n+1: none)
  int64_t slot_base;  // first K1 scratch slot of this plan
  int64_t flag_base;  // first K1 flag of this plan: per row [kmax + 1] (0: forward done, v: stages that published version v)
  int64_t pflags;     // 1 word written by K1: bit 0 = PRE_EF strictly increasing over t = 1..n
  int64_t kj;         // [m][n+1] u64 findCritical keys per pipeline and count: low word forward, high word
                      // backward, each rank(DEV[a_j][c]) << 7 | (127 - j) (R11: max key = max DEV, lowest j)
};

// K1 work items of a plan (forward rows, backward (row, kf), its tables):
// K2 evaluates the plan's candidates once pdone reaches this
__host__ __device__ inline int plan_items(const PlanDesc& d) { return d.rp + d.rp * (d.kmax + 1) + 1; }

// Everything a kernel needs: scalars + device pointers into the workspace.
struct Cfg {
  int32_t p, t, v, n, lc, policy, nb, ntp, E;
  int32_t nops;          // 2*n*v ops per stage
  int32_t icapc, icapm;  // interval capacity per stage: compute-free, comm-free
  int32_t kmax_all;      // max kmax over plans
  int32_t k0_trials;     // sum over stages of (Wdef_s + 1): K0 warm-up trials
  int32_t nk_max;        // max over TP options of the encoder's total kernel count (all layers, all branches)
  int32_t ci_n;          // 32-interval blocks per interval list: ceil(max(icapc, icapm) / 32)
  int32_t nflags;        // K1 flags (zeroed by k0_final)
  int32_t mmax;          // largest m over plans with candidates (K2 mode 1 scratch instance)
  int64_t T_ag, T_rs, pp_p2p, enc_p2p, L;
  // packed inputs
  const int32_t* lkind;   // kernel kinds, all lists concatenated
  const int64_t* lns;     // kernel durations
  const int32_t* loff;    // list id -> [loff[id], loff[id+1])
  const int32_t* blayers; // [nb] encoder layers per branch
  // template (K0)
  int32_t* W;             // [p] adjusted warm-up counts (policy 1) or defaults
  int32_t* Wdef;          // [p]
  int64_t* scal;          // [0] span_def, [1] T_end, [2] ok flag, [3] K0 wave: span_def + 1 once known (0 before)
  int64_t* F;             // [n]
  int64_t* B;             // [n]
  int64_t* w;             // [p] first LLM compute instant
  int64_t* z;             // [p] last LLM compute end
  int64_t* opstart;       // [p][nops]
  int32_t* ncomp;         // [p]
  int32_t* ncomm;         // [p]
  int64_t* comp_lo;       // [p][icapc] compute-free interval starts
  int64_t* comp_hi;       // [p][icapc] compute-free interval ends
  int64_t* comm_lo;       // [p][icapm]
  int64_t* comm_hi;       // [p][icapm]
  int64_t* bmax;          // [p][2 resources][2 orientations][ci_n]: max base capacity (hi - lo) per 32-interval block
  unsigned long long* ivagg;  // [p][8] k0_intervals per-block interval counts (compute | comm << 32)
  int32_t* ivflag;            // [p][8] ... published (zeroed by k0_final)
  int32_t* bestw;         // [p] K0 warm-up search: smallest successful w per stage
  int64_t* k0res;         // [1 + k0_trials] K0 wave: span of each simulation, -1 if it deadlocks
  // plans + tables (K1)
  const PlanDesc* plans;  // [E]
  int64_t* tables;
  int64_t* snap;          // [slots][icapc+icapm] forward fill snapshots (slot k=0 is the working copy)
  int64_t* bfill;         // [slots][icapc+icapm] backward (mirrored) fill state
  int16_t* snap_own;      // [slots][2][ci_n] owner version of each 32-block of each snapshot (-1 untouched)
  int32_t* k1flags;       // K1 forward -> backward progress flags (PlanDesc::flag_base); zeroed by k0_final
  const int32_t* k1units; // K1 work list: type << 30 | e << 16 | a << 8 | kf (type 0 forward, 1 backward, 2 plan tables)
  int32_t k1_total;       // K1 work items
  int32_t sms;            // SM count of the device (persistent grids)
  int32_t k1_grid;        // persistent K1 grid (set at load)
  int32_t* k1next;        // K1 work counter (persistent blocks); zeroed by k0_final
  int32_t* pdone;         // [E] K1 work items of each plan completed (release); zeroed by k0_final
  unsigned long long* pclaim;  // [E] K2 chunks of each plan claimed; zeroed by K3
  const int32_t* k2order; // plans with candidates, in the order K2 takes them (short chains first)
  int32_t n_k2order;
  const uint32_t* binom32;  // the same table saturated to 32 bits
  const uint64_t* binom;  // [S*S], S = B + 1 of the K2 mode 1 instance (33 / 65 / 129): C(a, b) at [a*S+b]; mode 0 reads it at S = 33
};

// Per-op identity in the Megatron interleaved 1F1B order (R2).
struct OpRef {
  int fwd, chunk, mb;
};

__host__ __device__ inline OpRef op_at(int p, int v, int n, int W, int pos) {
  int nv = n * v, k, fwd;
  if (pos < W) {
    k = pos;
    fwd = 1;
  } else {
    int r = pos - W;
    if (r < 2 * (nv - W)) {
      k = (r & 1) ? r / 2 : W + r / 2;
      fwd = (r & 1) ? 0 : 1;
    } else {
      k = (nv - W) + (r - 2 * (nv - W));
      fwd = 0;
    }
  }
  int ch = (k % (p * v)) / p;
  int mb = (k / (p * v)) * p + (k % p);
  return OpRef{fwd, fwd ? ch : v - 1 - ch, mb};
}

}  // namespace optimus

// Host launchers (defined in the .cu files).
namespace optimus {
cudaError_t launch_template(const Cfg& c, cudaStream_t st, int* launches);
cudaError_t launch_chain_tables(const Cfg& c, cudaStream_t st, int* launches);
size_t k1_smem_for(int nk, int p, int ci, int kmax_all);
int k1_grid(const Cfg& c);
size_t baseline_ws_bytes(int L, int VP, int p, int v, int n);
cudaError_t launch_baseline(const Cfg& c, int kind, int L, int Le, void* ws, int64_t** d_out, cudaStream_t st);
void template_attrs();
void chains_attrs();
void eval_thread_attrs();
cudaError_t launch_record(const Cfg& c, int e, int a, int kf, int klimit, int64_t* d_rec, cudaStream_t st);
cudaError_t launch_eff(const Cfg& c, const int64_t* d_explain, unsigned long long* d_out, cudaStream_t st);
struct EvalArgs {
  uint64_t begin, end;       // global index range (eval_candidates)
  uint32_t rank, world, block;
  const uint64_t* index;     // explicit indices (eval_indices) or nullptr
  uint64_t count;            // number of indices (explicit) / this rank's candidates
  int64_t* lat_out;          // nullable
  int64_t* best2;            // [2]
  int64_t* partials;         // [grid][2]
  unsigned long long* counter;
  uint64_t total;
  int grid;
  int mode;                   // 0: one candidate per warp (eval.cu), 1: one per thread (eval_thread.cu)
  cudaEvent_t ev0, ev1;       // optional: recorded around K2 for per-kernel timing
  unsigned long long* pclaim;  // [nplans] K2 per-plan chunk counters, reset by K3
  int nplans;
  unsigned long long* stats;  // [12] cumulative loop counts (optimus_eval_stats)
  // K2 mode 1, split: the fast kernel hands candidates the general kernel
  // evaluates through a global queue, a chunk of the range at a time
  unsigned long long* gq;     // [gqcap] g (~0: unused slot)
  unsigned long long* gqo;    // [gqcap] lat_out position | plan << 56
  unsigned long long* gqc;    // [gqcap] the packed composition (plans of m <= kPackParts) | first forward pick + 1
  long long* gqd;             // [gqcap] forward shift after that pick's commit (B = 32)
  unsigned int* gqn;          // slots reserved (warps take batches of kGqBatch)
  uint64_t gqcap;
  int64_t* partials2;         // [grid2][2] general kernel's block bests
  unsigned long long* counter2;  // general kernel's work counter
  unsigned int* gdone;        // general kernel blocks finished (its last block resets the counters)
  int grid2;
  int first_chunk;            // 1: blocks write their partials, 0: merge into them
};
#ifndef K2_GQBATCH
#define K2_GQBATCH 32  // >= 32 (one step of a warp); 64 measured 1% / 4% slower on 1 / 4 ranks (more half-used batches)
#endif
constexpr int kGqBatch = K2_GQBATCH;  // queue slots a fast-kernel warp reserves at a time
cudaError_t launch_eval(const Cfg& c, const EvalArgs& a, cudaStream_t st, int* launches);
cudaError_t launch_eval_thread(const Cfg& c, const EvalArgs& a, cudaStream_t st);
cudaError_t launch_explain(const Cfg& c, uint64_t g, int64_t* d_out, cudaStream_t st);
cudaError_t launch_order_dump(const Cfg& c, const int64_t* d_explain, int64_t* d_out, cudaStream_t st);
int eval_grid(int sms);
int eval_thread_grid(int sms, int instance);
int eval_general_grid(int sms, int instance);
int eval_thread_chunks(const EvalArgs& a);
int eval_thread_instance(int n, int mmax);
}  // namespace optimus
