// capi.cu — host side of liboptimus (include/optimus.h).
//
// Validation, model-planner enumeration + memory prune (§4.1/§4.5, P:296-314,
// P:482-496; a1 of SURVEY §8(a), host work at load), workspace layout,
// host->device copy of the packed problem, and the launches of the build
// kernels (template.cu, chains.cu) and the evaluation kernels (eval.cu).
// No search step runs on the host; there is no CPU fallback.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/optimus.h"
#include "optimus_dev.cuh"

using namespace optimus;

#ifndef K2_QUEUE_LOG2
#define K2_QUEUE_LOG2 26
#endif

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) return fail(OPTIMUS_ECUDA, "%s: %s", #x, cudaGetErrorString(e_));    \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct HostPlan {
  PlanDesc d;
  bool kept;
  int64_t dp_enc;
};

// Everything derived from the problem on the host: packed inputs, plans, layout.
struct Prep {
  int32_t p, t, v, n, lc, nb, ntp, nops, icapc, icapm;
  std::vector<int32_t> lkind, loff, blayers;
  std::vector<int64_t> lns;
  std::vector<uint64_t> binom;
  std::vector<uint32_t> binom32;  // the same, saturated to 32 bits (K2 unranks plans of < 2^32 candidates in 32 bits)
  std::vector<HostPlan> plans;
  uint64_t total = 0;
  int64_t n_tables = 0, n_slots = 0, fwd_units = 0, bwd_units = 0, n_flags = 0;
  std::vector<int32_t> units, k2order;
  int kmax_all = 0;
  int nk_max = 0;
  int k0_trials = 0;
  // layout (byte offsets in the workspace)
  size_t o_lkind, o_lns, o_loff, o_blayers, o_binom, o_binom32, o_plans, inputs_bytes;
  size_t o_W, o_Wdef, o_scal, o_F, o_B, o_w, o_z, o_opstart, o_ncomp, o_ncomm, o_comp_lo, o_comp_hi, o_comm_lo,
      o_comm_hi, o_bmax, o_sim, o_k0res, o_tables, o_snap, o_bfill, o_snap_own, o_units, o_k1flags, o_k2order, o_sync, o_iv, o_partials, o_counter, o_stats, o_gq, o_gqo, o_gqc, o_gqd, o_gqn, o_partials2, o_explain, o_order, o_rec, o_base, total_bytes;
  int base_L = 0, base_Le = 0;
  uint64_t gqcap = 0;  // Megatron baselines: layers in the sequence, encoder layers among them
  int grid;
};

int check_seq(const optimus_seq& s, const char* what, bool need_compute, bool allow_empty) {
  if (s.len < 0 || (s.len == 0 && !allow_empty)) return fail(OPTIMUS_EINVAL, "%s: empty kernel list", what);
  if (s.len > 0 && (!s.kind || !s.ns)) return fail(OPTIMUS_EINVAL, "%s: null array", what);
  bool comp = false;
  for (int i = 0; i < s.len; ++i) {
    if (s.kind[i] > 1) return fail(OPTIMUS_EINVAL, "%s[%d]: kind must be 0 (compute) or 1 (comm)", what, i);
    if (s.ns[i] <= 0) return fail(OPTIMUS_EINVAL, "%s[%d]: duration must be > 0 ns", what, i);
    comp |= s.kind[i] == 0;
  }
  if (need_compute && !comp) return fail(OPTIMUS_EINVAL, "%s: needs at least one compute kernel", what);
  return OPTIMUS_OK;
}

int runs_of(const optimus_seq& s, int kind) {
  int r = 0;
  for (int i = 0; i < s.len; ++i)
    if (s.kind[i] == kind && (i == 0 || s.kind[i - 1] != kind)) ++r;
  return r;
}

uint64_t binom_sat(int a, int b) {
  if (b < 0 || b > a) return 0;
  unsigned __int128 r = 1;
  b = b < a - b ? b : a - b;
  for (int i = 1; i <= b; ++i) {
    r = r * (unsigned __int128)(a - b + i) / (unsigned __int128)i;
    if (r > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
  }
  return (uint64_t)r;
}

int prepare(const optimus_problem* pb, Prep& X) {
  if (!pb) return fail(OPTIMUS_EINVAL, "problem is NULL");
  const optimus_plan& L = pb->llm;
  if (L.dp < 1 || L.pp < 1 || L.tp < 1 || L.v < 1) return fail(OPTIMUS_EINVAL, "LLM plan fields must be >= 1");
  if ((int64_t)L.dp * L.pp * L.tp != pb->n_gpu)
    return fail(OPTIMUS_EINVAL, "dp*pp*tp = %lld != n_gpu = %d", (long long)L.dp * L.pp * L.tp, pb->n_gpu);
  if (pb->llm_layers < 1 || pb->llm_layers % (L.pp * L.v) != 0)
    return fail(OPTIMUS_EINVAL, "llm_layers = %d is not a multiple of PP*V = %d", pb->llm_layers, L.pp * L.v);
  if (pb->n_mb < 1 || pb->n_mb % L.pp != 0)
    return fail(OPTIMUS_EINVAL, "n_mb = %d must be a positive multiple of PP = %d (interleaved 1F1B)", pb->n_mb, L.pp);
  if (pb->warmup_policy != 0 && pb->warmup_policy != 1) return fail(OPTIMUS_EINVAL, "warmup_policy must be 0 or 1");
  if (L.pp > kMaxP) return fail(OPTIMUS_ERANGE, "PP = %d exceeds the supported %d stages", L.pp, kMaxP);
  if (pb->n_mb > kMaxN) return fail(OPTIMUS_ERANGE, "n_mb = %d exceeds the supported %d", pb->n_mb, kMaxN);
  if (pb->dp_allgather_ns < 0 || pb->dp_reducescatter_ns < 0 || pb->pp_p2p_ns < 0 || pb->enc_p2p_ns < 0 ||
      pb->enc_llm_p2p_ns < 0)
    return fail(OPTIMUS_EINVAL, "DP/P2P durations must be >= 0");
  if (pb->bytes_per_param < 0 || pb->gpu_mem_bytes < 0 || pb->reserve_bytes < 0 || pb->llm_params < 0)
    return fail(OPTIMUS_EINVAL, "memory fields must be >= 0");
  int rc;
  if ((rc = check_seq(pb->llm_fwd_layer, "llm_fwd_layer", true, false))) return rc;
  if ((rc = check_seq(pb->llm_bwd_layer, "llm_bwd_layer", true, false))) return rc;
  if (pb->llm_fwd_layer.len > 256 || pb->llm_bwd_layer.len > 256)
    return fail(OPTIMUS_ERANGE, "LLM layer kernel lists longer than 256 kernels are not supported");
  if ((runs_of(pb->llm_fwd_layer, 1) > 0) != (runs_of(pb->llm_bwd_layer, 1) > 0))
    return fail(OPTIMUS_EINVAL, "llm_fwd_layer and llm_bwd_layer must both have TP comm kernels or neither");
  if (pb->n_branches < 1 || !pb->branch_layers || !pb->branch_params)
    return fail(OPTIMUS_EINVAL, "need at least one encoder branch");
  for (int b = 0; b < pb->n_branches; ++b)
    if (pb->branch_layers[b] < 1) return fail(OPTIMUS_EINVAL, "branch %d has %d layers (< 1)", b, pb->branch_layers[b]);
  // tp_opts must be exactly the divisors of llm.tp, ascending
  std::vector<int> divs;
  for (int d = 1; d <= L.tp; ++d)
    if (L.tp % d == 0) divs.push_back(d);
  if (pb->n_tp_opts != (int)divs.size() || !pb->tp_opts)
    return fail(OPTIMUS_EINVAL, "tp_opts must list the %zu divisors of tp = %d", divs.size(), L.tp);
  for (size_t i = 0; i < divs.size(); ++i)
    if (pb->tp_opts[i] != divs[i]) return fail(OPTIMUS_EINVAL, "tp_opts[%zu] = %d, expected %d", i, pb->tp_opts[i], divs[i]);
  if (!pb->enc_fwd_layer || !pb->enc_bwd_layer) return fail(OPTIMUS_EINVAL, "encoder layer lists are NULL");
  for (int i = 0; i < pb->n_branches * pb->n_tp_opts; ++i) {
    char nm[64];
    snprintf(nm, sizeof nm, "enc_fwd_layer[%d]", i);
    if ((rc = check_seq(pb->enc_fwd_layer[i], nm, false, true))) return rc;
    snprintf(nm, sizeof nm, "enc_bwd_layer[%d]", i);
    if ((rc = check_seq(pb->enc_bwd_layer[i], nm, false, true))) return rc;
  }

  X.p = L.pp; X.t = L.tp; X.v = L.v; X.n = pb->n_mb;
  X.lc = pb->llm_layers / (L.pp * L.v);
  X.nb = pb->n_branches;
  X.ntp = pb->n_tp_opts;
  X.nops = 2 * X.n * X.v;
  const int64_t nv = (int64_t)X.n * X.v;
  for (int s = 0; s < X.p; ++s) {  // K0 warm-up trials: every (stage, w <= Megatron default)
    const int d = X.v == 1 ? std::min(X.n, X.p - 1 - s)
                           : X.n == X.p ? X.n * X.v : std::min(X.n * X.v, 2 * (X.p - 1 - s) + (X.v - 1) * X.p);
    X.k0_trials += d + 1;
  }
  X.icapc = (int)(nv * X.lc * (runs_of(pb->llm_fwd_layer, 0) + runs_of(pb->llm_bwd_layer, 0)) + 1);
  X.icapm = (int)(nv * X.lc * (runs_of(pb->llm_fwd_layer, 1) + runs_of(pb->llm_bwd_layer, 1)) + 2);

  // packed kernel lists
  auto push = [&](const optimus_seq& s) {
    X.loff.push_back((int32_t)X.lkind.size());
    for (int i = 0; i < s.len; ++i) { X.lkind.push_back(s.kind[i]); X.lns.push_back(s.ns[i]); }
  };
  push(pb->llm_fwd_layer);
  push(pb->llm_bwd_layer);
  for (int b = 0; b < X.nb; ++b)
    for (int ti = 0; ti < X.ntp; ++ti) {
      push(pb->enc_fwd_layer[b * X.ntp + ti]);
      push(pb->enc_bwd_layer[b * X.ntp + ti]);
    }
  X.loff.push_back((int32_t)X.lkind.size());
  if (X.lkind.empty()) { X.lkind.push_back(0); X.lns.push_back(0); }
  X.blayers.assign(pb->branch_layers, pb->branch_layers + X.nb);
  for (int ti = 0; ti < X.ntp; ++ti) {  // encoder kernels per chain (K1 stages them in shared memory)
    int64_t nk = 0;
    for (int b = 0; b < X.nb; ++b)
      nk += (int64_t)pb->branch_layers[b] *
            std::max(pb->enc_fwd_layer[b * X.ntp + ti].len, pb->enc_bwd_layer[b * X.ntp + ti].len);
    if (nk > 8192) return fail(OPTIMUS_ERANGE, "encoder has %lld kernels per microbatch (> 8192 supported)", (long long)nk);
    X.nk_max = std::max<int>(X.nk_max, (int)nk);
  }
  if ((size_t)X.p * 2 * X.v * X.n * 8 + (size_t)X.p * X.nops * 8 + 4 * (size_t)X.n * X.v + 16 > 200 * 1024 ||
      (size_t)X.p * 2 * X.v * X.n > 32767)
    return fail(OPTIMUS_ERANGE, "PP*V*N_mb too large for the K0 shared-memory simulation");
  if ((size_t)(std::max(X.icapc, X.icapm) + 31) / 32 * 32 + (size_t)X.nops * 5 + 64 > 160 * 1024)
    return fail(OPTIMUS_ERANGE, "too many bubble intervals per stage for the K0 interval kernel");
  {  // row stride 33 / 65 / 129 by K2 mode 1 instance (mode 0 runs only at 33)
    const int S = (X.n <= 32 ? 32 : X.n <= 64 ? 64 : 128) + 1;  // = the K2 mode 1 instance's B + 1
    X.binom.assign((size_t)S * S, 0);
    for (int a = 0; a < S; ++a)
      for (int b = 0; b < S; ++b) X.binom[a * S + b] = binom_sat(a, b);
    X.binom32.resize(X.binom.size());
    for (size_t i = 0; i < X.binom.size(); ++i) X.binom32[i] = (uint32_t)std::min<uint64_t>(X.binom[i], UINT32_MAX);
  }

  // model planner: encoder plans (P | PP_llm, T | TP_llm), memory prune (R17, R19)
  int64_t phi_enc = 0;
  for (int b = 0; b < X.nb; ++b) phi_enc += pb->branch_params[b];
  const int64_t dp_llm = L.dp;
  uint64_t first = 0;
  int64_t toff = 0, slot = 0;
  for (int P = 1; P <= X.p; ++P) {
    if (X.p % P) continue;
    for (int ti = 0; ti < X.ntp; ++ti) {
      const int T = pb->tp_opts[ti];
      HostPlan hp;
      memset(&hp, 0, sizeof hp);
      PlanDesc& d = hp.d;
      d.P = P; d.T = T; d.ti = ti;
      d.rp = X.p / P; d.rt = X.t / T; d.m = d.rp * d.rt;
      hp.dp_enc = (int64_t)pb->n_gpu / ((int64_t)P * T);
      __int128 lhs = (__int128)pb->bytes_per_param * ((__int128)hp.dp_enc * phi_enc + (__int128)dp_llm * pb->llm_params) +
                     (__int128)pb->reserve_bytes * pb->n_gpu;
      __int128 rhs = (__int128)pb->gpu_mem_bytes * pb->n_gpu;
      hp.kept = lhs <= rhs;
      d.count = (hp.kept && d.m <= X.n) ? binom_sat(X.n - 1, d.m - 1) : 0;
      d.first = first;
      if (d.count > UINT64_MAX - first) return fail(OPTIMUS_ERANGE, "candidate count overflows uint64");
      first += d.count;
      if (d.count) {
        d.kmax = X.n - d.m + 1;  // most microbatches one pipeline can hold
        const int64_t np1 = X.n + 1;
        toff = (toff + 15) & ~int64_t(15);  // own 128-byte lines: K2 reads a plan's tables while K1 writes others
        d.preF = toff; toff += (int64_t)P * np1;
        d.preB = toff; toff += (int64_t)P * np1;
        d.devF = toff; toff += (int64_t)d.rp * np1;
        d.devB = toff; toff += (int64_t)d.rp * np1;
        d.devK = toff; toff += (int64_t)d.rp * np1;
        d.bpF = toff; toff += (int64_t)d.rp * d.kmax;
        d.pflags = toff; toff += 1;
        d.kj = toff; toff += (int64_t)d.m * np1;
        d.inbF = toff; toff += (int64_t)d.rp * d.kmax;
        d.lenF = toff; toff += d.rp;
        d.inbB = toff; toff += (int64_t)d.rp * (d.kmax + 1) * d.kmax;
        d.lenB = toff; toff += (int64_t)d.rp * (d.kmax + 1);
        d.slot_base = slot;
        slot += (int64_t)X.p * (d.kmax + 1);
        d.flag_base = X.n_flags;
        X.n_flags += (int64_t)d.rp * (d.kmax + 1);
        X.fwd_units += d.rp;
        X.bwd_units += (int64_t)d.rp * (d.kmax + 1);
        X.kmax_all = std::max(X.kmax_all, d.kmax);
      }
      X.plans.push_back(hp);
    }
  }
  X.total = first;
  {  // K1's per-block shared memory (kernel lists, coarse indices, block owners, chain status)
    const size_t per = k1_smem_for(X.nk_max, X.p, (std::max(X.icapc, X.icapm) + 31) / 32, X.kmax_all);
    if (per > 220 * 1024) return fail(OPTIMUS_ERANGE, "K1 shared-memory footprint %zu B exceeds 220 KB", per);
  }
  if (X.plans.size() > (size_t)kMaxE) return fail(OPTIMUS_ERANGE, "%zu encoder plans (> %d supported)", X.plans.size(), kMaxE);
  // K2 takes plans with more stages first: their chains are shorter, so K1
  // can finish them first
  for (size_t e = 0; e < X.plans.size(); ++e)
    if (X.plans[e].d.count) X.k2order.push_back((int32_t)e);
  // (fewer stages first measured 1.7x slower K2 on config 4)
  std::stable_sort(X.k2order.begin(), X.k2order.end(),
                   [&](int32_t x, int32_t y) { return X.plans[x].d.P > X.plans[y].d.P; });
  // K1 work list: every forward unit first (all start at once; a backward
  // unit only waits on forward units already taken), then every plan's
  // tables, then the backward units
  for (int32_t e : X.k2order)
    for (int a = 0; a < X.plans[e].d.rp; ++a) X.units.push_back((int32_t)(e << 16 | a << 8));
  // backward units by kf across the plans (kf-major): a unit comes after
  // every unit of a smaller kf, so it is usually taken once its version is
  // published, and the units of the long forward chains (the plans with the
  // largest kmax) come last (config 4's build 0.253 -> 0.221 ms against
  // plan by plan)
  for (int32_t e : X.k2order) X.units.push_back((int32_t)(2u << 30 | e << 16));
  for (int kf = 0; kf <= X.kmax_all; ++kf)
    for (int32_t e : X.k2order) {
      const PlanDesc& d = X.plans[e].d;
      if (kf > d.kmax) continue;
      for (int a = 0; a < d.rp; ++a) X.units.push_back((int32_t)(1u << 30 | e << 16 | a << 8 | kf));
    }
  X.n_flags = std::max<int64_t>(X.n_flags, 1);
  X.n_tables = std::max<int64_t>(toff, 1);
  X.n_slots = std::max<int64_t>(slot, 1);

  // workspace layout
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align256(o + bytes); return r; };
  X.o_lkind = take(X.lkind.size() * 4);
  X.o_lns = take(X.lns.size() * 8);
  X.o_loff = take(X.loff.size() * 4);
  X.o_blayers = take(X.blayers.size() * 4);
  X.o_binom = take(X.binom.size() * 8);
  X.o_binom32 = take(X.binom32.size() * 4);
  X.o_plans = take(X.plans.size() * sizeof(PlanDesc));
  X.o_units = take(std::max<size_t>(X.units.size(), 1) * 4);
  X.o_k2order = take(std::max<size_t>(X.k2order.size(), 1) * 4);
  X.inputs_bytes = o;
  X.o_W = take(X.p * 4);
  X.o_Wdef = take(X.p * 4);
  X.o_scal = take(4 * 8);
  X.o_F = take(X.n * 8);
  X.o_B = take(X.n * 8);
  X.o_w = take(X.p * 8);
  X.o_z = take(X.p * 8);
  X.o_opstart = take((size_t)X.p * X.nops * 8);
  X.o_ncomp = take(X.p * 4);
  X.o_ncomm = take(X.p * 4);
  X.o_comp_lo = take((size_t)X.p * X.icapc * 8);
  X.o_comp_hi = take((size_t)X.p * X.icapc * 8);
  X.o_comm_lo = take((size_t)X.p * X.icapm * 8);
  X.o_comm_hi = take((size_t)X.p * X.icapm * 8);
  X.o_bmax = take((size_t)X.p * 4 * ((std::max(X.icapc, X.icapm) + 31) / 32) * 8);
  X.o_sim = take((size_t)X.p * 4);
  X.o_k0res = take((size_t)(1 + X.k0_trials) * 8);
  X.o_tables = take((size_t)X.n_tables * 8);
  X.o_snap = take((size_t)X.n_slots * (X.icapc + X.icapm) * 8);
  X.o_bfill = take((size_t)X.n_slots * (X.icapc + X.icapm) * 8);
  X.o_k1flags = take((size_t)X.n_flags * 4);
  X.o_sync = take(64 + (size_t)kMaxE * (4 + 8));  // k1next (+ development probes), pdone[E], pclaim[E]
  X.o_iv = take((size_t)X.p * 8 * (8 + 4));          // k0_intervals block exchange
  X.o_snap_own = take((size_t)X.n_slots * 2 * ((std::max(X.icapc, X.icapm) + 31) / 32) * 2);
  X.grid = 148 * 8;  // upper bound for partials; actual grid set at load
  X.o_partials = take((size_t)4096 * 2 * 8);
  // K2 mode 1's queue from the fast to the general kernel: a chunk of up to
  // 2^K2_QUEUE_LOG2 candidates + the batches the fast warps (<= 4096 blocks
  // of 4) may leave partly used (16 B per slot)
  X.gqcap = std::min<uint64_t>(X.total, (uint64_t)1 << K2_QUEUE_LOG2) + (uint64_t)kGqBatch * 4096 * 4;
  X.o_gq = take((size_t)X.gqcap * 8);
  X.o_gqo = take((size_t)X.gqcap * 8);
  X.o_gqc = take((size_t)X.gqcap * 8);
  X.o_gqd = take((size_t)X.gqcap * 8);
  X.o_gqn = take(64);  // [0] u32 reserved slots, [8] u64 general kernel's work counter, [16] u32 blocks done
  X.o_partials2 = take((size_t)4096 * 2 * 8);
  X.o_counter = take(8);
  X.o_stats = take(16 * 8);
  X.o_explain = take((size_t)(8 + 2 * kMaxN + 3 * kMaxN + 4) * 8);  // + the efficiency sums
  X.o_order = take((size_t)2 * kMaxN * 8);
  X.o_rec = take((size_t)std::max(1, X.kmax_all) * std::max(1, X.nk_max) * 4 * 8);
  for (int b = 0; b < X.nb; ++b) X.base_Le += X.blayers[b];
  X.base_L = X.base_Le + pb->llm_layers;
  X.o_base = take(baseline_ws_bytes(X.base_L, X.p * X.v, X.p, X.v, X.n));
  X.total_bytes = o;
  return OPTIMUS_OK;
}

}  // namespace

struct optimus_ctx {
  Prep X;
  Cfg cfg;
  char* ws = nullptr;
  int sms = 0;
  int grid = 0, grid_thread = 0, grid_general = 0;
  int mode = 1;  // K2 variant: 1 = one candidate per thread (default), 0 = one per warp
  int build_launches = 0, eval_launches = 0;
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};  // build start/end, K2 start/end
  ~optimus_ctx() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

// Per-device launch state.  Function attributes (large dynamic shared memory
// opt-ins) are per device, so they are set the first time a device is used;
// the occupancy-derived persistent grids follow.  Guarded for loads from
// several host threads (distinct ctxs are independent, §8(b)).
struct DeviceInfo {
  int grid = 0;
  int grid_thread[6] = {0, 0, 0, 0, 0, 0};
  int grid_general[6] = {0, 0, 0, 0, 0, 0};
};

DeviceInfo device_info(int dev, int sms) {
  static std::mutex mu;
  static std::map<int, DeviceInfo> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  template_attrs();
  chains_attrs();
  eval_thread_attrs();
  DeviceInfo d;
  d.grid = std::min(4096, eval_grid(sms));
  for (int i = 0; i < 6; ++i) d.grid_thread[i] = std::min(4096, eval_thread_grid(sms, i));
  for (int i = 0; i < 6; ++i) d.grid_general[i] = std::min(4096, eval_general_grid(sms, i));
  cache[dev] = d;
  return d;
}

// largest m over plans with candidates (sizes K2 mode 1's per-thread scratch)
static int plans_mmax(const Prep& X) {
  int mm = 1;
  for (const auto& h : X.plans)
    if (h.d.count) mm = std::max(mm, (int)h.d.m);
  return mm;
}

Cfg make_cfg(const Prep& X, const optimus_problem* pb, char* ws) {
  Cfg c;
  memset(&c, 0, sizeof c);
  c.mmax = plans_mmax(X);
  c.p = X.p; c.t = X.t; c.v = X.v; c.n = X.n; c.lc = X.lc; c.policy = pb->warmup_policy;
  c.nb = X.nb; c.ntp = X.ntp; c.E = (int)X.plans.size(); c.nops = X.nops;
  c.icapc = X.icapc; c.icapm = X.icapm; c.kmax_all = X.kmax_all; c.nk_max = std::max(1, X.nk_max);
  c.T_ag = pb->dp_allgather_ns; c.T_rs = pb->dp_reducescatter_ns; c.pp_p2p = pb->pp_p2p_ns;
  c.enc_p2p = pb->enc_p2p_ns; c.L = pb->enc_llm_p2p_ns;
  c.lkind = (const int32_t*)(ws + X.o_lkind);
  c.lns = (const int64_t*)(ws + X.o_lns);
  c.loff = (const int32_t*)(ws + X.o_loff);
  c.blayers = (const int32_t*)(ws + X.o_blayers);
  c.binom = (const uint64_t*)(ws + X.o_binom);
  c.binom32 = (const uint32_t*)(ws + X.o_binom32);
  c.plans = (const PlanDesc*)(ws + X.o_plans);
  c.W = (int32_t*)(ws + X.o_W);
  c.Wdef = (int32_t*)(ws + X.o_Wdef);
  c.scal = (int64_t*)(ws + X.o_scal);
  c.F = (int64_t*)(ws + X.o_F);
  c.B = (int64_t*)(ws + X.o_B);
  c.w = (int64_t*)(ws + X.o_w);
  c.z = (int64_t*)(ws + X.o_z);
  c.opstart = (int64_t*)(ws + X.o_opstart);
  c.ncomp = (int32_t*)(ws + X.o_ncomp);
  c.ncomm = (int32_t*)(ws + X.o_ncomm);
  c.comp_lo = (int64_t*)(ws + X.o_comp_lo);
  c.comp_hi = (int64_t*)(ws + X.o_comp_hi);
  c.comm_lo = (int64_t*)(ws + X.o_comm_lo);
  c.comm_hi = (int64_t*)(ws + X.o_comm_hi);
  c.bmax = (int64_t*)(ws + X.o_bmax);
  c.ci_n = (std::max(X.icapc, X.icapm) + 31) / 32;
  c.nflags = (int32_t)X.n_flags;
  c.bestw = (int32_t*)(ws + X.o_sim);
  c.k0res = (int64_t*)(ws + X.o_k0res);
  c.k0_trials = X.k0_trials;
  c.tables = (int64_t*)(ws + X.o_tables);
  c.snap = (int64_t*)(ws + X.o_snap);
  c.bfill = (int64_t*)(ws + X.o_bfill);
  c.snap_own = (int16_t*)(ws + X.o_snap_own);
  c.k1flags = (int32_t*)(ws + X.o_k1flags);
  c.k1units = (const int32_t*)(ws + X.o_units);
  c.k1_total = (int32_t)X.units.size();
  c.k1next = (int32_t*)(ws + X.o_sync);
  c.pdone = (int32_t*)(ws + X.o_sync + 64);
  c.pclaim = (unsigned long long*)(ws + X.o_sync + 64 + (size_t)kMaxE * 4);
  c.k2order = (const int32_t*)(ws + X.o_k2order);
  c.ivagg = (unsigned long long*)(ws + X.o_iv);
  c.ivflag = (int32_t*)(ws + X.o_iv + (size_t)X.p * 8 * 8);
  c.n_k2order = (int32_t)X.k2order.size();
  return c;
}

int build(optimus_ctx* c, cudaStream_t st) {
  c->build_launches = 0;
  if (c->timing) CK(cudaEventRecord(c->ev[0], st));
  CK(launch_template(c->cfg, st, &c->build_launches));
  CK(launch_chain_tables(c->cfg, st, &c->build_launches));
  if (c->timing) CK(cudaEventRecord(c->ev[1], st));
  return OPTIMUS_OK;
}

}  // namespace

extern "C" {

const char* optimus_last_error(void) { return g_err.c_str(); }

int optimus_workspace_bytes(const optimus_problem* pb, size_t* bytes) {
  if (!bytes) return fail(OPTIMUS_EINVAL, "bytes is NULL");
  Prep X;
  int rc = prepare(pb, X);
  if (rc) return rc;
  *bytes = X.total_bytes;
  return OPTIMUS_OK;
}

int optimus_load_costs(const optimus_problem* pb, void* d_workspace, size_t bytes, void* cuda_stream,
                       optimus_ctx** out) {
  if (!out) return fail(OPTIMUS_EINVAL, "out is NULL");
  *out = nullptr;
  optimus_ctx* c = new optimus_ctx;
  int rc = prepare(pb, c->X);
  if (rc) { delete c; return rc; }
  const Prep& X = c->X;
  if (c->X.total == 0) { delete c; return fail(OPTIMUS_EINFEASIBLE, "no feasible plan"); }
  if (!d_workspace || ((uintptr_t)d_workspace & 255)) { delete c; return fail(OPTIMUS_EINVAL, "workspace must be a 256-byte aligned device pointer"); }
  if (bytes < X.total_bytes) {
    delete c;
    return fail(OPTIMUS_ENOSPACE, "workspace has %zu bytes, needs %zu", bytes, X.total_bytes);
  }
  int dev = 0;
  int sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) { delete c; return fail(OPTIMUS_ECUDA, "no usable CUDA device: %s", cudaGetErrorString(e)); }
  c->sms = sms;
  const DeviceInfo di = device_info(dev, sms);  // function attributes + occupancy, once per device
  c->grid = di.grid;
  c->grid_thread = di.grid_thread[eval_thread_instance(X.n, plans_mmax(X))];  // K2 mode 1 instance
  c->grid_general = di.grid_general[eval_thread_instance(X.n, plans_mmax(X))];
  c->ws = (char*)d_workspace;
  c->cfg = make_cfg(X, pb, c->ws);
  c->cfg.sms = sms;
  c->cfg.k1_grid = k1_grid(c->cfg);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  // one host->device copy of the packed inputs (the problem's cost tables)
  std::vector<char> h(X.inputs_bytes, 0);
  memcpy(h.data() + X.o_lkind, X.lkind.data(), X.lkind.size() * 4);
  memcpy(h.data() + X.o_lns, X.lns.data(), X.lns.size() * 8);
  memcpy(h.data() + X.o_loff, X.loff.data(), X.loff.size() * 4);
  memcpy(h.data() + X.o_blayers, X.blayers.data(), X.blayers.size() * 4);
  memcpy(h.data() + X.o_binom, X.binom.data(), X.binom.size() * 8);
  memcpy(h.data() + X.o_binom32, X.binom32.data(), X.binom32.size() * 4);
  for (size_t i = 0; i < X.plans.size(); ++i) memcpy(h.data() + X.o_plans + i * sizeof(PlanDesc), &X.plans[i].d, sizeof(PlanDesc));
  memcpy(h.data() + X.o_units, X.units.data(), X.units.size() * 4);
  memcpy(h.data() + X.o_k2order, X.k2order.data(), X.k2order.size() * 4);
  e = cudaMemcpyAsync(c->ws, h.data(), h.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + X.o_counter, 0, 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + X.o_stats, 0, 16 * 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + X.o_scal, 0, 4 * 8, st);  // scal[3] = 0: K0 wave protocol
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + X.o_sync, 0, 64 + (size_t)kMaxE * 12, st);  // K1/K2 counters
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + X.o_iv, 0, (size_t)X.p * 8 * 12, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->ws + X.o_gqn, 0, 64, st);  // K2 queue counters (then kept by k2_general)
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // h is pageable and goes out of scope
  if (e != cudaSuccess) { delete c; return fail(OPTIMUS_ECUDA, "copying inputs: %s", cudaGetErrorString(e)); }
  rc = build(c, st);
  if (rc) { delete c; return rc; }
  *out = c;
  return OPTIMUS_OK;
}

int optimus_plan_only(const optimus_problem* pb, optimus_ctx** out) {
  if (!out) return fail(OPTIMUS_EINVAL, "out is NULL");
  *out = nullptr;
  optimus_ctx* c = new optimus_ctx;
  int rc = prepare(pb, c->X);
  if (rc) { delete c; return rc; }
  *out = c;
  return OPTIMUS_OK;
}

int optimus_rebuild(optimus_ctx* c, void* cuda_stream) {
  if (!c) return fail(OPTIMUS_EINVAL, "ctx is NULL");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  return build(c, (cudaStream_t)cuda_stream);
}

int optimus_num_candidates(const optimus_ctx* c, uint64_t* total, int32_t* n_plans) {
  if (!c) return fail(OPTIMUS_EINVAL, "ctx is NULL");
  if (total) *total = c->X.total;
  if (n_plans) *n_plans = (int32_t)c->X.plans.size();
  return OPTIMUS_OK;
}

int optimus_get_plan(const optimus_ctx* c, int32_t i, optimus_plan* enc, int32_t* m, uint64_t* first, uint64_t* count) {
  if (!c) return fail(OPTIMUS_EINVAL, "ctx is NULL");
  if (i < 0 || i >= (int)c->X.plans.size()) return fail(OPTIMUS_ERANGE, "plan %d out of range", i);
  const HostPlan& hp = c->X.plans[i];
  if (enc) { enc->dp = (int32_t)hp.dp_enc; enc->pp = hp.d.P; enc->tp = hp.d.T; enc->v = 1; }
  if (m) *m = hp.d.m;
  if (first) *first = hp.d.first;
  if (count) *count = hp.d.count;
  return OPTIMUS_OK;
}

static int eval_common(optimus_ctx* c, EvalArgs& a, cudaStream_t st) {
  a.partials = (int64_t*)(c->ws + c->X.o_partials);
  a.counter = (unsigned long long*)(c->ws + c->X.o_counter);
  a.total = c->X.total;
  a.mode = c->mode;
  if (c->mode == 0 && c->X.n > kMaxNWarp)
    return fail(OPTIMUS_ERANGE, "eval mode 0 (one lane per slot) takes n_mb <= %d; n_mb = %d needs mode 1", kMaxNWarp, c->X.n);
  a.grid = c->mode == 1 ? c->grid_thread : c->grid;
  a.stats = (unsigned long long*)(c->ws + c->X.o_stats);
  a.gq = (unsigned long long*)(c->ws + c->X.o_gq);
  a.gqo = (unsigned long long*)(c->ws + c->X.o_gqo);
  a.gqc = (unsigned long long*)(c->ws + c->X.o_gqc);
  a.gqd = (long long*)(c->ws + c->X.o_gqd);
  a.gqn = (unsigned int*)(c->ws + c->X.o_gqn);
  a.counter2 = (unsigned long long*)(c->ws + c->X.o_gqn + 8);
  a.gdone = (unsigned int*)(c->ws + c->X.o_gqn + 16);
  a.gqcap = c->X.gqcap;
  a.partials2 = (int64_t*)(c->ws + c->X.o_partials2);
  a.grid2 = c->mode == 1 ? c->grid_general : 0;
  a.pclaim = c->cfg.pclaim;
  a.nplans = c->cfg.E;
  a.ev0 = c->timing ? c->ev[2] : nullptr;
  a.ev1 = c->timing ? c->ev[3] : nullptr;
  c->eval_launches = 0;
  CK(launch_eval(c->cfg, a, st, &c->eval_launches));
  return OPTIMUS_OK;
}

int optimus_eval_candidates(optimus_ctx* c, uint64_t begin, uint64_t end, uint32_t rank, uint32_t world, uint32_t block,
                            int64_t* d_lat_out, int64_t* d_best2, void* cuda_stream) {
  if (!c || !d_best2) return fail(OPTIMUS_EINVAL, "ctx/best2 is NULL");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  if (begin > end || end > c->X.total)
    return fail(OPTIMUS_ERANGE, "range [%llu, %llu) outside [0, %llu)", (unsigned long long)begin,
                (unsigned long long)end, (unsigned long long)c->X.total);
  if (world == 0 || rank >= world) return fail(OPTIMUS_EINVAL, "rank %u / world %u", rank, world);
  if (block == 0) block = 4096;
  if (block % 64) return fail(OPTIMUS_EINVAL, "block must be a multiple of 64");
  EvalArgs a;
  memset(&a, 0, sizeof a);
  a.begin = begin; a.end = end; a.rank = rank; a.world = world; a.block = block;
  const uint64_t nblocks = (end - begin + block - 1) / block;
  a.count = rank < nblocks ? ((nblocks - 1 - rank) / world + 1) * (uint64_t)block : 0;
  a.lat_out = d_lat_out;
  a.best2 = d_best2;
  return eval_common(c, a, (cudaStream_t)cuda_stream);
}

int optimus_eval_indices(optimus_ctx* c, const uint64_t* d_index, uint64_t count, int64_t* d_lat_out, int64_t* d_best2,
                         void* cuda_stream) {
  if (!c || !d_best2 || (!d_index && count)) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  EvalArgs a;
  memset(&a, 0, sizeof a);
  a.index = d_index;
  a.count = count;
  a.lat_out = d_lat_out;
  a.best2 = d_best2;
  a.end = c->X.total;
  a.world = 1;
  a.block = 64;
  if (!d_index) {  // count == 0: nothing to do but a valid empty answer
    a.index = (const uint64_t*)(c->ws + c->X.o_counter);
  }
  return eval_common(c, a, (cudaStream_t)cuda_stream);
}

int optimus_best_plan(const optimus_ctx* c, const int64_t* h_best2_all_ranks, int32_t world, optimus_result* out,
                      int32_t* counts_out) {
  if (!c || !h_best2_all_ranks || !out || world < 1) return fail(OPTIMUS_EINVAL, "NULL argument");
  int64_t bl = INT64_MAX;
  uint64_t bg = 0;
  bool any = false;
  for (int r = 0; r < world; ++r) {
    const int64_t l = h_best2_all_ranks[2 * r];
    const int64_t g = h_best2_all_ranks[2 * r + 1];
    if (l == INT64_MAX || g < 0) continue;
    if (!any || l < bl || (l == bl && (uint64_t)g < bg)) { bl = l; bg = (uint64_t)g; any = true; }
  }
  if (!any) return fail(OPTIMUS_EINVAL, "no rank reported a candidate");
  if (bg >= c->X.total) return fail(OPTIMUS_ERANGE, "index %llu >= total", (unsigned long long)bg);
  for (const HostPlan& hp : c->X.plans) {
    if (!hp.d.count || bg < hp.d.first || bg >= hp.d.first + hp.d.count) continue;
    out->lat_ns = bl;
    out->index = bg;
    out->enc.dp = (int32_t)hp.dp_enc; out->enc.pp = hp.d.P; out->enc.tp = hp.d.T; out->enc.v = 1;
    out->m = hp.d.m;
    if (counts_out) {  // lexicographic unranking of the composition (R17)
      uint64_t rank = bg - hp.d.first;
      int rem = c->X.n;
      for (int j = 0; j < hp.d.m - 1; ++j) {
        const int parts = hp.d.m - j;
        int x = 1;
        for (; x <= rem - (parts - 1); ++x) {
          const uint64_t cnt = binom_sat(rem - x - 1, parts - 2);
          if (rank < cnt) break;
          rank -= cnt;
        }
        counts_out[j] = x;
        rem -= x;
      }
      counts_out[hp.d.m - 1] = rem;
    }
    return OPTIMUS_OK;
  }
  return fail(OPTIMUS_ERANGE, "index not in any plan");
}

int optimus_explain(const optimus_ctx* c, uint64_t g, int64_t* h_out, size_t cap, size_t* len, void* cuda_stream) {
  if (!c || !h_out || !len) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  if (g >= c->X.total) return fail(OPTIMUS_ERANGE, "index %llu >= %llu", (unsigned long long)g, (unsigned long long)c->X.total);
  int m = 0;
  for (const auto& hp : c->X.plans)
    if (hp.d.count && g >= hp.d.first && g < hp.d.first + hp.d.count) m = hp.d.m;
  const size_t need = 8 + 2 * (size_t)c->X.n + 3 * (size_t)m;
  if (cap < need) return fail(OPTIMUS_ERANGE, "cap %zu < %zu", cap, need);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int64_t* d = (int64_t*)(c->ws + c->X.o_explain);
  CK(launch_explain(c->cfg, g, d, st));
  std::vector<int64_t> buf(8 + 2 * kMaxN + 3 * kMaxN);
  CK(cudaMemcpyAsync(buf.data(), d, buf.size() * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int n = c->X.n;
  size_t o = 0;
  for (int i = 0; i < 8; ++i) h_out[o++] = buf[i];
  for (int i = 0; i < 2 * n; ++i) h_out[o++] = buf[8 + i];
  for (int i = 0; i < 3 * m; ++i) h_out[o++] = buf[8 + 2 * n + i];
  *len = o;
  return OPTIMUS_OK;
}

int optimus_efficiency(const optimus_ctx* c, uint64_t g, int64_t* h_out3, void* cuda_stream) {
  if (!c || !h_out3) return fail(OPTIMUS_EINVAL, "NULL argument");
  std::vector<int64_t> x(8 + 2 * kMaxN + 3 * kMaxN);
  size_t xl = 0;
  int rc = optimus_explain(c, g, x.data(), x.size(), &xl, cuda_stream);  // leaves its device output in place
  if (rc != OPTIMUS_OK) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int64_t* d = (int64_t*)(c->ws + c->X.o_explain);
  unsigned long long* dsum = (unsigned long long*)(d + 8 + 2 * kMaxN + 3 * kMaxN);
  CK(cudaMemsetAsync(dsum, 0, 3 * 8, st));
  CK(launch_eff(c->cfg, d, dsum, st));
  CK(cudaMemcpyAsync(h_out3, dsum, 3 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return OPTIMUS_OK;
}

int optimus_emit_schedule(const optimus_ctx* c, uint64_t g, int64_t* h_out, size_t cap, size_t* n_records,
                          void* cuda_stream) {
  if (!c || !h_out || !n_records) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  const Prep& X = c->X;
  std::vector<int64_t> x(8 + 2 * kMaxN + 3 * kMaxN);
  size_t xl = 0;
  int rc = optimus_explain(c, g, x.data(), x.size(), &xl, cuda_stream);
  if (rc != OPTIMUS_OK) return rc;
  const int n = X.n, e = (int)x[5], m = (int)x[6], nf = (int)x[3], nbk = (int)x[4];
  const PlanDesc& d = X.plans[e].d;
  const int64_t* N = &x[8 + 2 * n];
  const int64_t* cf = N + m;
  const int64_t* cbf = N + 2 * m;
  auto nk = [&](int bwd) {  // kernels of one chain (whole encoder, R8)
    int64_t t = 0;
    for (int b = 0; b < X.nb; ++b) {
      const int id = enc_list_id(b, d.ti, X.ntp, bwd);
      t += (int64_t)X.blayers[b] * (X.loff[id + 1] - X.loff[id]);
    }
    return t;
  };
  const int64_t nkF = nk(0), nkB = nk(1);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int64_t T_end = 0;
  CK(cudaMemcpyAsync(&T_end, c->cfg.scal + 1, 8, cudaMemcpyDeviceToHost, st));
  int64_t* drec = (int64_t*)(c->ws + X.o_rec);
  size_t out = 0;
  auto emit = [&](bool bwd, const std::vector<int64_t>& moves) -> int {
    // replays per (row, kf), as many chains as the row's pipelines need
    std::vector<int> taken(m, 0);
    std::vector<std::pair<int, int>> units;  // (row, kf)
    std::vector<int> need;
    for (int j = 0; j < m; ++j) {
      const int k = bwd ? (int)(N[j] - cbf[j]) : (int)(N[j] - cf[j]);
      if (k <= 0) continue;
      const std::pair<int, int> u{j / d.rt, bwd ? (int)(N[j] - cf[j]) : -1};
      size_t q = 0;
      while (q < units.size() && units[q] != u) ++q;
      if (q == units.size()) { units.push_back(u); need.push_back(0); }
      need[q] = std::max(need[q], k);
    }
    const int64_t per = bwd ? nkB : nkF;
    std::vector<std::vector<int64_t>> recs(units.size());
    for (size_t q = 0; q < units.size(); ++q) {
      CK(launch_record(c->cfg, e, units[q].first, units[q].second, need[q], drec, st));
      recs[q].resize((size_t)need[q] * per * 4);
      CK(cudaMemcpyAsync(recs[q].data(), drec, recs[q].size() * 8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    for (size_t t = 0; t < moves.size(); ++t) {
      const int js = (int)moves[t];
      const std::pair<int, int> u{js / d.rt, bwd ? (int)(N[js] - cf[js]) : -1};
      size_t q = 0;
      while (units[q] != u) ++q;
      const int k = taken[js]++;
      for (int64_t i = 0; i < per; ++i) {
        const int64_t* r = &recs[q][((size_t)k * per + i) * 4];
        if (out + 6 > cap) return fail(OPTIMUS_ERANGE, "cap too small for the schedule");
        h_out[out++] = js;
        h_out[out++] = r[0];
        h_out[out++] = r[1];
        h_out[out++] = bwd ? T_end - r[3] : r[2];  // backward: mirrored time back to real time (R15)
        h_out[out++] = bwd ? T_end - r[2] : r[3];
        h_out[out++] = (int64_t)t;
      }
    }
    return OPTIMUS_OK;
  };
  std::vector<int64_t> mf(x.begin() + 8, x.begin() + 8 + nf), mb(x.begin() + 8 + n, x.begin() + 8 + n + nbk);
  if ((rc = emit(false, mf)) != OPTIMUS_OK) return rc;
  const size_t nfwd = out / 6;
  if ((rc = emit(true, mb)) != OPTIMUS_OK) return rc;
  n_records[0] = nfwd;
  n_records[1] = out / 6 - nfwd;
  return OPTIMUS_OK;
}

int optimus_emit_p2p(const optimus_ctx* c, uint64_t g, int64_t* h_out, size_t cap, size_t* n_records,
                     void* cuda_stream) {
  if (!c || !h_out || !n_records) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  const Prep& X = c->X;
  const int n = X.n;
  if (cap < (size_t)n * 2 * 9) return fail(OPTIMUS_ERANGE, "cap %zu < %d", cap, n * 2 * 9);
  std::vector<int64_t> x(8 + 2 * kMaxN + 3 * kMaxN);
  size_t xl = 0;
  int rc = optimus_explain(c, g, x.data(), x.size(), &xl, cuda_stream);  // leaves its device output in place
  if (rc != OPTIMUS_OK) return rc;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int64_t* d_ord = (int64_t*)(c->ws + X.o_order);
  CK(launch_order_dump(c->cfg, (const int64_t*)(c->ws + X.o_explain), d_ord, st));
  std::vector<int64_t> ord(2 * (size_t)n), F(n), B(n);
  CK(cudaMemcpyAsync(ord.data(), d_ord, ord.size() * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(F.data(), c->cfg.F, n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(B.data(), c->cfg.B, n * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const PlanDesc& d = X.plans[(int)x[5]].d;
  const int64_t L = c->cfg.L;
  size_t o = 0;
  for (int i = 0; i < n; ++i) {  // a pair per microbatch and direction
    const int j = (int)ord[2 * i], a = j / d.rt, b = j % d.rt;
    const int64_t last = (int64_t)a * d.P + d.P - 1;  // LLM stage hosting pipeline j's last encoder stage (R7)
    const int64_t rf[9] = {0, i, j, last, b, 0, b, ord[2 * i + 1], ord[2 * i + 1] + L};
    const int64_t rb[9] = {1, i, j, 0, b, last, b, B[i], B[i] + L};
    for (int q = 0; q < 9; ++q) h_out[o++] = rf[q];
    for (int q = 0; q < 9; ++q) h_out[o++] = rb[q];
  }
  *n_records = 2 * (size_t)n;
  return OPTIMUS_OK;
}

int optimus_debug_template(const optimus_ctx* c, int64_t* h_out, size_t cap, size_t* len, void* cuda_stream) {
  if (!c || !h_out || !len) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  const Prep& X = c->X;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  CK(cudaStreamSynchronize(st));
  const int p = X.p, n = X.n;
  std::vector<int32_t> W(p), nc(p), nm(p);
  std::vector<int64_t> scal(4), F(n), B(n), w(p), z(p);
  CK(cudaMemcpy(W.data(), c->cfg.W, p * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(nc.data(), c->cfg.ncomp, p * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(nm.data(), c->cfg.ncomm, p * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(scal.data(), c->cfg.scal, 4 * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(F.data(), c->cfg.F, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(B.data(), c->cfg.B, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(w.data(), c->cfg.w, p * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(z.data(), c->cfg.z, p * 8, cudaMemcpyDeviceToHost));
  std::vector<int64_t> o;
  o.push_back(p); o.push_back(n); o.push_back(scal[1]); o.push_back(scal[0]);
  for (int s = 0; s < p; ++s) o.push_back(W[s]);
  for (int i = 0; i < n; ++i) o.push_back(F[i]);
  for (int i = 0; i < n; ++i) o.push_back(B[i]);
  for (int s = 0; s < p; ++s) o.push_back(w[s]);
  for (int s = 0; s < p; ++s) o.push_back(z[s]);
  for (int s = 0; s < p; ++s) o.push_back(nc[s]);
  for (int s = 0; s < p; ++s) o.push_back(nm[s]);
  for (int s = 0; s < p; ++s) {
    if (nc[s] < 0 || nc[s] > X.icapc || nm[s] < 0 || nm[s] > X.icapm) return fail(OPTIMUS_ERANGE, "interval count out of range");
    std::vector<int64_t> a(nc[s]), b(nc[s]), cc(nm[s]), d(nm[s]);
    CK(cudaMemcpy(a.data(), c->cfg.comp_lo + (size_t)s * X.icapc, nc[s] * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), c->cfg.comp_hi + (size_t)s * X.icapc, nc[s] * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cc.data(), c->cfg.comm_lo + (size_t)s * X.icapm, nm[s] * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(d.data(), c->cfg.comm_hi + (size_t)s * X.icapm, nm[s] * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < nc[s]; ++i) { o.push_back(a[i]); o.push_back(b[i]); }
    for (int i = 0; i < nm[s]; ++i) { o.push_back(cc[i]); o.push_back(d[i]); }
  }
  *len = o.size();
  if (o.size() > cap) return fail(OPTIMUS_ERANGE, "need %zu int64", o.size());
  memcpy(h_out, o.data(), o.size() * 8);
  return OPTIMUS_OK;
}

int optimus_debug_plan_tables(const optimus_ctx* c, int32_t i, int64_t* h_out, size_t cap, size_t* len,
                              void* cuda_stream) {
  if (!c || !h_out || !len) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (i < 0 || i >= (int)c->X.plans.size()) return fail(OPTIMUS_ERANGE, "plan %d out of range", i);
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  const PlanDesc& d = c->X.plans[i].d;
  if (!d.count) { *len = 0; return OPTIMUS_OK; }
  CK(cudaStreamSynchronize((cudaStream_t)cuda_stream));
  const int64_t np1 = c->X.n + 1;
  auto get = [&](int64_t off, int64_t cnt, std::vector<int64_t>& o) -> cudaError_t {
    std::vector<int64_t> tmp(cnt);
    cudaError_t e = cudaMemcpy(tmp.data(), c->cfg.tables + off, cnt * 8, cudaMemcpyDeviceToHost);
    o.insert(o.end(), tmp.begin(), tmp.end());
    return e;
  };
  std::vector<int64_t> o{d.rp, d.kmax};
  CK(get(d.lenF, d.rp, o));
  CK(get(d.inbF, (int64_t)d.rp * d.kmax, o));
  CK(get(d.lenB, (int64_t)d.rp * (d.kmax + 1), o));
  CK(get(d.inbB, (int64_t)d.rp * (d.kmax + 1) * d.kmax, o));
  CK(get(d.preF, d.P * np1, o));
  CK(get(d.preB, d.P * np1, o));
  *len = o.size();
  if (o.size() > cap) return fail(OPTIMUS_ERANGE, "need %zu int64", o.size());
  memcpy(h_out, o.data(), o.size() * 8);
  return OPTIMUS_OK;
}

int optimus_launch_count(const optimus_ctx* c, int32_t* build_launches, int32_t* eval_launches) {
  if (!c) return fail(OPTIMUS_EINVAL, "ctx is NULL");
  if (build_launches) *build_launches = c->build_launches;
  if (eval_launches) *eval_launches = c->eval_launches;
  return OPTIMUS_OK;
}

int optimus_baseline(optimus_ctx* c, int32_t kind, int64_t* h_out, size_t cap, size_t* len, void* cuda_stream) {
  if (!c || !h_out || !len) return fail(OPTIMUS_EINVAL, "NULL argument");
  if (!c->ws) return fail(OPTIMUS_EINVAL, "host-only context (optimus_plan_only) has no device state");
  if (kind != 0 && kind != 1) return fail(OPTIMUS_EINVAL, "kind must be 0 (naive) or 1 (balanced)");
  const Prep& X = c->X;
  if (kind == 1 && X.nb != 1)
    return fail(OPTIMUS_EINVAL, "the balanced partitioner is defined for a single encoder (P:778); %d branches", X.nb);
  const int VP = X.p * X.v;
  if (kind == 1 && X.base_L < VP)
    return fail(OPTIMUS_ERANGE, "%d layers cannot fill %d virtual stages", X.base_L, VP);
  const size_t need = 2 + 3 * (size_t)VP;
  if (cap < need) return fail(OPTIMUS_ERANGE, "cap %zu < %zu", cap, need);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  int64_t* d_out = nullptr;
  CK(launch_baseline(c->cfg, kind, X.base_L, X.base_Le, c->ws + X.o_base, &d_out, st));
  CK(cudaMemcpyAsync(h_out, d_out, need * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h_out[0] < 0) return fail(OPTIMUS_ECUDA, "baseline schedule deadlocked");
  *len = need;
  return OPTIMUS_OK;
}

int optimus_eval_instance(const optimus_ctx* c, int32_t* instance, int32_t* grid) {
  if (!c) return fail(OPTIMUS_EINVAL, "ctx is NULL");
  if (instance) *instance = eval_thread_instance(c->X.n, plans_mmax(c->X));
  if (grid) *grid = c->grid_thread;
  return OPTIMUS_OK;
}

int optimus_set_eval_mode(optimus_ctx* c, int mode) {
  if (!c || (mode != 0 && mode != 1)) return fail(OPTIMUS_EINVAL, "mode must be 0 (warp per candidate) or 1 (thread per candidate)");
  c->mode = mode;
  return OPTIMUS_OK;
}

int optimus_set_timing(optimus_ctx* c, int on) {
  if (!c || !c->ws) return fail(OPTIMUS_EINVAL, "ctx is NULL or host-only");
  if (on && !c->ev[0])
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
  c->timing = on != 0;
  return OPTIMUS_OK;
}

int optimus_last_timing(const optimus_ctx* c, float* build_ms, float* eval_ms) {
  if (!c || !c->timing) return fail(OPTIMUS_EINVAL, "timing is off (optimus_set_timing)");
  if (build_ms) {
    CK(cudaEventSynchronize(c->ev[1]));
    CK(cudaEventElapsedTime(build_ms, c->ev[0], c->ev[1]));
  }
  if (eval_ms) {
    CK(cudaEventSynchronize(c->ev[3]));
    CK(cudaEventElapsedTime(eval_ms, c->ev[2], c->ev[3]));
  }
  return OPTIMUS_OK;
}

int optimus_eval_stats(const optimus_ctx* c, uint64_t* h_out, void* cuda_stream) {
  if (!c || !c->ws || !h_out) return fail(OPTIMUS_EINVAL, "NULL argument or host-only ctx");
  CK(cudaStreamSynchronize((cudaStream_t)cuda_stream));
  uint64_t v[12];
  CK(cudaMemcpy(v, c->ws + c->X.o_stats, 12 * 8, cudaMemcpyDeviceToHost));
  // algorithmic 32-bit lane-ops per candidate (int64 add/compare/max = 2):
  // (17n + 4 + 2n lg) + 2m + 2 m it_f + 4 it_f + (10n+4) at_f + 2 m it_b + 4 it_b + (9n+4) at_b
  const uint64_t n = (uint64_t)c->X.n;
  uint64_t lg = 0;
  while ((1ull << lg) < std::max<uint64_t>(n, 2)) ++lg;
  h_out[0] = v[0];
  h_out[1] = v[0] * (17 * n + 4 + 2 * n * lg) + 2 * v[1] + 2 * v[2] + 4 * v[3] + (10 * n + 4) * v[4] + 2 * v[5] +
             4 * v[6] + (9 * n + 4) * v[7];
  h_out[2] = v[3];
  h_out[3] = v[4];
  h_out[4] = v[6];
  h_out[5] = v[7];
  h_out[6] = v[8];
  h_out[7] = v[9];
  h_out[8] = v[10];
  h_out[9] = v[11];
  return OPTIMUS_OK;
}

int optimus_io_bytes(const optimus_ctx* c, uint64_t* h2d, uint64_t* d2h) {
  if (!c) return fail(OPTIMUS_EINVAL, "ctx is NULL");
  if (h2d) *h2d = c->X.inputs_bytes;
  if (d2h) *d2h = 16;
  return OPTIMUS_OK;
}

void optimus_free(optimus_ctx* c) { delete c; }

// ---------------------------------------------------------------- NEXT-3
// A sweep over LLM templates (LLM plan, V, N_mb, warm-up policy): the
// planner fixes the LLM plan; the sweep makes it an outer axis
// of one search.  One context per template, laid out back to back in one
// workspace; eval enqueues every template's build and evaluation on one
// stream (each K2 overlapping its own K1) and writes each template's best.
struct optimus_sweep {
  std::vector<optimus_ctx*> ctx;
  ~optimus_sweep() {
    for (auto* c : ctx) delete c;
  }
};

int optimus_sweep_workspace_bytes(const optimus_problem* pbs, int32_t count, size_t* bytes) {
  if (!pbs || count < 1 || !bytes) return fail(OPTIMUS_EINVAL, "NULL argument or count < 1");
  size_t t = 0;
  for (int i = 0; i < count; ++i) {
    size_t b = 0;
    const int rc = optimus_workspace_bytes(&pbs[i], &b);
    if (rc) return rc;
    t += align256(b);
  }
  *bytes = t;
  return OPTIMUS_OK;
}

int optimus_sweep_load(const optimus_problem* pbs, int32_t count, void* d_workspace, size_t bytes, void* cuda_stream,
                       optimus_sweep** out) {
  if (!out) return fail(OPTIMUS_EINVAL, "out is NULL");
  *out = nullptr;
  size_t need = 0;
  int rc = optimus_sweep_workspace_bytes(pbs, count, &need);
  if (rc) return rc;
  if (bytes < need) return fail(OPTIMUS_ENOSPACE, "workspace has %zu bytes, the sweep needs %zu", bytes, need);
  optimus_sweep* sw = new optimus_sweep;
  size_t off = 0;
  for (int i = 0; i < count; ++i) {
    size_t b = 0;
    optimus_workspace_bytes(&pbs[i], &b);
    optimus_ctx* c = nullptr;
    rc = optimus_load_costs(&pbs[i], (char*)d_workspace + off, b, cuda_stream, &c);
    if (rc) {
      delete sw;
      return rc;
    }
    sw->ctx.push_back(c);
    off += align256(b);
  }
  *out = sw;
  return OPTIMUS_OK;
}

int optimus_sweep_eval(optimus_sweep* sw, uint32_t rank, uint32_t world, int64_t* d_best, void* cuda_stream) {
  if (!sw || !d_best) return fail(OPTIMUS_EINVAL, "NULL argument");
  for (size_t i = 0; i < sw->ctx.size(); ++i) {
    optimus_ctx* c = sw->ctx[i];
    int rc = optimus_rebuild(c, cuda_stream);
    if (!rc) rc = optimus_eval_candidates(c, 0, c->X.total, rank, world, 4096, nullptr, d_best + 2 * i, cuda_stream);
    if (rc) return rc;
  }
  return OPTIMUS_OK;
}

int optimus_sweep_ctx(optimus_sweep* sw, int32_t i, optimus_ctx** ctx) {
  if (!sw || !ctx || i < 0 || i >= (int)sw->ctx.size()) return fail(OPTIMUS_EINVAL, "bad sweep index");
  *ctx = sw->ctx[i];
  return OPTIMUS_OK;
}

void optimus_sweep_free(optimus_sweep* sw) { delete sw; }

}  // extern "C"
