/* optimus.h — C ABI of liboptimus: the data-parallel hot path of Optimus
 * (arXiv 2408.03505, "Accelerating Large-Scale Multi-Modal LLM Training by
 * Bubble Exploitation") on NVIDIA B200 (sm_100a).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, P:<line>):
 *   Alg. 1: over every encoder parallel plan kept by the model
 *   planner (§4.1; memory prune §4.5) and every
 *   partition of the N_mb microbatches over the m = DP_enc/DP_llm encoder
 *   pipelines, run BubbleScheduler (Alg. 2):
 *   coarse-grained initialisation, then OptimizeSchedule for the forward and
 *   the backward encoder work (findCritical -> ScheduleKernels ->
 *   checkEncLLMDep), packing encoder kernels into the bubbles of the LLM's
 *   interleaved-1F1B timeline (§4.2-4.3; multi-branch §4.4,
 *   P:470-480), and return the schedule with the smallest latency.
 *   Readings of every point the paper leaves open: DESIGN.md §3 (R1-R22).
 *
 * Conventions
 *   - All times are int64 nanoseconds; nothing is floating point.
 *   - Every int-returning call returns OPTIMUS_OK (0) or a negative code;
 *     optimus_last_error() then holds a thread-local message.
 *   - Device work is enqueued on the caller's CUDA stream (`cuda_stream`,
 *     a cudaStream_t; NULL = legacy default stream) and is asynchronous:
 *     synchronise that stream before reading device outputs.
 *   - The library never allocates device memory: the caller provides one
 *     workspace of optimus_workspace_bytes() bytes (256-byte aligned) and
 *     keeps it alive until optimus_free().  It never calls NCCL.
 *   - There is no CPU fallback: every step of the search runs in the
 *     library's sm_100a kernels; a missing/unsupported GPU -> OPTIMUS_ECUDA.
 *   - A context is not thread-safe; distinct contexts are independent.
 */
#ifndef OPTIMUS_H_
#define OPTIMUS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OPTIMUS_OK = 0,
  OPTIMUS_EINVAL = -1,      /* malformed problem or argument (message says which)      */
  OPTIMUS_EINFEASIBLE = -2, /* memory prune left no plan with m <= N_mb: "no feasible plan" */
  OPTIMUS_ECUDA = -3,       /* a CUDA error; message has cudaGetErrorString             */
  OPTIMUS_ENOSPACE = -4,    /* workspace smaller than optimus_workspace_bytes()         */
  OPTIMUS_ERANGE = -5       /* index range outside [0, total) or size limit exceeded    */
};

/* ParallelPlan (DP, PP, TP, V) — §4.1; V = model chunks (1 for encoders). */
typedef struct {
  int32_t dp, pp, tp, v;
} optimus_plan;

/* One profiled kernel sequence (a layer pass), in execution order.
 * kind[i]: 0 = compute kernel, 1 = TP communication kernel.
 * ns[i] > 0: duration.  Host arrays, owned by the caller, read during load. */
typedef struct {
  const uint8_t* kind;
  const int64_t* ns;
  int32_t len;
} optimus_seq;

/* The problem statement of Alg. 1: the MLLM (encoder branches +
 * LLM), the cluster, the LLM plan chosen "based on insights in Megatron-LM"
 * (P:303), N_mb, and profiled kernel durations. */
typedef struct {
  int32_t n_gpu;              /* GPUs; must equal llm.dp * llm.pp * llm.tp             */
  int64_t gpu_mem_bytes;      /* per-GPU capacity (§4.5 prune)                   */
  int64_t reserve_bytes;      /* per-GPU activation reserve subtracted from capacity    */
  int32_t bytes_per_param;    /* k in MEM_model (6 for bf16 params+fp32 grads)   */
  optimus_plan llm;           /* LLM (DP, PP, TP, V); interleaved 1F1B needs N_mb % PP == 0 */
  int32_t llm_layers;         /* multiple of PP * V                                      */
  int32_t n_mb;               /* N_mb, microbatches per LLM pipeline; <= 128 (ERANGE) */
  int32_t warmup_policy;      /* 0 = Megatron default warm-up, 1 = adjusted (§4.3) */
  optimus_seq llm_fwd_layer;  /* one LLM layer forward, >= 1 compute, <= 256 kernels     */
  optimus_seq llm_bwd_layer;  /* one LLM layer backward, >= 1 compute, <= 256 kernels    */
  int64_t dp_allgather_ns;    /* DP all-gather bubble before any LLM op          */
  int64_t dp_reducescatter_ns;/* DP reduce-scatter bubble after the last op      */
  int64_t pp_p2p_ns;          /* LLM stage-to-stage activation/gradient latency          */
  int64_t enc_p2p_ns;         /* encoder stage-to-stage latency                          */
  int64_t enc_llm_p2p_ns;     /* encoder <-> LLM latency L: EF_i+L <= F_i, EB_i >= B_i+L */
  int64_t llm_params;         /* phi_llm                                                 */
  int32_t n_branches;         /* encoder branches (§4.4), >= 1                           */
  const int32_t* branch_layers;  /* [n_branches], each >= 1                              */
  const int64_t* branch_params;  /* [n_branches]; phi_enc = their sum                    */
  int32_t n_tp_opts;          /* number of divisors of llm.tp                            */
  const int32_t* tp_opts;     /* all divisors of llm.tp, ascending (TP_enc options)      */
  const optimus_seq* enc_fwd_layer; /* [branch * n_tp_opts + tp_idx]: one encoder layer fwd at that TP */
  const optimus_seq* enc_bwd_layer; /* [branch * n_tp_opts + tp_idx]: one encoder layer bwd at that TP */
} optimus_problem;

/* One search answer: the best candidate (Alg. 1's bestSchedule). */
typedef struct {
  int64_t lat_ns;   /* schedule latency (Alg. 2 .lat)               */
  uint64_t index;   /* global candidate index (plan-major, lexicographic)  */
  optimus_plan enc; /* encoder (DP_enc, PP_enc, TP_enc, 1)                 */
  int32_t m;        /* encoder pipelines per LLM pipeline                  */
} optimus_result;

typedef struct optimus_ctx optimus_ctx; /* opaque; host memory owned by the library */

/* Size of the device workspace this problem needs.  Validates `pb`. */
int optimus_workspace_bytes(const optimus_problem* pb, size_t* bytes);

/* Validate and copy the problem (host -> device, on `cuda_stream`), enumerate
 * and prune the encoder plans (host), then build on the GPU: the LLM template
 * (interleaved-1F1B timeline, warm-up adjustment, dependency points F_i/B_i,
 * compute-free and comm-free bubble intervals per stage) and, per plan, the
 * coarse GPipe tables and the kernel-level first-fit chain tables.
 * d_workspace: device pointer, >= optimus_workspace_bytes().  *out receives
 * the context (NULL on error). */
int optimus_load_costs(const optimus_problem* pb, void* d_workspace, size_t bytes, void* cuda_stream,
                       optimus_ctx** out);

/* Host-only context: validation, plan enumeration, memory prune and
 * candidate counting, without touching a GPU.  Supports num_candidates,
 * get_plan, best_plan and free; device calls on it return OPTIMUS_EINVAL.
 * (Used by the multi-rank driver to decode gathered results, and by tests.) */
int optimus_plan_only(const optimus_problem* pb, optimus_ctx** out);

/* Re-run the GPU build (template + per-plan tables) from the device-resident
 * copy of the problem made by load (no host traffic).  For timing the whole
 * hot path with inputs already in HBM. */
int optimus_rebuild(optimus_ctx* c, void* cuda_stream);

/* Total candidates (sum over kept plans of C(N_mb-1, m-1)) and number of
 * enumerated plans (kept or not). */
int optimus_num_candidates(const optimus_ctx* c, uint64_t* total, int32_t* n_plans);

/* Plan i (0 <= i < n_plans) in enumeration order (ascending PP_enc, then
 * TP_enc): its plan, m, first global index and candidate count (0 if pruned
 * or m > N_mb). */
int optimus_get_plan(const optimus_ctx* c, int32_t i, optimus_plan* enc, int32_t* m, uint64_t* first,
                     uint64_t* count);

/* Evaluate candidates of [begin, end) owned by `rank` of `world`: the range
 * is cut into blocks of `block` indices (block % 64 == 0; 0 = default 4096)
 * and block b belongs to rank b % world.  d_lat_out (nullable, device,
 * int64[end-begin]): lat of every evaluated candidate at [g-begin] (other
 * ranks' entries untouched).  d_best2 (device, int64[2]): (lat, index) of
 * this rank's best candidate, ties -> lowest index; (INT64_MAX, -1) if the
 * rank owns nothing.  ERANGE if end > total or begin > end. */
int optimus_eval_candidates(optimus_ctx* c, uint64_t begin, uint64_t end, uint32_t rank, uint32_t world,
                            uint32_t block, int64_t* d_lat_out, int64_t* d_best2, void* cuda_stream);

/* Evaluate an explicit list of candidate indices (device uint64[count], each
 * < total): lat into d_lat_out[i] (nullable) and the best into d_best2. */
int optimus_eval_indices(optimus_ctx* c, const uint64_t* d_index, uint64_t count, int64_t* d_lat_out,
                         int64_t* d_best2, void* cuda_stream);

/* Host-side final step of Alg. 1 across ranks: lexicographic minimum of the
 * `world` (lat, index) pairs in h_best2_all_ranks (host int64[2*world]),
 * decoded into the plan and the microbatch partition: counts_out (host,
 * length >= N_mb) receives N_enc_1..N_enc_m.  EINVAL if no rank had one. */
int optimus_best_plan(const optimus_ctx* c, const int64_t* h_best2_all_ranks, int32_t world, optimus_result* out,
                      int32_t* counts_out);

/* Schedule decisions of one candidate g (the step after the
 * argmin; Alg. 2 P:335-354 and §4.2 P:387-400 for the moves):
 * re-evaluates g on the GPU and returns, in host h_out (int64, cap >= 8 +
 * 2*N_mb + 3*m, *len = entries written):
 *   [0] lat  [1] Delta_f  [2] Delta_b  [3] forward moves  [4] backward moves
 *   [5] plan index  [6] m  [7] N_mb
 *   [8, 8+N_mb)            pipeline of each committed forward move, in order
 *   [8+N_mb, 8+2*N_mb)     pipeline of each committed backward move, in order
 *   then N[m], the coarse forward counts c[m] and coarse backward counts cb[m]
 *   after both phases.  Pipeline j's k-th forward move is row (j / r_t)'s
 *   k-th chain (R-FACT), so these decisions and the chain tables fix every
 *   kernel placement.  ERANGE if g >= total or cap is too small; synchronises
 *   `cuda_stream`. */
int optimus_explain(const optimus_ctx* c, uint64_t g, int64_t* h_out, size_t cap, size_t* len, void* cuda_stream);

/* Scheduling efficiency of candidate g (§5.3.2
 * P:665 Eff_coarse / Eff_fine, reading R-EFF in DESIGN.md §3): host int64
 * h_out3 = [encoder work inside LLM bubbles with g's moves (fine + coarse),
 * the same without moves (coarse only), total encoder work], integer ns;
 * Eff_fine = h_out3[0] / h_out3[2], Eff_coarse = h_out3[1] / h_out3[2].
 * Synchronises `cuda_stream`. */
int optimus_efficiency(const optimus_ctx* c, uint64_t g, int64_t* h_out3, void* cuda_stream);

/* Schedule emission for candidate g: every encoder kernel
 * placed into the LLM bubbles by g's committed moves, replayed on the GPU
 * from the build's chain state (§4.2 ScheduleKernels P:347-400; R12, R15).
 * h_out (host int64, cap entries) receives records of 6 values
 *   [pipeline j, encoder stage, kind (0 compute, 1 comm), start, end, move t]
 * in real LLM-template time: first the forward moves in commit order, then
 * the backward ones; within a move, kernels in placement order (stage by
 * stage).  n_records[0] / [1] = forward / backward records.  Coarse (pre/
 * post-LLM) work is not listed: it is the GPipe fill of R9.  ERANGE if cap
 * is too small; synchronises `cuda_stream`. */
int optimus_emit_schedule(const optimus_ctx* c, uint64_t g, int64_t* h_out, size_t cap, size_t* n_records,
                          void* cuda_stream);

/* Introspection for parity tests (synchronises `cuda_stream`; device->host).
 * Template: h_out = [p, n, T_end, span_def, W'[p], F[n], B[n], w[p], z[p],
 * ncomp[p], ncomm[p], then per stage: compute-free (lo,hi)..., comm-free
 * (lo,hi)...]; *len = number of int64 written (ERANGE if cap too small). */
int optimus_debug_template(const optimus_ctx* c, int64_t* h_out, size_t cap, size_t* len, void* cuda_stream);

/* NEXT-4: the encoder-LLM P2P pairs of candidate g's schedule: for
 * every LLM microbatch i (the global ordering, R14, designates its encoder
 * pipeline j) a forward pair, activations from the last stage of pipeline j
 * to the first LLM stage, sent at j's forward finish EF_i and arriving at
 * EF_i + L <= F_i, and a backward pair, gradients from the first LLM stage
 * at B_i (end of its backward) to pipeline j's last stage, arriving at
 * B_i + L.  Reading R-P2P: endpoints are (LLM stage, TP slot b of pipeline
 * j = a r_t + b); pipeline j's last stage sits on LLM stage a P + P - 1
 * (R7).  Times are LLM-relative (template) ns: the executed schedule adds
 * Df.  h_out (cap >= 18 n): per record [dir 0 fwd / 1 bwd, microbatch i,
 * pipeline j, src stage, src slot, dst stage, dst slot, send ns, arrive ns],
 * 2 n records in slot order (forward, backward).  Synchronises the stream. */
int optimus_emit_p2p(const optimus_ctx* c, uint64_t g, int64_t* h_out, size_t cap, size_t* n_records,
                     void* cuda_stream);

/* Chain tables of plan i: h_out = [r_p, kmax, lenF[r_p], INB_F[r_p][kmax],
 * lenB[r_p][kmax+1], INB_B[r_p][kmax+1][kmax], PRE_F[P][n+1], PRE_B[P][n+1]].
 * Entries past a length are unspecified. */
int optimus_debug_plan_tables(const optimus_ctx* c, int32_t i, int64_t* h_out, size_t cap, size_t* len,
                              void* cuda_stream);

/* Kernel launches the last build / eval enqueued (for launch accounting). */
int optimus_launch_count(const optimus_ctx* c, int32_t* build_launches, int32_t* eval_launches);

/* Megatron-LM baselines: the iteration time of the
 * systems the paper's headline speedups are measured against (Table 5
 * P:598-600), under the same cost model, simulated on the GPU:
 *   kind 0, naive: every encoder layer (all branches, at the LLM's
 *          TP) runs in the first pipeline stage, in front of virtual stage
 *          0's LLM layers;
 *   kind 1, balanced (App. B): the layer sequence (encoder,
 *          then LLM) cut into V x PP contiguous virtual stages by App. B's DP
 *          (max virtual-stage time minimised; ties to the smallest cut);
 *          single encoder only (EINVAL otherwise); ERANGE if there are
 *          fewer layers than virtual stages.
 * Both run Megatron's default interleaved 1F1B warm-up from T_ag, + T_rs.
 * h_out (cap >= 2 + 3 V PP): [iteration ns, V PP, layers per virtual stage
 * [V PP], forward op ns per (stage, chunk) [PP][V], backward [PP][V]].
 * Synchronises the stream. */
int optimus_baseline(optimus_ctx* c, int32_t kind, int64_t* h_out, size_t cap, size_t* len, void* cuda_stream);

/* K2 mode 1 instance this context launches (sized by n_mb and the largest m
 * of a plan with candidates): 0 = (B, BM) (32, 32), 1 = (64, 64),
 * 2 = (128, 64), 3 = (128, 128), 4 = (64, 16), 5 = (128, 16) slots and
 * pipelines per thread; grid = its persistent grid (blocks).  Host only. */
int optimus_eval_instance(const optimus_ctx* c, int32_t* instance, int32_t* grid);

/* K2 variant used by the eval calls: 1 (default) = one candidate per thread
 * (eval_thread.cu), 0 = one candidate per warp (eval.cu).  Both compute the
 * same lat for every candidate (bit-exact); they differ only in speed.
 * Mode 0 puts one LLM slot on each lane and takes N_mb <= 32: the eval calls
 * return OPTIMUS_ERANGE for mode 0 at larger N_mb.  Mode 1 takes N_mb <= 128
 * (a compact per-thread scratch for N_mb <= 32, a wide one above). */
int optimus_set_eval_mode(optimus_ctx* c, int mode);

/* Per-kernel timing: when on, the library records CUDA events around each
 * build (K0+K1 launches) and around the K2 evaluation kernel on the stream
 * it launches them on; optimus_last_timing waits for them and returns the
 * elapsed milliseconds of the most recent build / K2 launch. */
int optimus_set_timing(optimus_ctx* c, int on);
int optimus_last_timing(const optimus_ctx* c, float* build_ms, float* eval_ms);

/* Cumulative K2 work counters since load (synchronises the stream):
 * h_out[10] = candidates evaluated, algorithmic 32-bit integer lane-ops
 * (DESIGN.md §5), forward loop iterations, forward move attempts, backward
 * iterations, backward attempts, candidates finished by K2 mode 1's fast
 * path, candidates evaluated by its general path, warp claims and lane
 * unrankings of its range path (the last four: mode 1 only, 0 in mode 0). */
int optimus_eval_stats(const optimus_ctx* c, uint64_t* h_out, void* cuda_stream);

/* Bytes load copies host->device (the packed problem) and one evaluation
 * returns device->host through best2 (16). */
int optimus_io_bytes(const optimus_ctx* c, uint64_t* h2d, uint64_t* d2h);

void optimus_free(optimus_ctx* c);

/* NEXT-3: a sweep over LLM templates.  The planner fixes the LLM plan (P:254,
 * P:303); a sweep makes (LLM plan, V, N_mb, warm-up policy) an outer axis of
 * one search: count problems (one per template, each validated as by
 * optimus_load_costs) loaded back to back into one caller workspace
 * (optimus_sweep_workspace_bytes).  optimus_sweep_eval enqueues, on one
 * stream, every template's build and the evaluation of this rank's shard of
 * its whole space, and writes template i's (lat, index) to d_best[2 i ..]
 * (asynchronous; decode with optimus_best_plan on optimus_sweep_ctx(i), a
 * borrowed context valid until optimus_sweep_free).  Comparing lats across
 * templates is the caller's choice: templates with different N_mb train
 * different global batches. */
typedef struct optimus_sweep optimus_sweep;
int optimus_sweep_workspace_bytes(const optimus_problem* pbs, int32_t count, size_t* bytes);
int optimus_sweep_load(const optimus_problem* pbs, int32_t count, void* d_workspace, size_t bytes, void* cuda_stream,
                       optimus_sweep** out);
int optimus_sweep_eval(optimus_sweep* sw, uint32_t rank, uint32_t world, int64_t* d_best, void* cuda_stream);
int optimus_sweep_ctx(optimus_sweep* sw, int32_t i, optimus_ctx** ctx);
void optimus_sweep_free(optimus_sweep* sw);

const char* optimus_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* OPTIMUS_H_ */
