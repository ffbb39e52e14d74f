// baseline.cu — the Megatron-LM baselines the paper's headline speedups are
// measured against (Table 5):
//   naive the multimodal encoders run "in the first pipeline
//            stage": every encoder layer (all branches, at the LLM's TP)
//            joins virtual stage 0 in front of its LLM layers;
//   balanced (App. B) the layer sequence (encoder, then
//            LLM) is cut into V x PP contiguous virtual stages by the DP
//            F(l, m) = min_{j<l} max(F(j, m-1), sum_{i=j+1..l} t_i), t_i a
//            layer's forward + backward time; single encoder only.
// Each runs Megatron's interleaved 1F1B (default warm-up, R2) with the
// virtual stages' summed layer times, from T_ag, plus T_rs (R3).  Readings
// (DESIGN.md R-DP): t_i is the profiled kernel time, virtual stages are
// non-empty, DP ties go to the smallest cut j.
//
// k_base_dp:  one block: layer times, the DP (balanced) or the fixed
//             placement (naive), per-(stage, chunk) op times.
// k_base_sim: one warp, lane = LLM stage: ASAP list schedule of every
//             stage's ops in Megatron order, a round per warp barrier.
#include "optimus_dev.cuh"

namespace optimus {
namespace {

constexpr int kBaseThreads = 256;

__device__ int64_t list_ns(const Cfg& c, int id) {
  int64_t t = 0;
  for (int i = c.loff[id]; i < c.loff[id + 1]; ++i) t += c.lns[i];
  return t;
}

// layer i of the sequence (encoder layers of every branch in order, then the
// LLM's): forward / backward time
__device__ void layer_ns(const Cfg& c, int i, int64_t& f, int64_t& b) {
  for (int br = 0; br < c.nb; ++br) {
    if (i < c.blayers[br]) {
      f = list_ns(c, enc_list_id(br, c.ntp - 1, c.ntp, 0));  // the encoder at the LLM's TP (inside its stage)
      b = list_ns(c, enc_list_id(br, c.ntp - 1, c.ntp, 1));
      return;
    }
    i -= c.blayers[br];
  }
  f = list_ns(c, 0);
  b = list_ns(c, 1);
}

// ws: S[L+1], F[VP+1][L+1] (int64), arg[VP+1][L+1] (int32), sizes[VP], opF[VP], opB[VP] (out + 2 ...)
__global__ void __launch_bounds__(kBaseThreads) k_base_dp(Cfg c, int kind, int L, int Le, int64_t* S, int64_t* F,
                                                          int32_t* arg, int64_t* out) {
  const int p = c.p, v = c.v, VP = p * v, tid = threadIdx.x;
  int64_t* sizes = out + 2;
  int64_t* opF = out + 2 + VP;
  int64_t* opB = out + 2 + 2 * VP;
  if (kind == 0) {
    for (int k = tid; k < VP; k += blockDim.x) sizes[k] = c.lc + (k == 0 ? Le : 0);
  } else {
    if (tid == 0) {  // prefix sums of t_i = forward + backward
      S[0] = 0;
      for (int i = 0; i < L; ++i) {
        int64_t f, b;
        layer_ns(c, i, f, b);
        S[i + 1] = S[i] + f + b;
      }
    }
    __syncthreads();
    const int W = L + 1;
    for (int l = tid; l <= L; l += blockDim.x) F[1 * W + l] = l >= 1 ? S[l] : kInf;
    __syncthreads();
    for (int m = 2; m <= VP; ++m) {
      for (int l = tid; l <= L; l += blockDim.x) {
        int64_t best = kInf;
        int bj = -1;
        for (int j = m - 1; j < l; ++j) {  // ascending j, strict <: ties to the smallest j
          const int64_t x = max(F[(m - 1) * W + j], S[l] - S[j]);
          if (x < best) { best = x; bj = j; }
        }
        F[m * W + l] = best;
        arg[m * W + l] = bj;
      }
      __syncthreads();
    }
    if (tid == 0) {
      int l = L;
      for (int m = VP; m >= 2; --m) {
        const int j = arg[m * W + l];
        sizes[m - 1] = l - j;
        l = j;
      }
      sizes[0] = l;
    }
  }
  __syncthreads();
  for (int k = tid; k < VP; k += blockDim.x) {  // op times of virtual stage k = chunk k / p of stage k % p
    int i0 = 0;
    for (int q = 0; q < k; ++q) i0 += (int)sizes[q];
    int64_t tf = 0, tb = 0;
    for (int i = i0; i < i0 + (int)sizes[k]; ++i) {
      int64_t f, b;
      layer_ns(c, i, f, b);
      tf += f;
      tb += b;
    }
    const int s = k % p, ch = k / p;
    opF[s * v + ch] = tf;
    opB[s * v + ch] = tb;
  }
  if (tid == 0) out[1] = VP;
}

__device__ __forceinline__ int64_t ld_cv(const int64_t* a) { return __ldcv(const_cast<int64_t*>(a)); }

// done[((s * 2 + fwd) * v + chunk) * n + mb] = op end, -1 before
__global__ void k_base_sim(Cfg c, int64_t* done, int64_t* out) {
  const int p = c.p, v = c.v, n = c.n, VP = p * v, lane = threadIdx.x;
  const int64_t* opF = out + 2 + VP;
  const int64_t* opB = out + 2 + 2 * VP;
  for (int i = lane; i < p * 2 * v * n; i += 32) __stcg(&done[i], (int64_t)-1);
  __syncwarp();
  const int s = lane;
  const int nv = n * v, nops = 2 * nv;
  // Megatron's default warm-up (R2)
  const int W = s >= p ? 0 : v == 1 ? min(n, p - 1 - s) : n == p ? nv : min(nv, 2 * (p - 1 - s) + (v - 1) * p);
  int pos = s < p ? 0 : nops;
  int64_t free_at = 0;
  for (;;) {
    bool prog = false;
    while (pos < nops) {
      const OpRef op = op_at(p, v, n, W, pos);
      int ds = -1, df = 0, dc = 0;  // dependency (R2)
      if (op.fwd) {
        if (s > 0) { ds = s - 1; df = 1; dc = op.chunk; }
        else if (op.chunk > 0) { ds = p - 1; df = 1; dc = op.chunk - 1; }
      } else {
        if (s < p - 1) { ds = s + 1; df = 0; dc = op.chunk; }
        else if (op.chunk < v - 1) { ds = 0; df = 0; dc = op.chunk + 1; }
        else { ds = p - 1; df = 1; dc = v - 1; }
      }
      int64_t t = max(free_at, c.T_ag);  // every op from T_ag (R3)
      if (ds >= 0) {
        const int64_t e = ld_cv(&done[((ds * 2 + df) * v + dc) * n + op.mb]);
        if (e < 0) break;
        t = max(t, e + (ds != s ? c.pp_p2p : 0));
      }
      free_at = t + (op.fwd ? opF[s * v + op.chunk] : opB[s * v + op.chunk]);
      __stcg(&done[((s * 2 + op.fwd) * v + op.chunk) * n + op.mb], free_at);
      ++pos;
      prog = true;
    }
    __syncwarp();  // this round's ends, visible to the next round
    if (__all_sync(0xffffffffu, pos >= nops)) break;
    if (!__any_sync(0xffffffffu, prog)) {  // no stage can move: deadlock (not expected, R2)
      if (lane == 0) out[0] = -1;
      return;
    }
  }
  int64_t span = free_at;
  for (int o = 16; o > 0; o >>= 1) span = max(span, (int64_t)__shfl_xor_sync(0xffffffffu, span, o));
  if (lane == 0) out[0] = span + c.T_rs;
}

}  // namespace

// bytes of the workspace region launch_baseline uses (L layers, VP virtual stages)
size_t baseline_ws_bytes(int L, int VP, int p, int v, int n) {
  return (size_t)(L + 1) * 8 + (size_t)(VP + 1) * (L + 1) * 12 + (size_t)p * 2 * v * n * 8 + (size_t)(3 * VP + 8) * 8 + 64;
}

cudaError_t launch_baseline(const Cfg& c, int kind, int L, int Le, void* ws, int64_t** d_out, cudaStream_t st) {
  const int VP = c.p * c.v;
  char* w = (char*)ws;
  int64_t* S = (int64_t*)w;
  w += (size_t)(L + 1) * 8;
  int64_t* F = (int64_t*)w;
  w += (size_t)(VP + 1) * (L + 1) * 8;
  int32_t* arg = (int32_t*)w;
  w += ((size_t)(VP + 1) * (L + 1) * 4 + 7) / 8 * 8;
  int64_t* done = (int64_t*)w;
  w += (size_t)c.p * 2 * c.v * c.n * 8;
  int64_t* out = (int64_t*)w;
  *d_out = out;
  k_base_dp<<<1, kBaseThreads, 0, st>>>(c, kind, L, Le, S, F, arg, out);
  k_base_sim<<<1, 32, 0, st>>>(c, done, out);
  return cudaGetLastError();
}

}  // namespace optimus
