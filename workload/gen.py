"""Synthetic Optimus search inputs, integer nanoseconds.

Cost model (the paper gives shapes, not
durations):
  * compute kernels: model FLOPs / (989 TFLOP/s x 35%)      (P:508 peak)
    -> ViT-22B TP8 forward layer 1.44 ms (paper: ~1.4 ms)
  * LayerNorm / activation: HBM-bound at 3 TB/s
  * TP all-gather / reduce-scatter (Megatron-SP): 10 us +
    tok*w*2 B * (T-1)/T / 300 GB/s   -> GPT-175B TP8: 303.6 us (paper ~300 us)
  * backward compute = 2 x forward FLOPs, comm kernels equal in both directions
  * microbatch size 2, LLM sequence 2048
  * DP all-gather / reduce-scatter = Table 1's 0.167 s / 0.458 s
    scaled by LLM params per GPU relative to GPT-175B on PP x TP = 96
  * every rounding is exact-rational, half-up, minimum 1 ns.

Kernel kinds: 0 = compute, 1 = TP communication.
Per-layer forward order (R3): LN AG QKV ATTN PROJ RS LN AG FC1 ACT FC2 RS
(8 compute-only kernels at TP=1); backward = reversed order.

Nothing in this file simulates a pipeline or schedules anything.
"""
from __future__ import annotations

from fractions import Fraction

MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """Counter-based splitmix64 (Steele et al.); returns the mixed value of x."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def sample_indices(seed: int, count: int, total: int) -> list[int]:
    """Seeded sample g_i = splitmix64(seed + i) mod total."""
    return [splitmix64((seed + i) & MASK64) % total for i in range(count)]


def sample_indices_np(seed: int, count: int, total: int):
    """The same stream as sample_indices, vectorised (numpy uint64 wraps mod 2^64)."""
    import numpy as np
    z = np.arange(count, dtype=np.uint64) + np.uint64(seed & MASK64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return z % np.uint64(total)


def _rhu(x: Fraction) -> int:
    """Round half-up to an integer, minimum 1 (durations are >= 1 ns, R1)."""
    v = (x.numerator * 2 + x.denominator) // (2 * x.denominator)
    return max(1, int(v))


# ---------------------------------------------------------------- model shapes
# (width, depth, mlp, heads, head_dim)
VIT_L = (1024, 24, 4096, 16, 64)
VIT_3B = (2304, 48, 9216, 18, 128)       # App. A
VIT_11B = (4096, 48, 16384, 32, 128)     # App. A "ViT-10B"
VIT_22B = (6144, 48, 24576, 48, 128)     # App. A
AUDIO = (1280, 32, 5120, 20, 64)
GPT_1_3B = (2048, 24, 8192, 16, 128)
GPT_13B = (5120, 40, 20480, 40, 128)
GPT_70B = (8192, 80, 32768, 64, 128)     # LLAMA-70B-class width/depth
GPT_175B = (12288, 96, 49152, 96, 128)   # App. A

MB_SIZE = 2
LLM_SEQ = 2048
EFF_FLOP_PER_NS = Fraction(989 * 10**12 * 35, 100 * 10**9)   # 346150 FLOP/ns
HBM_B_PER_NS = Fraction(3 * 10**12, 10**9)                    # 3000 B/ns
TP_B_PER_NS = Fraction(300 * 10**9, 10**9)                    # 300 B/ns
TP_ALPHA_NS = 10_000
T_AG_175B_NS = 167_000_000
T_RS_175B_NS = 458_000_000
BYTES_PER_PARAM = 6                # k = 6, bf16 params + fp32 grads
GPU_MEM = 80 * 10**9               # 80 GB Hopper
RESERVE = GPU_MEM * 40 // 100      # activation reserve, 40%


def params(shape) -> int:
    """12 w^2 L-style parameter count: L (4 w^2 + 2 w f)."""
    w, L, f, _, _ = shape
    return L * (4 * w * w + 2 * w * f)


def layer_kernels(shape, seq: int, tp: int):
    """One transformer layer pass at TP degree `tp` -> (fwd list, bwd list).

    Lists of (kind, ns).  `seq` is tokens per sample; MB_SIZE samples/microbatch.
    """
    w, _, f, h, hd = shape
    assert w == h * hd
    tok = MB_SIZE * seq
    T = tp

    def flop(x):
        return Fraction(x, T) / EFF_FLOP_PER_NS

    def hbm(nbytes):
        return Fraction(nbytes, T) / HBM_B_PER_NS

    qkv = flop(2 * tok * w * 3 * w)
    attn = flop(4 * MB_SIZE * seq * seq * w)
    proj = flop(2 * tok * w * w)
    fc1 = flop(2 * tok * w * f)
    fc2 = flop(2 * tok * f * w)
    ln = hbm(2 * tok * w * 2)
    act = hbm(2 * tok * f * 2)
    comm = None
    if T > 1:
        comm = TP_ALPHA_NS + Fraction(tok * w * 2 * (T - 1), T) / TP_B_PER_NS
    names = ["LN", "AG", "QKV", "ATTN", "PROJ", "RS", "LN", "AG", "FC1", "ACT", "FC2", "RS"]
    fwd_t = {"LN": ln, "QKV": qkv, "ATTN": attn, "PROJ": proj, "FC1": fc1, "ACT": act, "FC2": fc2}
    fwd, bwd = [], []
    for nm in names:
        if nm in ("AG", "RS"):
            if T == 1:
                continue
            fwd.append((1, _rhu(comm)))
        else:
            fwd.append((0, _rhu(fwd_t[nm])))
    for nm in reversed(names):
        if nm in ("AG", "RS"):
            if T == 1:
                continue
            bwd.append((1, _rhu(comm)))
        else:
            bwd.append((0, _rhu(2 * fwd_t[nm])))
    return fwd, bwd


def divisors(x: int) -> list[int]:
    return [d for d in range(1, x + 1) if x % d == 0]


# ------------------------------------------------------------------- configs
CONFIGS = {
    1: dict(name="c1_vitl_gpt1.3b_8gpu", n_gpu=8, llm=(2, 2, 2, 2), n_mb=4,
            llm_model=GPT_1_3B, encoders=[(VIT_L, 2048)]),
    2: dict(name="c2_vit3b_gpt13b_128gpu", n_gpu=128, llm=(4, 4, 8, 2), n_mb=16,
            llm_model=GPT_13B, encoders=[(VIT_3B, 3072)]),
    3: dict(name="c3_vit11b_gpt70b_1024gpu", n_gpu=1024, llm=(16, 8, 8, 2), n_mb=32,
            llm_model=GPT_70B, encoders=[(VIT_11B, 3072)]),
    4: dict(name="c4_vit22b_gpt175b_3072gpu", n_gpu=3072, llm=(32, 12, 8, 2), n_mb=24,
            llm_model=GPT_175B, encoders=[(VIT_22B, 3072)]),
    5: dict(name="c5_dualenc_vit22b_audio_gpt175b_3072gpu", n_gpu=3072, llm=(48, 8, 8, 2),
            n_mb=16, llm_model=GPT_175B, encoders=[(VIT_22B, 3072), (AUDIO, 1500)]),
}


def config_problem(cfg: int, n_mb: int | None = None) -> dict:
    """Problem dict for BASELINE.json configs[cfg-1] (Appendix B of SURVEY.md)."""
    c = CONFIGS[cfg]
    dp, pp, tp, v = c["llm"]
    n = c["n_mb"] if n_mb is None else n_mb
    lm = c["llm_model"]
    llm_fwd, llm_bwd = layer_kernels(lm, LLM_SEQ, tp)
    phi_llm = params(lm)
    rho = Fraction(phi_llm * 96, pp * tp * params(GPT_175B))
    tp_opts = divisors(tp)
    branches = []
    for shape, seq in c["encoders"]:
        fw, bw = [], []
        for T in tp_opts:
            f_, b_ = layer_kernels(shape, seq, T)
            fw.append(f_)
            bw.append(b_)
        branches.append({"layers": shape[1], "params": params(shape), "fwd": fw, "bwd": bw})
    return {
        "name": c["name"] + ("" if n_mb is None else f"_n{n}"),
        "n_gpu": c["n_gpu"],
        "gpu_mem_bytes": GPU_MEM,
        "reserve_bytes": RESERVE,
        "bytes_per_param": BYTES_PER_PARAM,
        "llm": {"dp": dp, "pp": pp, "tp": tp, "v": v},
        "llm_layers": lm[1],
        "n_mb": n,
        "warmup_policy": 1,
        "llm_fwd_layer": llm_fwd,
        "llm_bwd_layer": llm_bwd,
        "dp_allgather_ns": _rhu(T_AG_175B_NS * rho),
        "dp_reducescatter_ns": _rhu(T_RS_175B_NS * rho),
        "pp_p2p_ns": 0,
        "enc_p2p_ns": 0,
        "enc_llm_p2p_ns": 0,
        "llm_params": phi_llm,
        "tp_opts": tp_opts,
        "branches": branches,
    }


def toy_problem() -> dict:
    """SURVEY.md Appendix C golden toy (regression target, not an independent pin)."""
    C, M = 0, 1
    fwd = [(M, 20), (C, 60), (M, 20), (C, 2), (M, 20), (C, 120), (M, 20), (C, 2)]
    bwd = [(M, 20), (C, 240), (M, 20), (C, 2), (M, 20), (C, 120), (M, 20), (C, 2)]
    e_f2 = [(M, 10), (C, 20), (M, 10), (C, 1), (M, 10), (C, 40), (M, 10), (C, 1)]
    e_b2 = [(M, 10), (C, 57), (M, 10), (C, 1), (M, 10), (C, 28), (M, 10), (C, 1)]
    e_f1 = [(C, 20), (C, 1), (C, 40), (C, 1)]
    e_b1 = [(C, 57), (C, 1), (C, 28), (C, 1)]
    return {
        "name": "toy_appendix_c",
        "n_gpu": 8,
        "gpu_mem_bytes": 10**15,
        "reserve_bytes": 0,
        "bytes_per_param": 6,
        "llm": {"dp": 1, "pp": 4, "tp": 2, "v": 2},
        "llm_layers": 16,
        "n_mb": 8,
        "warmup_policy": 1,
        "llm_fwd_layer": fwd,
        "llm_bwd_layer": bwd,
        "dp_allgather_ns": 300,
        "dp_reducescatter_ns": 700,
        "pp_p2p_ns": 0,
        "enc_p2p_ns": 0,
        "enc_llm_p2p_ns": 0,
        "llm_params": 1000,
        "tp_opts": [1, 2],
        "branches": [{"layers": 4, "params": 100, "fwd": [e_f1, e_f2], "bwd": [e_b1, e_b2]}],
    }


class _Rng:
    """Counter-based stream over splitmix64."""

    def __init__(self, seed: int):
        self.seed = seed & MASK64
        self.i = 0

    def next(self) -> int:
        self.i += 1
        return splitmix64((self.seed * 0x100000001B3 + self.i) & MASK64)

    def randint(self, lo: int, hi: int) -> int:  # inclusive
        return lo + self.next() % (hi - lo + 1)

    def choice(self, xs):
        return xs[self.next() % len(xs)]


def _rand_layer(rng: _Rng, T: int, scale: int, n_comp: int):
    """Random layer list: compute kernels with TP comm kernels interleaved (T>1)."""
    out = []
    for k in range(n_comp):
        if T > 1 and (k % 2 == 0 or rng.randint(0, 3) == 0):
            out.append((1, rng.randint(max(1, scale // 8), scale // 2)))
        out.append((0, rng.randint(1, scale)))
    return out


def random_problem(seed: int, max_p: int = 4, max_t: int = 4, max_n: int = 12,
                   p2p: bool = True, jitter: bool = True) -> dict:
    """Seeded small stress problem (parity + invariant suites, S:629 ranges).

    Random LLM plan, random kernel lists, nonzero P2P latencies and optional
    x U[0.9, 1.1] per-kernel jitter.  Memory is never binding.
    """
    rng = _Rng(seed)
    p = rng.choice([d for d in (1, 2, 3, 4, 6, 8) if d <= max_p])
    t = rng.choice([d for d in (1, 2, 4, 8) if d <= max_t])
    v = rng.choice([1, 2, 2, 3]) if p > 1 else rng.choice([1, 2])
    k = rng.randint(1, max(1, max_n // p))
    n = p * k
    lc = rng.randint(1, 3)
    layers = p * v * lc
    scale = rng.randint(20, 200)
    llm_fwd = _rand_layer(rng, t, scale, rng.randint(2, 4))
    llm_bwd = _rand_layer(rng, t, 2 * scale, rng.randint(2, 4))
    tp_opts = divisors(t)
    nb = rng.choice([1, 1, 2])
    branches = []
    for _ in range(nb):
        L = rng.randint(1, 6)
        escale = rng.randint(5, scale)
        nc = rng.randint(1, 3)
        fw, bw = [], []
        for T in tp_opts:
            fw.append(_rand_layer(rng, T, max(2, escale // T), nc))
            bw.append(_rand_layer(rng, T, max(2, 2 * escale // T), nc))
        branches.append({"layers": L, "params": 1000 * L, "fwd": fw, "bwd": bw})
    prob = {
        "name": f"stress_{seed}",
        "n_gpu": p * t * 2,
        "gpu_mem_bytes": 10**15,
        "reserve_bytes": 0,
        "bytes_per_param": 6,
        "llm": {"dp": 2, "pp": p, "tp": t, "v": v},
        "llm_layers": layers,
        "n_mb": n,
        "warmup_policy": 1,
        "llm_fwd_layer": llm_fwd,
        "llm_bwd_layer": llm_bwd,
        "dp_allgather_ns": rng.randint(0, 40 * scale),
        "dp_reducescatter_ns": rng.randint(0, 60 * scale),
        "pp_p2p_ns": rng.randint(0, scale // 4) if p2p else 0,
        "enc_p2p_ns": rng.randint(0, scale // 4) if p2p else 0,
        "enc_llm_p2p_ns": rng.randint(0, scale // 4) if p2p else 0,
        "llm_params": 10**6,
        "tp_opts": tp_opts,
        "branches": branches,
    }
    if jitter:
        _apply_jitter(prob, seed)
    return prob


def _apply_jitter(prob: dict, seed: int) -> None:
    """Seeded x U[0.9, 1.1] per-kernel jitter, exact integer rounding."""
    rng = _Rng(seed ^ 0x5EED)

    def jit(lst):
        return [(k, _rhu(Fraction(ns * (9000 + rng.randint(0, 2000)), 10000))) for k, ns in lst]

    prob["llm_fwd_layer"] = jit(prob["llm_fwd_layer"])
    prob["llm_bwd_layer"] = jit(prob["llm_bwd_layer"])
    for b in prob["branches"]:
        b["fwd"] = [jit(x) for x in b["fwd"]]
        b["bwd"] = [jit(x) for x in b["bwd"]]


def problem_summary(prob: dict) -> dict:
    """Shape facts used in configs/logs (no method arithmetic)."""
    llm = prob["llm"]
    return {
        "name": prob["name"],
        "n_gpu": prob["n_gpu"],
        "llm_plan": [llm["dp"], llm["pp"], llm["tp"], llm["v"]],
        "n_mb": prob["n_mb"],
        "branches": [b["layers"] for b in prob["branches"]],
    }
