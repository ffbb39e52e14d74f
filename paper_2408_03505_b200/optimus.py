"""Thin ctypes binding of liboptimus (include/optimus.h) — argument marshalling only.

Every step of the search runs in the library's sm_100a kernels.  PyTorch is
used only for device memory (the workspace and output tensors) and streams.
There is no CPU fallback: if the shared library or a CUDA device is missing,
every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboptimus.so")

OPTIMUS_OK = 0
ERRORS = {-1: "EINVAL", -2: "EINFEASIBLE", -3: "ECUDA", -4: "ENOSPACE", -5: "ERANGE"}

HEADER_SYMBOLS = [
    "optimus_workspace_bytes", "optimus_plan_only", "optimus_load_costs", "optimus_rebuild", "optimus_num_candidates",
    "optimus_get_plan", "optimus_eval_candidates", "optimus_eval_indices", "optimus_best_plan",
    "optimus_explain", "optimus_emit_schedule", "optimus_efficiency", "optimus_debug_template", "optimus_debug_plan_tables", "optimus_launch_count", "optimus_eval_instance", "optimus_baseline", "optimus_emit_p2p", "optimus_sweep_workspace_bytes", "optimus_sweep_load",
    "optimus_sweep_eval", "optimus_sweep_ctx", "optimus_sweep_free",
    "optimus_set_eval_mode",
    "optimus_set_timing",
    "optimus_last_timing", "optimus_eval_stats", "optimus_io_bytes", "optimus_free", "optimus_last_error",
]


class OptimusError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class optimus_plan(ctypes.Structure):
    _fields_ = [("dp", ctypes.c_int32), ("pp", ctypes.c_int32), ("tp", ctypes.c_int32), ("v", ctypes.c_int32)]


class optimus_seq(ctypes.Structure):
    _fields_ = [("kind", ctypes.POINTER(ctypes.c_uint8)), ("ns", ctypes.POINTER(ctypes.c_int64)),
                ("len", ctypes.c_int32)]


class optimus_problem(ctypes.Structure):
    _fields_ = [
        ("n_gpu", ctypes.c_int32), ("gpu_mem_bytes", ctypes.c_int64), ("reserve_bytes", ctypes.c_int64),
        ("bytes_per_param", ctypes.c_int32), ("llm", optimus_plan), ("llm_layers", ctypes.c_int32),
        ("n_mb", ctypes.c_int32), ("warmup_policy", ctypes.c_int32), ("llm_fwd_layer", optimus_seq),
        ("llm_bwd_layer", optimus_seq), ("dp_allgather_ns", ctypes.c_int64), ("dp_reducescatter_ns", ctypes.c_int64),
        ("pp_p2p_ns", ctypes.c_int64), ("enc_p2p_ns", ctypes.c_int64), ("enc_llm_p2p_ns", ctypes.c_int64),
        ("llm_params", ctypes.c_int64), ("n_branches", ctypes.c_int32),
        ("branch_layers", ctypes.POINTER(ctypes.c_int32)), ("branch_params", ctypes.POINTER(ctypes.c_int64)),
        ("n_tp_opts", ctypes.c_int32), ("tp_opts", ctypes.POINTER(ctypes.c_int32)),
        ("enc_fwd_layer", ctypes.POINTER(optimus_seq)), ("enc_bwd_layer", ctypes.POINTER(optimus_seq)),
    ]


class optimus_result(ctypes.Structure):
    _fields_ = [("lat_ns", ctypes.c_int64), ("index", ctypes.c_uint64), ("enc", optimus_plan), ("m", ctypes.c_int32)]


_lib = None


def lib():
    """Load liboptimus.so (built in-tree by __graft_entry__.build()).  Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        P = ctypes.POINTER
        sig = {
            "optimus_workspace_bytes": [P(optimus_problem), P(sz)],
            "optimus_load_costs": [P(optimus_problem), vp, sz, vp, P(vp)],
            "optimus_rebuild": [vp, vp],
            "optimus_plan_only": [P(optimus_problem), P(vp)],
            "optimus_num_candidates": [vp, P(ctypes.c_uint64), P(ctypes.c_int32)],
            "optimus_get_plan": [vp, ctypes.c_int32, P(optimus_plan), P(ctypes.c_int32), P(ctypes.c_uint64),
                                 P(ctypes.c_uint64)],
            "optimus_eval_candidates": [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32, vp, vp, vp],
            "optimus_eval_indices": [vp, vp, ctypes.c_uint64, vp, vp, vp],
            "optimus_best_plan": [vp, P(ctypes.c_int64), ctypes.c_int32, P(optimus_result), P(ctypes.c_int32)],
            "optimus_debug_template": [vp, P(ctypes.c_int64), sz, P(sz), vp],
            "optimus_explain": [vp, ctypes.c_uint64, P(ctypes.c_int64), sz, P(sz), vp],
            "optimus_emit_schedule": [vp, ctypes.c_uint64, P(ctypes.c_int64), sz, P(sz), vp],
            "optimus_efficiency": [vp, ctypes.c_uint64, P(ctypes.c_int64), vp],
            "optimus_debug_plan_tables": [vp, ctypes.c_int32, P(ctypes.c_int64), sz, P(sz), vp],
            "optimus_launch_count": [vp, P(ctypes.c_int32), P(ctypes.c_int32)],
            "optimus_eval_instance": [vp, P(ctypes.c_int32), P(ctypes.c_int32)],
            "optimus_baseline": [vp, ctypes.c_int32, P(ctypes.c_int64), sz, P(sz), vp],
            "optimus_emit_p2p": [vp, ctypes.c_uint64, P(ctypes.c_int64), sz, P(sz), vp],
            "optimus_sweep_workspace_bytes": [P(optimus_problem), ctypes.c_int32, P(sz)],
            "optimus_sweep_load": [P(optimus_problem), ctypes.c_int32, vp, sz, vp, P(vp)],
            "optimus_sweep_eval": [vp, ctypes.c_uint32, ctypes.c_uint32, vp, vp],
            "optimus_sweep_ctx": [vp, ctypes.c_int32, P(vp)],
            "optimus_set_timing": [vp, ctypes.c_int],
            "optimus_set_eval_mode": [vp, ctypes.c_int],
            "optimus_last_timing": [vp, P(ctypes.c_float), P(ctypes.c_float)],
            "optimus_eval_stats": [vp, P(ctypes.c_uint64), vp],
            "optimus_io_bytes": [vp, P(ctypes.c_uint64), P(ctypes.c_uint64)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.optimus_free.argtypes = [vp]
        L.optimus_free.restype = None
        L.optimus_last_error.argtypes = []
        L.optimus_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int):
    if rc != OPTIMUS_OK:
        raise OptimusError(rc, lib().optimus_last_error().decode())


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class Problem:
    """optimus_problem built from a problem dict (workload/ schema); owns its arrays."""

    def __init__(self, prob: dict):
        self._keep = []
        s = optimus_problem()
        llm = prob["llm"]
        s.n_gpu = prob["n_gpu"]
        s.gpu_mem_bytes = prob["gpu_mem_bytes"]
        s.reserve_bytes = prob["reserve_bytes"]
        s.bytes_per_param = prob["bytes_per_param"]
        s.llm = optimus_plan(llm["dp"], llm["pp"], llm["tp"], llm["v"])
        s.llm_layers = prob["llm_layers"]
        s.n_mb = prob["n_mb"]
        s.warmup_policy = prob["warmup_policy"]
        s.llm_fwd_layer = self._seq(prob["llm_fwd_layer"])
        s.llm_bwd_layer = self._seq(prob["llm_bwd_layer"])
        s.dp_allgather_ns = prob["dp_allgather_ns"]
        s.dp_reducescatter_ns = prob["dp_reducescatter_ns"]
        s.pp_p2p_ns = prob["pp_p2p_ns"]
        s.enc_p2p_ns = prob["enc_p2p_ns"]
        s.enc_llm_p2p_ns = prob["enc_llm_p2p_ns"]
        s.llm_params = prob["llm_params"]
        br = prob["branches"]
        s.n_branches = len(br)
        s.branch_layers = self._arr(ctypes.c_int32, [b["layers"] for b in br])
        s.branch_params = self._arr(ctypes.c_int64, [b["params"] for b in br])
        s.n_tp_opts = len(prob["tp_opts"])
        s.tp_opts = self._arr(ctypes.c_int32, prob["tp_opts"])
        fw = (optimus_seq * max(1, len(br) * len(prob["tp_opts"])))()
        bw = (optimus_seq * max(1, len(br) * len(prob["tp_opts"])))()
        for b, bb in enumerate(br):
            for ti in range(len(prob["tp_opts"])):
                fw[b * len(prob["tp_opts"]) + ti] = self._seq(bb["fwd"][ti])
                bw[b * len(prob["tp_opts"]) + ti] = self._seq(bb["bwd"][ti])
        self._keep += [fw, bw]
        s.enc_fwd_layer = ctypes.cast(fw, ctypes.POINTER(optimus_seq))
        s.enc_bwd_layer = ctypes.cast(bw, ctypes.POINTER(optimus_seq))
        self.s = s
        self.n_mb = prob["n_mb"]
        self.host_bytes = sum(ctypes.sizeof(x) for x in self._keep)

    def _arr(self, ct, vals):
        a = (ct * max(1, len(vals)))(*vals)
        self._keep.append(a)
        return ctypes.cast(a, ctypes.POINTER(ct))

    def _seq(self, lst):
        return optimus_seq(self._arr(ctypes.c_uint8, [k for k, _ in lst]), self._arr(ctypes.c_int64, [n for _, n in lst]),
                           len(lst))


def optimus_workspace_bytes(problem: Problem) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().optimus_workspace_bytes(ctypes.byref(problem.s), ctypes.byref(n)))
    return n.value


class Ctx:
    """A loaded search (optimus_ctx*).  Keeps the workspace tensor alive.

    workspace=None builds a host-only context (optimus_plan_only): plans,
    counts and best_plan decoding, no device work."""

    def __init__(self, problem: Problem, workspace, stream=None):
        self.problem = problem
        self.workspace = workspace
        h = ctypes.c_void_p()
        if workspace is None:
            _check(lib().optimus_plan_only(ctypes.byref(problem.s), ctypes.byref(h)))
        else:
            _check(lib().optimus_load_costs(ctypes.byref(problem.s), ctypes.c_void_p(workspace.data_ptr()),
                                            workspace.numel() * workspace.element_size(),
                                            ctypes.c_void_p(_stream(stream)), ctypes.byref(h)))
        self.h = h
        self.n_mb = problem.n_mb
        self._owned = True

    @classmethod
    def borrowed(cls, problem: Problem, workspace, h):
        """A context owned elsewhere (a Sweep's): never freed by this object."""
        c = cls.__new__(cls)
        c.problem, c.workspace, c.h, c.n_mb, c._owned = problem, workspace, h, problem.n_mb, False
        return c

    def rebuild(self, stream=None):
        _check(lib().optimus_rebuild(self.h, ctypes.c_void_p(_stream(stream))))

    def num_candidates(self):
        t, n = ctypes.c_uint64(), ctypes.c_int32()
        _check(lib().optimus_num_candidates(self.h, ctypes.byref(t), ctypes.byref(n)))
        return t.value, n.value

    def get_plan(self, i: int) -> dict:
        p, m, f, c = optimus_plan(), ctypes.c_int32(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().optimus_get_plan(self.h, i, ctypes.byref(p), ctypes.byref(m), ctypes.byref(f), ctypes.byref(c)))
        return {"dp": p.dp, "pp": p.pp, "tp": p.tp, "m": m.value, "first": f.value, "count": c.value}

    def eval_candidates(self, begin: int, end: int, best2, lat_out=None, rank: int = 0, world: int = 1,
                        block: int = 0, stream=None):
        _check(lib().optimus_eval_candidates(self.h, begin, end, rank, world, block, _ptr(lat_out), _ptr(best2),
                                             ctypes.c_void_p(_stream(stream))))

    def eval_indices(self, index, best2, lat_out=None, stream=None):
        _check(lib().optimus_eval_indices(self.h, _ptr(index), index.numel(), _ptr(lat_out), _ptr(best2),
                                          ctypes.c_void_p(_stream(stream))))

    def best_plan(self, best2_all_ranks) -> dict:
        a = np.ascontiguousarray(np.asarray(best2_all_ranks, dtype=np.int64).reshape(-1))
        r = optimus_result()
        counts = (ctypes.c_int32 * max(1, self.n_mb))()
        _check(lib().optimus_best_plan(self.h, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(a) // 2,
                                       ctypes.byref(r), counts))
        return {"lat_ns": r.lat_ns, "index": r.index, "enc": (r.enc.dp, r.enc.pp, r.enc.tp), "m": r.m,
                "counts": list(counts)[:r.m]}

    def explain(self, g: int, stream=None) -> dict:
        """The committed moves of candidate g (optimus_explain; NEXT-1)."""
        buf = (ctypes.c_int64 * (8 + 2 * 128 + 3 * 128))()
        n = ctypes.c_size_t()
        _check(lib().optimus_explain(self.h, ctypes.c_uint64(g), buf, len(buf), ctypes.byref(n),
                                     ctypes.c_void_p(_stream(stream))))
        v = list(buf[: n.value])
        nf, nb, m, nmb = v[3], v[4], v[6], v[7]
        return {"lat": v[0], "df": v[1], "db": v[2], "mf": nf, "mb": nb, "plan": v[5], "m": m,
                "moves_f": v[8:8 + nf], "moves_b": v[8 + nmb:8 + nmb + nb],
                "N": v[8 + 2 * nmb:8 + 2 * nmb + m], "c_final": v[8 + 2 * nmb + m:8 + 2 * nmb + 2 * m],
                "cb_final": v[8 + 2 * nmb + 2 * m:8 + 2 * nmb + 3 * m]}

    def emit_p2p(self, g: int, stream=None) -> list:
        """Encoder-LLM P2P send/recv pairs of candidate g (optimus_emit_p2p; NEXT-4): records
        [dir, microbatch, pipeline, src stage, src slot, dst stage, dst slot, send ns, arrive ns]."""
        cap = 18 * 128
        buf = (ctypes.c_int64 * cap)()
        n = ctypes.c_size_t()
        _check(lib().optimus_emit_p2p(self.h, ctypes.c_uint64(g), buf, cap, ctypes.byref(n),
                                      ctypes.c_void_p(_stream(stream))))
        v = list(buf)[:9 * n.value]
        return [v[9 * k:9 * k + 9] for k in range(n.value)]

    def efficiency(self, g: int, stream=None) -> dict:
        """Eff_fine / Eff_coarse of candidate g as exact work sums (optimus_efficiency; NEXT-1)."""
        out = (ctypes.c_int64 * 3)()
        _check(lib().optimus_efficiency(self.h, ctypes.c_uint64(g), out, ctypes.c_void_p(_stream(stream))))
        return {"in_bubble_fine": out[0], "in_bubble_coarse": out[1], "total": out[2]}

    def emit_schedule(self, g: int, cap_records: int = 1 << 20, stream=None) -> dict:
        """In-bubble kernel placements of candidate g (optimus_emit_schedule; NEXT-1)."""
        import numpy as np
        out = np.zeros(6 * cap_records, dtype=np.int64)
        nr = (ctypes.c_size_t * 2)()
        _check(lib().optimus_emit_schedule(self.h, ctypes.c_uint64(g), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                           out.size, nr, ctypes.c_void_p(_stream(stream))))
        rec = out[: 6 * (nr[0] + nr[1])].reshape(-1, 6).tolist()
        return {"fwd_place": rec[: nr[0]], "bwd_place": rec[nr[0]:]}

    def debug_template(self, stream=None) -> dict:
        cap = 1 << 24
        out = np.zeros(cap, dtype=np.int64)
        n = ctypes.c_size_t(0)
        _check(lib().optimus_debug_template(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap,
                                            ctypes.byref(n), ctypes.c_void_p(_stream(stream))))
        o = out[:n.value].tolist()
        p, nm = o[0], o[1]
        r = {"T_end": o[2], "span_def": o[3]}
        i = 4
        r["W"] = o[i:i + p]; i += p
        r["F"] = o[i:i + nm]; i += nm
        r["B"] = o[i:i + nm]; i += nm
        r["w"] = o[i:i + p]; i += p
        r["z"] = o[i:i + p]; i += p
        nc = o[i:i + p]; i += p
        nmm = o[i:i + p]; i += p
        r["comp_free"], r["comm_free"] = [], []
        for s in range(p):
            a = o[i:i + 2 * nc[s]]; i += 2 * nc[s]
            b = o[i:i + 2 * nmm[s]]; i += 2 * nmm[s]
            r["comp_free"].append(list(zip(a[0::2], a[1::2])))
            r["comm_free"].append(list(zip(b[0::2], b[1::2])))
        return r

    def debug_plan_tables(self, i: int, stream=None) -> dict | None:
        cap = 1 << 24
        out = np.zeros(cap, dtype=np.int64)
        n = ctypes.c_size_t(0)
        _check(lib().optimus_debug_plan_tables(self.h, i, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap,
                                               ctypes.byref(n), ctypes.c_void_p(_stream(stream))))
        if n.value == 0:
            return None
        o = out[:n.value]
        rp, kmax = int(o[0]), int(o[1])
        j = 2
        lenF = o[j:j + rp].tolist(); j += rp
        inbF = o[j:j + rp * kmax].reshape(rp, kmax).tolist(); j += rp * kmax
        lenB = o[j:j + rp * (kmax + 1)].reshape(rp, kmax + 1).tolist(); j += rp * (kmax + 1)
        inbB = o[j:j + rp * (kmax + 1) * kmax].reshape(rp, kmax + 1, kmax).tolist(); j += rp * (kmax + 1) * kmax
        rest = o[j:]
        P = len(rest) // (2 * (self.n_mb + 1))
        preF = rest[:P * (self.n_mb + 1)].reshape(P, -1).tolist()
        preB = rest[P * (self.n_mb + 1):].reshape(P, -1).tolist()
        return {"rp": rp, "kmax": kmax, "lenF": lenF, "INB_F": [inbF[a][:lenF[a]] for a in range(rp)],
                "lenB": lenB, "INB_B": [[inbB[a][k][:lenB[a][k]] for k in range(kmax + 1)] for a in range(rp)],
                "PRE_F": preF, "PRE_B": preB}

    def launch_count(self):
        b, e = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().optimus_launch_count(self.h, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def baseline(self, kind: int, stream=None) -> dict:
        """Megatron-LM baseline iteration time: kind 0 naive, 1 balanced (App. B)."""
        n = ctypes.c_size_t()
        cap = 2 + 3 * 4096
        buf = (ctypes.c_int64 * cap)()
        _check(lib().optimus_baseline(self.h, kind, buf, cap, ctypes.byref(n), ctypes.c_void_p(_stream(stream))))
        VP = buf[1]
        o = list(buf)[:n.value]
        return {"iter_ns": o[0], "sizes": o[2:2 + VP], "opF": o[2 + VP:2 + 2 * VP], "opB": o[2 + 2 * VP:2 + 3 * VP]}

    def eval_instance(self):
        """(K2 mode 1 instance 0-5, its persistent grid)."""
        i, g = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().optimus_eval_instance(self.h, ctypes.byref(i), ctypes.byref(g)))
        return i.value, g.value

    def set_eval_mode(self, mode: int):
        """1 = one candidate per thread (default), 0 = one candidate per warp."""
        _check(lib().optimus_set_eval_mode(self.h, mode))

    def set_timing(self, on: bool = True):
        _check(lib().optimus_set_timing(self.h, 1 if on else 0))

    def last_timing(self):
        """(build_ms, k2_ms) of the most recent build / K2 launch (events on the launch stream)."""
        b, e = ctypes.c_float(), ctypes.c_float()
        _check(lib().optimus_last_timing(self.h, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def eval_stats(self, stream=None) -> dict:
        a = (ctypes.c_uint64 * 10)()
        _check(lib().optimus_eval_stats(self.h, a, ctypes.c_void_p(_stream(stream))))
        keys = ("candidates", "ops", "iters_f", "attempts_f", "iters_b", "attempts_b", "fast", "general", "claims",
                "unranks")
        return dict(zip(keys, list(a)))

    def io_bytes(self):
        h, d = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().optimus_io_bytes(self.h, ctypes.byref(h), ctypes.byref(d)))
        return h.value, d.value

    def free(self):
        if getattr(self, "h", None):
            if getattr(self, "_owned", True):
                lib().optimus_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def optimus_load_costs(prob: dict, stream=None, device="cuda") -> Ctx:
    """Allocate the workspace with torch and load `prob` (a workload/ problem dict)."""
    import torch
    P = Problem(prob)
    nbytes = optimus_workspace_bytes(P)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return Ctx(P, ws, stream)


class Sweep:
    """NEXT-3: several LLM templates searched in one call (optimus_sweep_*)."""

    def __init__(self, probs: list, stream=None, device="cuda"):
        import torch
        self.problems = [Problem(p) for p in probs]
        arr = (optimus_problem * len(probs))(*[p.s for p in self.problems])
        self._arr = arr
        nb = ctypes.c_size_t()
        _check(lib().optimus_sweep_workspace_bytes(arr, len(probs), ctypes.byref(nb)))
        self.workspace = torch.empty(nb.value, dtype=torch.uint8, device=device)
        h = ctypes.c_void_p()
        _check(lib().optimus_sweep_load(arr, len(probs), ctypes.c_void_p(self.workspace.data_ptr()), nb.value,
                                        ctypes.c_void_p(_stream(stream)), ctypes.byref(h)))
        self.h = h
        self.ctxs = []
        for i in range(len(probs)):
            c = ctypes.c_void_p()
            _check(lib().optimus_sweep_ctx(self.h, i, ctypes.byref(c)))
            self.ctxs.append(Ctx.borrowed(self.problems[i], self.workspace, c))

    def eval(self, best, rank: int = 0, world: int = 1, stream=None):
        """best: int64 device tensor [count, 2] <- each template's (lat, index) over this rank's shard."""
        _check(lib().optimus_sweep_eval(self.h, rank, world, ctypes.c_void_p(best.data_ptr()),
                                        ctypes.c_void_p(_stream(stream))))

    def free(self):
        if self.h:
            for c in self.ctxs:
                c.h = None
            lib().optimus_sweep_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def optimus_plan_only(prob: dict) -> Ctx:
    """Host-only context: plans, candidate counts, best_plan decoding."""
    return Ctx(Problem(prob), None)


def search(prob: dict, stream=None) -> dict:
    """One full search on the current device: load + eval of every candidate + best."""
    import torch
    ctx = optimus_load_costs(prob, stream)
    total, _ = ctx.num_candidates()
    best2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, best2, stream=stream)
    b = best2.cpu().numpy()
    return ctx.best_plan(b)
