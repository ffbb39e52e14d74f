"""ctypes front end of the CPU oracle (oracle/optimus_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; never by the product path
(paper_2408_03505_b200/).  Shares no code with it: the problem encoding below
(`encode`) is the oracle's own.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "optimus_oracle.cpp")
LIB = os.path.join(HERE, "liboptimus_oracle.so")
INF_MARK = -1


def build(force: bool = False) -> str:
    """Compile the oracle (plain g++ -O2, no CUDA)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-g", "-fPIC", "-shared", "-pthread", SRC, "-o", LIB + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        P64 = ctypes.POINTER(ctypes.c_int64)
        L.oracle_template.restype = ctypes.c_longlong
        L.oracle_template.argtypes = [P64, ctypes.c_longlong, P64, ctypes.c_longlong]
        L.oracle_llm_kernels.restype = ctypes.c_longlong
        L.oracle_llm_kernels.argtypes = [P64, ctypes.c_longlong, ctypes.c_int, P64, ctypes.c_longlong]
        L.oracle_simulate.restype = ctypes.c_longlong
        L.oracle_simulate.argtypes = [P64, ctypes.c_longlong, ctypes.POINTER(ctypes.c_int32), P64, ctypes.c_longlong]
        L.oracle_baseline.restype = ctypes.c_longlong
        L.oracle_baseline.argtypes = [P64, ctypes.c_longlong, ctypes.c_int, P64, ctypes.c_longlong]
        L.oracle_partition_dp.restype = ctypes.c_longlong
        L.oracle_partition_dp.argtypes = [P64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int32)]
        L.oracle_plans.restype = ctypes.c_longlong
        L.oracle_plans.argtypes = [P64, ctypes.c_longlong, P64, ctypes.c_longlong]
        L.oracle_unrank.restype = ctypes.c_int
        L.oracle_unrank.argtypes = [ctypes.c_longlong, ctypes.c_longlong, ctypes.c_ulonglong,
                                    ctypes.POINTER(ctypes.c_int32)]
        L.oracle_binom.restype = ctypes.c_ulonglong
        L.oracle_binom.argtypes = [ctypes.c_longlong, ctypes.c_longlong]
        L.oracle_min_shift.restype = ctypes.c_longlong
        L.oracle_min_shift.argtypes = [P64, ctypes.c_longlong, P64, ctypes.c_longlong, P64]
        L.oracle_gpipe.restype = ctypes.c_int
        L.oracle_gpipe.argtypes = [P64, ctypes.c_int, ctypes.c_longlong, ctypes.c_int, P64]
        L.oracle_first_fit.restype = ctypes.c_longlong
        L.oracle_first_fit.argtypes = [ctypes.c_int, P64, P64, P64, ctypes.c_longlong, P64,
                                       ctypes.POINTER(ctypes.c_int)]
        L.oracle_global_order.restype = ctypes.c_int
        L.oracle_global_order.argtypes = [P64, ctypes.POINTER(ctypes.c_int32), ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_int32)]
        L.oracle_row_chains.restype = ctypes.c_int
        L.oracle_row_chains.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P64]
        L.oracle_open.restype = ctypes.c_void_p
        L.oracle_open.argtypes = [P64, ctypes.c_longlong]
        L.oracle_close.argtypes = [ctypes.c_void_p]
        L.oracle_total.restype = ctypes.c_ulonglong
        L.oracle_total.argtypes = [ctypes.c_void_p]
        L.oracle_eval.restype = ctypes.c_int
        L.oracle_eval.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_longlong, P64, P64,
                                  ctypes.c_int]
        L.oracle_eval_range.restype = ctypes.c_int
        L.oracle_eval_range.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong, ctypes.c_ulonglong, P64, ctypes.c_int]
        L.oracle_best.restype = ctypes.c_int
        L.oracle_best.argtypes = [ctypes.c_void_p, ctypes.c_int, P64]
        L.oracle_trace.restype = ctypes.c_longlong
        L.oracle_trace.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong, ctypes.c_char_p, ctypes.c_longlong]
    return _lib


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def encode(prob: dict) -> np.ndarray:
    """Problem dict -> the oracle's flat int64 blob."""
    llm = prob["llm"]
    o = [0x4F50544D, 1, prob["n_gpu"], prob["gpu_mem_bytes"], prob["reserve_bytes"], prob["bytes_per_param"],
         llm["dp"], llm["pp"], llm["tp"], llm["v"], prob["llm_layers"], prob["n_mb"], prob["warmup_policy"],
         prob["dp_allgather_ns"], prob["dp_reducescatter_ns"], prob["pp_p2p_ns"], prob["enc_p2p_ns"],
         prob["enc_llm_p2p_ns"], prob["llm_params"], len(prob["tp_opts"]), *prob["tp_opts"]]

    def lst(x):
        o.append(len(x))
        for k, ns in x:
            o.extend([k, ns])

    lst(prob["llm_fwd_layer"])
    lst(prob["llm_bwd_layer"])
    o.append(len(prob["branches"]))
    for b in prob["branches"]:
        o.extend([b["layers"], b["params"]])
        for t in range(len(prob["tp_opts"])):
            lst(b["fwd"][t])
            lst(b["bwd"][t])
    return np.array(o, dtype=np.int64)


def template(prob: dict) -> dict:
    blob = encode(prob)
    cap = 1 << 24
    out = np.zeros(cap, dtype=np.int64)
    r = lib().oracle_template(_p64(blob), len(blob), _p64(out), cap)
    if r < 0:
        raise ValueError(f"oracle_template failed ({r})")
    o = out[:r].tolist()
    p, n = o[0], o[1]
    res = {"p": p, "n": n, "T_end": o[2], "span_def": o[3], "span": o[4]}
    i = 5
    res["W"] = o[i:i + p]; i += p
    res["Wdef"] = o[i:i + p]; i += p
    res["F"] = o[i:i + n]; i += n
    res["B"] = o[i:i + n]; i += n
    res["w"] = o[i:i + p]; i += p
    res["z"] = o[i:i + p]; i += p
    nc = o[i:i + p]; i += p
    nm = o[i:i + p]; i += p
    res["comp_free"], res["comm_free"] = [], []
    for s in range(p):
        c = o[i:i + 2 * nc[s]]; i += 2 * nc[s]
        m = o[i:i + 2 * nm[s]]; i += 2 * nm[s]
        res["comp_free"].append(list(zip(c[0::2], c[1::2])))
        res["comm_free"].append(list(zip(m[0::2], m[1::2])))
    return res


def llm_kernels(prob: dict, stage: int):
    blob = encode(prob)
    cap = 1 << 24
    out = np.zeros(cap, dtype=np.int64)
    r = lib().oracle_llm_kernels(_p64(blob), len(blob), stage, _p64(out), cap)
    if r < 0:
        raise ValueError(r)
    o = out[:r].tolist()
    nc, nm = o[0], o[1]
    comp = list(zip(o[2:2 + 2 * nc:2], o[3:3 + 2 * nc:2]))
    j = 2 + 2 * nc
    comm = list(zip(o[j:j + 2 * nm:2], o[j + 1:j + 2 * nm:2]))
    return comp, comm


def simulate(prob: dict, W: list[int]) -> dict:
    blob = encode(prob)
    p, n = prob["llm"]["pp"], prob["n_mb"]
    w = (ctypes.c_int32 * p)(*W)
    out = np.zeros(2 + 2 * n + p, dtype=np.int64)
    r = lib().oracle_simulate(_p64(blob), len(blob), w, _p64(out), len(out))
    if r < 0:
        raise ValueError(r)
    o = out.tolist()
    return {"ok": bool(o[0]), "span": o[1], "F": o[2:2 + n], "B": o[2 + n:2 + 2 * n], "last_end": o[2 + 2 * n:]}


def plans(prob: dict) -> dict:
    blob = encode(prob)
    out = np.zeros(4096, dtype=np.int64)
    r = lib().oracle_plans(_p64(blob), len(blob), _p64(out), len(out))
    if r < 0:
        raise ValueError(r)
    o = out[:r].tolist()
    pl = []
    for q in range(o[0]):
        P, T, dpe, m, kept, cnt, first = o[2 + 7 * q:9 + 7 * q]
        pl.append({"P": P, "T": T, "dp_enc": dpe, "m": m, "kept": bool(kept), "count": cnt, "first": first})
    return {"total": o[1], "plans": pl}


def baseline(prob: dict, kind: int) -> dict | None:
    """Megatron-LM baseline iteration time (kind 0 naive P:519, 1 balanced P:521 / App. B)."""
    blob = encode(prob)
    out = np.zeros(16 + 3 * 4096, dtype=np.int64)
    k = lib().oracle_baseline(_p64(blob), len(blob), kind, _p64(out), len(out))
    if k < 0:
        return None
    VP = int(out[1])
    return {"iter_ns": int(out[0]), "sizes": out[2:2 + VP].tolist(), "opF": out[2 + VP:2 + 2 * VP].tolist(),
            "opB": out[2 + 2 * VP:2 + 3 * VP].tolist()}


def partition_dp(t, VP: int):
    """App. B's DP: (F(L, VP), group sizes) or (-1, [])."""
    a = np.array(t, dtype=np.int64)
    sz = (ctypes.c_int32 * max(1, VP))()
    r = lib().oracle_partition_dp(_p64(a), len(a), VP, sz)
    return int(r), (list(sz)[:VP] if r >= 0 else [])


def unrank(n: int, m: int, rank: int) -> list[int]:
    out = (ctypes.c_int32 * m)()
    k = lib().oracle_unrank(n, m, rank, out)
    return list(out)[:k]


def binom(a: int, b: int) -> int:
    return lib().oracle_binom(a, b)


def min_shift(pre, fixed, deadlines):
    """min Delta >= 0: sortasc(pre - Delta U fixed) <= deadlines; None if none."""
    a = np.array(pre, dtype=np.int64)
    b = np.array(fixed, dtype=np.int64)
    d = np.array(deadlines, dtype=np.int64)
    assert len(d) == len(a) + len(b)
    r = lib().oracle_min_shift(_p64(a), len(a), _p64(b), len(b), _p64(d))
    return None if r == -1 else r


def gpipe(tau, p2p: int, c: int):
    t = np.array(tau, dtype=np.int64)
    out = np.zeros(len(tau) * (c + 1), dtype=np.int64)
    lib().oracle_gpipe(_p64(t), len(tau), p2p, c, _p64(out))
    return out.reshape(len(tau), c + 1).tolist()


def first_fit(ivs, lists, wst, p2p: int):
    """ivs[s] = (compute_free, comm_free) lists of (lo, hi); lists[s] = [(kind, ns)].

    Returns (EF or None, placements [(stage, kind, start, end)])."""
    P = len(lists)
    a = []
    for s in range(P):
        for r in range(2):
            a.append(len(ivs[s][r]))
            for lo, hi in ivs[s][r]:
                a.extend([lo, hi])
    b = []
    for s in range(P):
        b.append(len(lists[s]))
        for k, ns in lists[s]:
            b.extend([k, ns])
    A = np.array(a, dtype=np.int64)
    B = np.array(b, dtype=np.int64)
    W = np.array(wst, dtype=np.int64)
    out = np.zeros(4 * max(1, sum(len(x) for x in lists)), dtype=np.int64)
    npl = ctypes.c_int(0)
    ef = lib().oracle_first_fit(P, _p64(A), _p64(B), _p64(W), p2p, _p64(out), ctypes.byref(npl))
    pl = [tuple(out[4 * k:4 * k + 4].tolist()) for k in range(npl.value)]
    return (None if ef == -1 else ef), pl


def global_order(values_per_pipeline):
    """values_per_pipeline[j] = encoder forward finishes of pipeline j ->
    list of 1-based LLM microbatch positions per pipeline (R14)."""
    vals, pipe = [], []
    for j, vs in enumerate(values_per_pipeline):
        for x in vs:
            vals.append(x)
            pipe.append(j)
    V = np.array(vals, dtype=np.int64)
    Pp = (ctypes.c_int32 * len(pipe))(*pipe)
    own = (ctypes.c_int32 * len(pipe))()
    lib().oracle_global_order(_p64(V), Pp, len(pipe), len(values_per_pipeline), own)
    out = [[] for _ in values_per_pipeline]
    for i, j in enumerate(list(own)):
        out[j].append(i + 1)
    return out


class Oracle:
    """Search handle: template + plans built once, candidates evaluated literally."""

    def __init__(self, prob: dict):
        self.prob = prob
        self.blob = encode(prob)
        self.h = lib().oracle_open(_p64(self.blob), len(self.blob))
        if not self.h:
            raise ValueError("oracle_open failed (invalid problem)")
        self.total = lib().oracle_total(self.h)

    def close(self):
        if self.h:
            lib().oracle_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def eval(self, idx, threads: int = 1, aux: bool = False):
        idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
        lat = np.zeros(len(idx), dtype=np.int64)
        ax = np.zeros(4 * len(idx), dtype=np.int64) if aux else None
        rc = lib().oracle_eval(self.h, idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(idx), _p64(lat),
                               _p64(ax) if aux else None, threads)
        if rc:
            raise ValueError(f"oracle_eval rc={rc}")
        return (lat, ax.reshape(-1, 4)) if aux else lat

    def eval_range(self, begin: int, end: int, threads: int = 1):
        lat = np.zeros(end - begin, dtype=np.int64)
        rc = lib().oracle_eval_range(self.h, begin, end, _p64(lat), threads)
        if rc:
            raise ValueError(f"oracle_eval_range rc={rc}")
        return lat

    def best(self, threads: int = 1):
        b = np.zeros(2, dtype=np.int64)
        rc = lib().oracle_best(self.h, threads, _p64(b))
        if rc:
            raise ValueError(rc)
        return int(b[0]), int(b[1])

    def row_chains(self, e: int, a: int, kf: int, kmax: int):
        """Debug: successive chain EFs on fresh instances of row a of plan e
        (forward if kf < 0, else backward after kf forward chains)."""
        out = np.zeros(max(1, kmax), dtype=np.int64)
        k = lib().oracle_row_chains(self.h, e, a, kf, kmax, _p64(out))
        return None if k < 0 else out[:k].tolist()

    def trace(self, g: int) -> dict:
        cap = 1 << 26
        buf = ctypes.create_string_buffer(cap)
        r = lib().oracle_trace(self.h, g, buf, cap)
        if r < 0:
            raise ValueError(r)
        return json.loads(buf.value.decode())
