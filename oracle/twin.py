"""Independent Python twin of the oracle, for tiny problems — TEST INFRASTRUCTURE.

A second, separately written implementation of the same readings (SURVEY.md
§8(c) R1-R22) used to cross-check the C++ oracle where no paper
value pins the greedy trajectory.  It deliberately takes different routes:
  * LLM template: memoised recursion over the op dependency graph with cycle
    detection (the C++ oracle sweeps stages until no progress);
  * minimal shift: scan of the finitely many breakpoints x - d (the C++ oracle
    binary-searches the definition);
  * first fit: plain linear scan from the first interval;
  * compositions: itertools enumeration (the C++ oracle unranks by counting).
Pure Python, slow, small cases only.  Shares no code with the C++ oracle or
with the CUDA path.
"""
from __future__ import annotations

import itertools
import sys

INF = float("inf")


# ----------------------------------------------------------- LLM template
def _order(p, v, n, W):
    """Per-stage op order (Megatron interleaved 1F1B, R2): W fwd, pairs, rest."""
    nv = n * v

    def op(k, fwd):
        ch = (k % (p * v)) // p
        mb = (k // (p * v)) * p + k % p
        return ("F", ch, mb) if fwd else ("B", v - 1 - ch, mb)

    seq = [op(k, True) for k in range(W)]
    for i in range(nv - W):
        seq.append(op(W + i, True))
        seq.append(op(i, False))
    seq += [op(i, False) for i in range(nv - W, nv)]
    return seq


def _default_W(p, v, n):
    if v == 1:
        return [min(n, p - 1 - s) for s in range(p)]
    if n == p:
        return [n * v] * p
    return [min(n * v, 2 * (p - 1 - s) + (v - 1) * p) for s in range(p)]


def _sim(pb, W):
    """Return (ok, starts{(s,op)}, ends{(s,op)}, last_end[s]) via memoised recursion."""
    llm = pb["llm"]
    p, v, n = llm["pp"], llm["v"], pb["n_mb"]
    lc = pb["llm_layers"] // (p * v)
    df = lc * sum(ns for _, ns in pb["llm_fwd_layer"])
    db = lc * sum(ns for _, ns in pb["llm_bwd_layer"])
    orders = [_order(p, v, n, W[s]) for s in range(p)]
    index = {(s, op): q for s in range(p) for q, op in enumerate(orders[s])}
    end = {}
    visiting = set()
    sys.setrecursionlimit(100000)

    def dep(s, op):
        kind, c, i = op
        if kind == "F":
            if s > 0:
                return (s - 1, ("F", c, i))
            if c > 0:
                return (p - 1, ("F", c - 1, i))
            return None
        if s < p - 1:
            return (s + 1, ("B", c, i))
        if c < v - 1:
            return (0, ("B", c + 1, i))
        return (p - 1, ("F", v - 1, i))

    def finish(s, q):
        key = (s, q)
        if key in end:
            return end[key]
        if key in visiting:
            raise RecursionError("deadlock")
        visiting.add(key)
        op = orders[s][q]
        t = pb["dp_allgather_ns"]
        if q > 0:
            t = max(t, finish(s, q - 1))
        d = dep(s, op)
        if d is not None:
            ds, dop = d
            t = max(t, finish(ds, index[(ds, dop)]) + (pb["pp_p2p_ns"] if ds != s else 0))
        visiting.discard(key)
        end[key] = t + (df if op[0] == "F" else db)
        return end[key]

    try:
        last = [finish(s, len(orders[s]) - 1) for s in range(p)]
    except RecursionError:
        return False, None, None, None, None
    starts = {}
    for (s, q), e in end.items():
        op = orders[s][q]
        starts[(s, op)] = e - (df if op[0] == "F" else db)
    ends = {(s, orders[s][q]): e for (s, q), e in end.items()}
    return True, starts, ends, last, orders


def template(pb):
    llm = pb["llm"]
    p, v, n = llm["pp"], llm["v"], pb["n_mb"]
    Wd = _default_W(p, v, n)
    r = _sim(pb, Wd)
    span_def = max(r[3])
    W = list(Wd)
    if pb["warmup_policy"] == 1:
        for s in reversed(range(p)):
            for w in range(0, Wd[s] + 1):
                Wt = list(W)
                Wt[s] = w
                rr = _sim(pb, Wt)
                if rr[0] and max(rr[3]) == span_def:
                    W[s] = w
                    break
    ok, starts, ends, last, orders = _sim(pb, W)
    T_end = max(x + pb["dp_reducescatter_ns"] for x in last)
    F = [starts[(0, ("F", 0, i))] for i in range(n)]
    B = [ends[(0, ("B", 0, i))] for i in range(n)]
    lc = pb["llm_layers"] // (p * v)
    w, z, compf, commf = [], [], [], []
    for s in range(p):
        comp, comm = [], []
        for op in orders[s]:
            t = starts[(s, op)]
            lst = pb["llm_fwd_layer"] if op[0] == "F" else pb["llm_bwd_layer"]
            for _ in range(lc):
                for k, ns in lst:
                    (comp if k == 0 else comm).append((t, t + ns))
                    t += ns
        comp.sort()
        comm.sort()
        ws, zs = comp[0][0], max(e for _, e in comp)
        # compute-free: uncovered gaps of [ws, zs] by compute
        cf, cur = [], ws
        for a, b in comp:
            if a > cur:
                cf.append((cur, a))
            cur = max(cur, b)
        mf, cur = [], ws
        for a, b in comm:
            if b <= cur:
                continue
            if a >= zs:
                break
            if a > cur:
                mf.append((cur, a))
            cur = max(cur, b)
        if cur < zs:
            mf.append((cur, zs))
        w.append(ws)
        z.append(zs)
        compf.append(cf)
        commf.append(mf)
    return {"W": W, "Wdef": Wd, "T_end": T_end, "F": F, "B": B, "w": w, "z": z,
            "comp_free": compf, "comm_free": commf, "span": span_def}


# ------------------------------------------------------------- planner
def plan_list(pb):
    llm = pb["llm"]
    p, t, n = llm["pp"], llm["tp"], pb["n_mb"]
    dp_llm = pb["n_gpu"] // (p * t)
    phi_enc = sum(b["params"] for b in pb["branches"])
    out = []
    for P in [d for d in range(1, p + 1) if p % d == 0]:
        for T in [d for d in pb["tp_opts"] if t % d == 0]:
            dpe = pb["n_gpu"] // (P * T)
            mem = pb["bytes_per_param"] * (dpe * phi_enc + dp_llm * pb["llm_params"])
            if mem + pb["reserve_bytes"] * pb["n_gpu"] > pb["gpu_mem_bytes"] * pb["n_gpu"]:
                continue
            m = (p // P) * (t // T)
            if m > n:
                continue
            out.append((P, T, m))
    return out


def compositions(n, m):
    for cuts in itertools.combinations(range(1, n), m - 1):
        b = (0,) + cuts + (n,)
        yield [b[k + 1] - b[k] for k in range(m)]


def candidates(pb):
    for e, (P, T, m) in enumerate(plan_list(pb)):
        for N in compositions(pb["n_mb"], m):
            yield e, (P, T, m), N


# ------------------------------------------------------------- helpers
def stage_lists(pb, P, T):
    ti = pb["tp_opts"].index(T)
    fw, bm = [], []
    for s in range(P):
        layers = []
        for bi, b in enumerate(pb["branches"]):
            L = b["layers"]
            layers += [(bi, l) for l in range(s * L // P, (s + 1) * L // P)]
        f = [k for bi, l in layers for k in pb["branches"][bi]["fwd"][ti]]
        real_b = [k for bi, l in reversed(layers) for k in pb["branches"][bi]["bwd"][ti]]
        fw.append(f)
        bm.append(list(reversed(real_b)))
    return fw, bm


def fill(tau, p2p, c):
    """GPipe fill end times end[s][x] (R9)."""
    e = [[0] * (c + 1) for _ in tau]
    for x in range(1, c + 1):
        for s in range(len(tau)):
            st = e[s][x - 1] if s == 0 else max(e[s][x - 1], e[s - 1][x] + p2p)
            e[s][x] = st + tau[s]
    return e


def min_shift(pre, fixed, dl):
    """min D >= 0 with sorted(pre - D + fixed) <= dl elementwise, by breakpoint scan."""
    def ok(D):
        vals = sorted([x - D for x in pre] + list(fixed))
        return all(a <= b for a, b in zip(vals, dl))

    cands = sorted({0} | {x - d for x in pre for d in dl if x - d > 0})
    for D in cands:
        if ok(D):
            return D
    return INF


def chain(inst, lists, wst, p2p):
    """First fit of one microbatch chain; inst[s] = [compute_free, comm_free] lists of [lo, hi]."""
    prev = None
    for s, lst in enumerate(lists):
        ready = wst[s] if s == 0 else max(prev + p2p, wst[s])
        for kind, d in lst:
            for iv in inst[s][kind]:
                if iv[1] <= ready:
                    continue
                x = max(ready, iv[0])
                if x + d <= iv[1]:
                    iv[0] = x + d
                    ready = x + d
                    break
            else:
                return None
        prev = ready
    return ready


def _copy(inst):
    return [[[list(iv) for iv in r] for r in st] for st in inst]


# ------------------------------------------------------------ candidate
def evaluate(pb, tpl, P, T, m, N):
    llm = pb["llm"]
    p, t, n = llm["pp"], llm["tp"], pb["n_mb"]
    rt = t // T
    L = pb["enc_llm_p2p_ns"]
    Tend = tpl["T_end"]
    fw, bm = stage_lists(pb, P, T)
    tf = [sum(ns for _, ns in x) for x in fw]
    tb = [sum(ns for _, ns in x) for x in bm]
    pf = fill(tf, pb["enc_p2p_ns"], n)
    pbk = fill(tb, pb["enc_p2p_ns"], n)
    rows = [j // rt for j in range(m)]
    inst = [[[[list(iv) for iv in tpl["comp_free"][rows[j] * P + s]],
              [list(iv) for iv in tpl["comm_free"][rows[j] * P + s]]] for s in range(P)] for j in range(m)]

    def phase(c, Q, pre_tab, wv, lists, inst, depfn):
        moves = 0
        while True:
            devs = [max(pre_tab[s][c[j]] - wv[rows[j] * P + s] for s in range(P)) if c[j] else -INF
                    for j in range(m)]
            dev = max(devs)
            D = max(0, dev, depfn(c, Q))
            if D == 0 or sum(c) == 0:
                return D, moves
            js = devs.index(dev)
            trial = _copy(inst[js])
            ef = chain(trial, lists, [wv[rows[js] * P + s] for s in range(P)], pb["enc_p2p_ns"])
            if ef is None:
                return D, moves
            c2 = list(c)
            c2[js] -= 1
            Q2 = [list(q) for q in Q]
            Q2[js].append(ef)
            if depfn(c2, Q2) > D:
                return D, moves
            c[:] = c2
            Q[:] = Q2
            inst[js] = trial
            moves += 1

    G = [f - L for f in tpl["F"]]

    def dep_f(c, Q):
        pre = [pf[P - 1][x] for j in range(m) for x in range(1, c[j] + 1)]
        fixed = [q for j in range(m) for q in Q[j]]
        return min_shift(pre, fixed, G)

    c = list(N)
    Q = [[] for _ in range(m)]
    Df, mf = phase(c, Q, pf, tpl["w"], fw, inst, dep_f)
    ent = [(pf[P - 1][x] - Df, j, x - 1) for j in range(m) for x in range(1, c[j] + 1)]
    ent += [(q, j, c[j] + k) for j in range(m) for k, q in enumerate(Q[j])]
    ent.sort()
    S = [[i for i, e in enumerate(ent) if e[1] == j] for j in range(m)]
    Dl = [sorted(Tend - tpl["B"][i] - L for i in S[j]) for j in range(m)]
    wm = [Tend - zz for zz in tpl["z"]]
    minst = []
    for j in range(m):
        st = []
        for s in range(P):
            st.append([[[Tend - hi, Tend - lo] for lo, hi in reversed(inst[j][s][r]) if hi > lo] for r in range(2)])
        minst.append(st)

    def dep_b(c, Q):
        d = 0
        for j in range(m):
            d = max(d, min_shift([pbk[P - 1][x] for x in range(1, c[j] + 1)], Q[j], Dl[j]))
        return d

    cb = list(N)
    Qb = [[] for _ in range(m)]
    Db, mb = phase(cb, Qb, pbk, wm, bm, minst, dep_b)
    return {"lat": Tend + Df + Db, "df": Df, "db": Db, "mf": mf, "mb": mb}


def search(pb):
    """Alg. 1 over all candidates: list of lat in global index order and the best (lat, g)."""
    tpl = template(pb)
    lats = [evaluate(pb, tpl, P, T, m, N)["lat"] for _, (P, T, m), N in candidates(pb)]
    best = min(range(len(lats)), key=lambda g: (lats[g], g))
    return lats, (lats[best], best)
