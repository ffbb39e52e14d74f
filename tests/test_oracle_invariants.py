"""Invariant suite and independent-twin cross-check of the CPU oracle (-m "not gpu").

Invariants are the paper's constraints:
encoder kernels only in LLM bubbles of their own resource, never overlapping
each other, encoder stage order, encoder-LLM dependencies, iteration bounds,
refinement never increases Delta.  The twin (oracle/twin.py) is a separately
written implementation of the same readings.
"""
import random
from collections import defaultdict

import pytest

from workload import random_problem, toy_problem


def _problems(count=40, max_n=8):
    out = [toy_problem()]
    seed = 0
    while len(out) < count:
        out.append(random_problem(seed, max_n=max_n))
        seed += 1
    return out


def test_twin_matches_oracle_all_candidates(oracle_mod):
    from oracle import twin
    checked = moved = 0
    for pb in _problems(70):
        o = oracle_mod.Oracle(pb)
        if o.total > 2500:
            continue
        lats, best = twin.search(pb)
        lat, aux = o.eval(range(o.total), aux=True)
        assert lats == lat.tolist(), pb["name"]
        assert best == o.best()
        checked += o.total
        moved += int(((aux[:, 2] + aux[:, 3]) > 0).sum())
    assert checked > 1000 and moved > 100


def _check_trace(O, pb, tpl, tr, Ttot_cache):
    n = pb["n_mb"]
    L = pb["enc_llm_p2p_ns"]
    p2p = pb["enc_p2p_ns"]
    P, rt, m = tr["P"], tr["r_t"], tr["m"]
    T_end = tpl["T_end"]
    df, db = tr["df"], tr["db"]
    assert tr["lat"] == T_end + df + db >= T_end
    # Delta never increases over committed moves; at most n commits per phase (R13)
    for key, moves in (("deltas_f", tr["mf"]), ("deltas_b", tr["mb"])):
        d = tr[key]
        assert len(d) == moves + 1 and all(a >= b for a, b in zip(d, d[1:]))
        assert moves <= n
    # every in-bubble kernel lies in a free interval of its resource (R6: encoder
    # compute only in compute bubbles, encoder comm never in LLM TP comm)
    # and kernels of one device instance never overlap each other
    occ = defaultdict(list)
    for ph in ("fwd_place", "bwd_place"):
        for j, s, kind, a, b, ch in tr[ph]:
            q = (j // rt) * P + s
            ivs = tpl["comp_free"][q] if kind == 0 else tpl["comm_free"][q]
            assert any(lo <= a and b <= hi for lo, hi in ivs), (ph, j, s, kind, a, b)
            assert tpl["w"][q] <= a < b <= tpl["z"][q]
            occ[(j, s, kind)].append((a, b))
    for lst in occ.values():
        lst.sort()
        assert all(x[1] <= y[0] for x, y in zip(lst, lst[1:]))
    # encoder stage order inside each chain: fwd upstream->downstream,
    # bwd in reverse order
    chains = defaultdict(list)
    for ph in ("fwd_place", "bwd_place"):
        for j, s, kind, a, b, ch in tr[ph]:
            chains[(ph, j, ch)].append((s, a, b))
    for (ph, j, ch), ks in chains.items():
        for s in range(P - 1):
            up = [x for x in ks if x[0] == s]
            dn = [x for x in ks if x[0] == s + 1]
            if not up or not dn:
                continue
            if ph == "fwd_place":
                assert max(b for _, _, b in up) + p2p <= min(a for _, a, _ in dn)
            else:
                assert max(b for _, _, b in dn) + p2p <= min(a for _, a, _ in up)
    # forward encoder-LLM dependency (R20): EF_i + L <= F_i (LLM-relative)
    order = tr["order"]
    assert [v for v, _ in order] == sorted(v for v, _ in order)
    assert all(v + L <= f for (v, _), f in zip(order, tpl["F"]))
    # backward: each pipeline's gradients come back only after B_i + L
    preB = O.gpipe(tr["tau_b"], p2p, n)
    preF = O.gpipe(tr["tau_f"], p2p, n)
    for j in range(m):
        pos = [i for i, (_, jj) in enumerate(order) if jj == j]
        assert len(pos) == tr["N"][j]
        starts = sorted([T_end - (preB[P - 1][t] - db) for t in range(1, tr["cb_final"][j] + 1)] +
                        [T_end - x for x in tr["Qb"][j]])
        need = sorted(tpl["B"][i] + L for i in pos)
        assert all(s_ >= b_ for s_, b_ in zip(starts, need))
        # coarse work stays in the pre / post regions: fwd ends before the shifted
        # LLM starts on that stage, bwd starts after it ends
        a = j // rt
        for s in range(P):
            q = a * P + s
            if tr["c_final"][j]:
                assert preF[s][tr["c_final"][j]] <= tpl["w"][q] + df
            if tr["cb_final"][j]:
                assert tr["lat"] - preB[s][tr["cb_final"][j]] >= tpl["z"][q] + df


def test_schedule_invariants(oracle_mod):
    rng = random.Random(1)
    n_tr = 0
    for pb in _problems(60, max_n=12):
        o = oracle_mod.Oracle(pb)
        tpl = oracle_mod.template(pb)
        gs = list(range(o.total)) if o.total <= 40 else rng.sample(range(o.total), 40)
        for g in gs:
            _check_trace(oracle_mod, pb, tpl, o.trace(g), None)
            n_tr += 1
    assert n_tr > 1000


def test_tp_sibling_permutations_tie(oracle_mod):
    # R7: TP siblings (same PP row) see the same LLM timeline, so permuting their
    # microbatch counts cannot change lat; the argmin keeps the lowest index (R18)
    for pb in [toy_problem()] + [random_problem(s, max_n=8) for s in range(20)]:
        o = oracle_mod.Oracle(pb)
        if o.total > 3000:
            continue
        lat = o.eval(range(o.total)).tolist()
        pl = oracle_mod.plans(pb)["plans"]
        rt_of = {}
        for x in pl:
            if x["count"]:
                rt_of[x["first"]] = (x, pb["llm"]["tp"] // x["T"])
        groups = defaultdict(set)
        for first, (x, rt) in rt_of.items():
            for r in range(x["count"]):
                N = oracle_mod.unrank(pb["n_mb"], x["m"], r)
                key = (first, tuple(tuple(sorted(N[a * rt:(a + 1) * rt])) for a in range(x["m"] // rt)))
                groups[key].add(lat[first + r])
        assert all(len(v) == 1 for v in groups.values())
        best = min(range(len(lat)), key=lambda g: (lat[g], g))
        assert o.best() == (lat[best], best)


def test_oracle_deterministic_and_thread_invariant(oracle_mod):
    from workload import config_problem, sample_indices
    pb = config_problem(2)
    o = oracle_mod.Oracle(pb)
    idx = sample_indices(3, 300, o.total)
    a = o.eval(idx, threads=1)
    b = o.eval(idx, threads=4)
    assert a.tolist() == b.tolist()


def test_vectorised_sample_stream_matches_scalar():
    """bench.py --sample draws its indices with the vectorised splitmix64; it
    must be the scalar stream SURVEY §8(d) defines, index for index."""
    from workload import sample_indices, sample_indices_np
    for seed, count, total in [(7, 3000, 357426663480), (2**64 - 5, 40, 12345), (20241019, 1000, 2213201944)]:
        assert sample_indices_np(seed, count, total).tolist() == sample_indices(seed, count, total)
