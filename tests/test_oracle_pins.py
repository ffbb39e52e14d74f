"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the passage it pins (P:line = PAPER.md, S:line = SPEC.md).
None of these re-types the oracle's own formula: they use printed values,
closed forms from a different derivation, brute force, or an independent
implementation.
"""
import itertools
import json
import os
import random

import pytest

from workload import config_problem, random_problem, toy_problem

HERE = os.path.dirname(os.path.abspath(__file__))


def uniform_problem(p, v, n, tf, tb, t=1, T_ag=0, T_rs=0, pp_p2p=0, policy=1, enc=None, lc=1):
    """LLM whose chunk ops are one compute kernel each (uniform ops)."""
    enc = enc or {"layers": 1, "params": 1, "fwd": [[(0, 1)]] * len([d for d in range(1, t + 1) if t % d == 0]),
                  "bwd": [[(0, 1)]] * len([d for d in range(1, t + 1) if t % d == 0])}
    return {
        "name": "uniform", "n_gpu": p * t, "gpu_mem_bytes": 10**15, "reserve_bytes": 0, "bytes_per_param": 6,
        "llm": {"dp": 1, "pp": p, "tp": t, "v": v}, "llm_layers": p * v * lc, "n_mb": n, "warmup_policy": policy,
        "llm_fwd_layer": [(0, tf)], "llm_bwd_layer": [(0, tb)],
        "dp_allgather_ns": T_ag, "dp_reducescatter_ns": T_rs, "pp_p2p_ns": pp_p2p, "enc_p2p_ns": 0,
        "enc_llm_p2p_ns": 0, "llm_params": 10, "tp_opts": [d for d in range(1, t + 1) if t % d == 0],
        "branches": [enc],
    }


# ------------------------------------------------------------- a1 plans
def _plan_problem(p, t, n_gpu, n_mb=None, v=1):
    pb = uniform_problem(p, v, n_mb or p, 3, 5, t=t)
    pb["n_gpu"] = n_gpu
    pb["llm"]["dp"] = n_gpu // (p * t)
    return pb


def test_plan_count_28_for_pp64_tp8(oracle_mod):
    # "no more than 28 encoder parallel plans ... up to 7 options for PP_enc and 4 for TP_enc"
    pl = oracle_mod.plans(_plan_problem(64, 8, 512))["plans"]
    assert len(pl) == 28
    assert len({x["P"] for x in pl}) == 7 and len({x["T"] for x in pl}) == 4


def test_plan_count_small(oracle_mod):
    # PP_llm=4, TP_llm=2, n_gpu=8 -> 6 plans; PP=TP=1 -> 1 plan
    pl = oracle_mod.plans(_plan_problem(4, 2, 8))["plans"]
    assert [(x["P"], x["T"]) for x in pl] == [(1, 1), (1, 2), (2, 1), (2, 2), (4, 1), (4, 2)]
    assert [x["dp_enc"] for x in pl] == [8, 4, 4, 2, 2, 1]
    assert len(oracle_mod.plans(_plan_problem(1, 1, 4))["plans"]) == 1


@pytest.mark.parametrize("p,t", [(6, 4), (12, 8), (8, 2), (9, 1), (16, 8)])
def test_plans_divisor_bruteforce(oracle_mod, p, t):
    # PP_enc | PP_llm and TP_enc | TP_llm; m = DP_enc / DP_llm
    n_gpu = p * t * 3
    pl = oracle_mod.plans(_plan_problem(p, t, n_gpu))["plans"]
    brute = [(P, T) for P in range(1, p + 1) for T in range(1, t + 1) if p % P == 0 and t % T == 0]
    assert [(x["P"], x["T"]) for x in pl] == brute
    for x in pl:
        assert x["m"] * (n_gpu // (p * t)) == x["dp_enc"]


def test_memory_prune_worked_example(oracle_mod):
    # §4.5 via SPEC's worked example S:127: k=6, n_gpu=512, DP_llm=8,
    # phi_llm=175e9, DP_enc=32, phi_enc=22e9 -> MEM_model ~= 24.66 GB.
    def kept_with(reserve):
        pb = _plan_problem(8, 8, 512)
        pb["llm_params"] = 175 * 10**9
        pb["branches"][0]["params"] = 22 * 10**9
        pb["gpu_mem_bytes"] = 80 * 10**9
        pb["reserve_bytes"] = reserve
        pl = [x for x in oracle_mod.plans(pb)["plans"] if x["dp_enc"] == 32]
        assert pl and all(x["dp_enc"] == 32 for x in pl)
        return pl[0]["kept"]

    cap = 80 * 10**9
    assert kept_with(cap - 24_665_000_000)          # MEM_model <= 24.665 GB
    assert not kept_with(cap - 24_655_000_000)      # MEM_model >  24.655 GB


def test_memory_prune_config4_keeps_20(oracle_mod):
    # config 4 keeps the 20 plans with PP_enc*TP_enc >= 4; totals [V]
    r = oracle_mod.plans(config_problem(4))
    kept = [(x["P"], x["T"]) for x in r["plans"] if x["kept"]]
    assert len(kept) == 20 and all(P * T >= 4 for P, T in kept)
    assert r["total"] == 5_845_247


@pytest.mark.parametrize("cfg,total", [(1, 8), (2, 20_703), (3, 912_152_435), (4, 5_845_247)])
def test_candidate_totals(oracle_mod, cfg, total):
    assert oracle_mod.plans(config_problem(cfg))["total"] == total


# ------------------------------------------------------- a2 compositions
def test_partitions_n8_m2_paper(oracle_mod):
    # "8 microbatches and m=2 ... a total of 7 possible partitioning options,
    # such as [1, 7], [2, 6], ..., [7, 1]"
    assert oracle_mod.binom(7, 1) == 7
    assert [oracle_mod.unrank(8, 2, r) for r in range(7)] == [[k, 8 - k] for k in range(1, 8)]


def test_partitions_count_and_order(oracle_mod):
    # n=6, m=3 -> 10; lexicographic order == itertools over cut positions
    assert oracle_mod.binom(5, 2) == 10
    for n in range(1, 11):
        for m in range(1, n + 1):
            brute = []
            for cuts in itertools.combinations(range(1, n), m - 1):
                b = (0,) + cuts + (n,)
                brute.append([b[k + 1] - b[k] for k in range(m)])
            assert brute == sorted(brute)
            got = [oracle_mod.unrank(n, m, r) for r in range(oracle_mod.binom(n - 1, m - 1))]
            assert got == brute


# ------------------------------------------------------------ a3 template
@pytest.mark.parametrize("policy", [0, 1])
def test_interleaved_makespan_closed_form(oracle_mod, policy):
    # Interleaved 1F1B (Megatron-LM): with uniform chunk ops and no P2P
    # latency the pipeline takes (n v + p - 1)(t_f + t_b); v = 1 gives classic 1F1B.
    rng = random.Random(7)
    for _ in range(60):
        p = rng.choice([1, 2, 3, 4, 6, 8])
        v = rng.choice([1, 2, 3, 4])
        n = p * rng.randint(1, 4)
        tf, tb = rng.randint(1, 50), rng.randint(1, 100)
        t = oracle_mod.template(uniform_problem(p, v, n, tf, tb, policy=policy))
        assert t["span"] == (n * v + p - 1) * (tf + tb)


def test_classic_1f1b_bubble_fraction(oracle_mod):
    # device-0 idle fraction (p-1)/(n+p-1) with balanced stages, v=1, t_f=t_b.
    # Compute-free time on stage 0 inside [w, z] plus the cool-down after z equals
    # (p-1)(t_f+t_b) out of the span (n+p-1)(t_f+t_b).
    for p in (2, 3, 4, 8):
        for n in (p, 2 * p, 5 * p):
            tf = tb = 7
            t = oracle_mod.template(uniform_problem(p, 1, n, tf, tb))
            idle = sum(b - a for a, b in t["comp_free"][0]) + (t["span"] - t["z"][0]) + t["w"][0]
            assert idle * (n + p - 1) == (p - 1) * t["span"]


def test_fig9_warmup_adjustment(oracle_mod):
    # P:444 (Fig. 9, p=4, v=2, n=8): "deferring forward data dependency points for the
    # last four microbatches (F5 through F8) is feasible without ... adverse effects
    # on the overall pipeline latency"
    t1 = oracle_mod.template(uniform_problem(4, 2, 8, 10, 20, policy=1))
    t0 = oracle_mod.template(uniform_problem(4, 2, 8, 10, 20, policy=0))
    assert t1["span"] == t0["span"]
    assert t1["F"][:4] == t0["F"][:4]
    assert all(a > b for a, b in zip(t1["F"][4:], t0["F"][4:]))
    assert t1["W"] == [7, 6, 5, 4]


def test_warmup_closed_form_and_monotone(oracle_mod):
    # R5 with pp_p2p = 0 and uniform ops: W_s = min(nv, (v-1)p + (p-1-s)) [SURVEY App. A];
    # the adjustment never moves an F earlier and keeps the makespan.
    rng = random.Random(11)
    for _ in range(40):
        p = rng.choice([2, 3, 4, 6, 8])
        v = rng.choice([1, 2, 3])
        n = p * rng.randint(1, 4)
        tf, tb = rng.randint(1, 30), rng.randint(1, 60)
        t1 = oracle_mod.template(uniform_problem(p, v, n, tf, tb, policy=1))
        t0 = oracle_mod.template(uniform_problem(p, v, n, tf, tb, policy=0))
        if v > 1:
            assert t1["W"] == [min(n * v, (v - 1) * p + (p - 1 - s)) for s in range(p)]
        assert t1["span"] == t0["span"]
        assert all(a >= b for a, b in zip(t1["F"], t0["F"]))


def test_dependency_points_invariants(oracle_mod):
    # F, B ascending; B_i >= F_i (causality)
    for seed in range(30):
        t = oracle_mod.template(random_problem(seed))
        assert t["F"] == sorted(t["F"]) and t["B"] == sorted(t["B"])
        assert all(b >= f for f, b in zip(t["F"], t["B"]))


def test_interval_conservation(oracle_mod):
    # S:225 per-device conservation: LLM busy + free = [w, z] on each resource,
    # and no free interval intersects an LLM kernel of its own resource (R6).
    for pb in [toy_problem()] + [random_problem(s) for s in range(12)]:
        t = oracle_mod.template(pb)
        for s in range(pb["llm"]["pp"]):
            comp, comm = oracle_mod.llm_kernels(pb, s)
            w, z = t["w"][s], t["z"][s]
            busy = sorted(comp)
            assert busy[0][0] == w and max(e for _, e in busy) == z
            assert sum(b - a for a, b in busy) + sum(b - a for a, b in t["comp_free"][s]) == z - w
            cm = sum(max(0, min(b, z) - max(a, w)) for a, b in comm)
            assert cm + sum(b - a for a, b in t["comm_free"][s]) == z - w
            for lo, hi in t["comp_free"][s]:
                assert all(b <= lo or a >= hi for a, b in comp)
            for lo, hi in t["comm_free"][s]:
                assert all(b <= lo or a >= hi for a, b in comm)


def test_template_matches_twin(oracle_mod):
    from oracle import twin
    for pb in [toy_problem()] + [random_problem(s) for s in range(10)]:
        a, b = oracle_mod.template(pb), twin.template(pb)
        for k in ("W", "T_end", "F", "B", "w", "z"):
            assert a[k] == b[k], k
        assert [list(map(tuple, x)) for x in a["comp_free"]] == [list(map(tuple, x)) for x in b["comp_free"]]
        assert [list(map(tuple, x)) for x in a["comm_free"]] == [list(map(tuple, x)) for x in b["comm_free"]]


# -------------------------------------------------------- a4 coarse fill
def test_gpipe_uniform_closed_form(oracle_mod):
    # R9 with uniform tau: end(s, x) = (s + x) tau + s * enc_p2p
    for P in (1, 2, 3, 5):
        for tau in (1, 7):
            for p2p in (0, 3):
                e = oracle_mod.gpipe([tau] * P, p2p, 6)
                for s in range(P):
                    for x in range(1, 7):
                        assert e[s][x] == (s + x) * tau + s * p2p


# ------------------------------------------------------- a5 first fit
def test_first_fit_paper_example(oracle_mod):
    # one 300 us bubble holds three 100 us compute kernels; bubble fully packed
    ef, pl = oracle_mod.first_fit([([(0, 300_000)], [])], [[(0, 100_000)] * 3], [0], 0)
    assert ef == 300_000 and [(a, b) for _, _, a, b in pl] == [(0, 100_000), (100_000, 200_000), (200_000, 300_000)]
    ef, _ = oracle_mod.first_fit([([(0, 300_000)], [])], [[(0, 100_000)] * 4], [0], 0)
    assert ef is None


def _brute_chain(ivs, lists, wst, p2p):
    """Exhaustive DFS: every kernel in any interval of its resource at its earliest
    feasible point; returns the minimal chain completion (fresh intervals, one chain)."""
    best = [None]

    def rec(s, k, ready, used):
        if s == len(lists):
            if best[0] is None or ready < best[0]:
                best[0] = ready
            return
        if k == len(lists[s]):
            nxt = max(ready + p2p, wst[s + 1]) if s + 1 < len(lists) else ready
            rec(s + 1, 0, nxt, used)
            return
        kind, d = lists[s][k]
        for q, (lo, hi) in enumerate(ivs[s][kind]):
            lo2 = used.get((s, kind, q), lo)
            x = max(ready, lo2)
            if x + d <= hi:
                u2 = dict(used)
                u2[(s, kind, q)] = x + d
                rec(s, k + 1, x + d, u2)

    rec(0, 0, wst[0], {})
    return best[0]


def test_first_fit_equals_bruteforce(oracle_mod):
    rng = random.Random(3)
    n_ok = 0
    for _ in range(400):
        P = rng.randint(1, 3)
        ivs, lists, wst = [], [], []
        for s in range(P):
            res = []
            for r in range(2):
                t, lst = rng.randint(0, 5), []
                for _ in range(rng.randint(0, 4)):
                    a = t + rng.randint(0, 6)
                    b = a + rng.randint(1, 12)
                    lst.append((a, b))
                    t = b
                res.append(lst)
            ivs.append(res)
            lists.append([(rng.randint(0, 1), rng.randint(1, 6)) for _ in range(rng.randint(0, 4))])
            wst.append(rng.randint(0, 6))
        p2p = rng.randint(0, 2)
        ef, _ = oracle_mod.first_fit(ivs, lists, wst, p2p)
        assert ef == _brute_chain(ivs, lists, wst, p2p)
        n_ok += ef is not None
    assert n_ok > 50


# --------------------------------------------------- Δ (R10, R15) closed form
def test_min_shift_closed_form(oracle_mod):
    # R10's closed form (a different derivation from the oracle's binary search):
    # need_i = i - #{q <= d_i}; INF if need_i > |pre|; else
    # dep = max(0, max_{need_i > 0} sorted(pre)[need_i] - d_i)
    rng = random.Random(5)
    for _ in range(3000):
        n = rng.randint(1, 8)
        k = rng.randint(0, n)
        pre = sorted(rng.randint(0, 60) for _ in range(n - k))
        fixed = [rng.randint(-10, 60) for _ in range(k)]
        dl = sorted(rng.randint(-5, 70) for _ in range(n))
        exp = 0
        for i in range(1, n + 1):
            need = i - sum(q <= dl[i - 1] for q in fixed)
            if need > len(pre):
                exp = None
                break
            if need > 0:
                exp = max(exp, pre[need - 1] - dl[i - 1])
        assert oracle_mod.min_shift(pre, fixed, dl) == exp


# ------------------------------------------------------- a7 ordering
def test_global_order_fig10(oracle_mod):
    # "activations from encoder pipeline 1 are designated as the 1st, 3rd, 7th,
    # and 8th microbatches, while activations from encoder pipeline 2 are used as the
    # 2nd, 4th, 5th, and 6th microbatches"
    assert oracle_mod.global_order([[10, 30, 70, 80], [20, 40, 50, 60]]) == [[1, 3, 7, 8], [2, 4, 5, 6]]
    # ties: lower pipeline first (R14)
    assert oracle_mod.global_order([[5, 9], [5, 7]]) == [[1, 4], [2, 3]]


# --------------------------------------------------------- special case
def test_special_case_closed_form(oracle_mod):
    # p=v=t=1, P=T=1, no P2P, compute-only kernels: m=1, no interleaved bubbles, so
    # the loop never moves a chain and lat has the closed form of SURVEY §8(c)
    rng = random.Random(9)
    for _ in range(120):
        n = rng.randint(1, 8)
        tf, tb = rng.randint(1, 40), rng.randint(1, 80)
        T_ag, T_rs = rng.randint(0, 300), rng.randint(0, 300)
        L = rng.randint(1, 4)
        ef_, eb_ = rng.randint(1, 30), rng.randint(1, 60)
        enc = {"layers": L, "params": 1, "fwd": [[(0, ef_)]], "bwd": [[(0, eb_)]]}
        pb = uniform_problem(1, 1, n, tf, tb, T_ag=T_ag, T_rs=T_rs, enc=enc)
        o = oracle_mod.Oracle(pb)
        assert o.total == 1
        lat = int(o.eval([0])[0])
        tauf, taub = L * ef_, L * eb_
        T_end = T_ag + n * (tf + tb) + T_rs
        df = max([0, n * tauf - T_ag] + [i * tauf - T_ag - (i - 1) * (tf + tb) for i in range(1, n + 1)])
        db = max([0, n * taub - T_rs] + [k * taub - T_rs - (k - 1) * (tf + tb) for k in range(1, n + 1)])
        assert lat == T_end + df + db


def test_zero_layer_encoder(oracle_mod):
    # R21 / S:268: an encoder with no kernels leaves every lat at T_end; best g = 0
    pb = toy_problem()
    pb["branches"][0]["fwd"] = [[], []]
    pb["branches"][0]["bwd"] = [[], []]
    o = oracle_mod.Oracle(pb)
    lat = o.eval(range(o.total))
    assert set(lat.tolist()) == {oracle_mod.template(pb)["T_end"]}
    assert o.best() == (int(lat[0]), 0)


# ------------------------------------------------------------- golden toy
def test_appendix_c_golden_toy(oracle_mod):
    gold = json.load(open(os.path.join(HERE, "golden", "toy_appendix_c.json")))
    pb = toy_problem()
    t = oracle_mod.template(pb)
    g = gold["template"]
    assert t["W"] == g["W"] and t["T_end"] == g["T_end"] and t["F"] == g["F"] and t["B"] == g["B"]
    assert [list(x) for x in zip(t["w"], t["z"])] == g["wz"]
    assert all(len(x) == g["n_comp_free"] for x in t["comp_free"])
    assert all(len(x) == g["n_comm_free"] for x in t["comm_free"])
    pl = oracle_mod.plans(pb)
    assert pl["total"] == gold["total"]
    assert [[x["P"], x["T"], x["m"], x["count"]] for x in pl["plans"]] == gold["plans"]
    o = oracle_mod.Oracle(pb)
    lat, aux = o.eval(range(o.total), aux=True)
    for row in gold["plan_2_2"]:
        gi = row["g"]
        assert [lat[gi]] + aux[gi].tolist() == [row["lat"], row["df"], row["db"], row["mf"], row["mb"]]
    for row in gold["plan_min"]:
        first = [x for x in pl["plans"] if [x["P"], x["T"]] == row["plan"]][0]
        seg = lat[first["first"]:first["first"] + first["count"]]
        assert int(seg.min()) == row["lat"] and first["first"] + int(seg.argmin()) == row["g"]
        assert oracle_mod.unrank(8, first["m"], row["g"] - first["first"]) == row["N"]
        if "df" in row:
            assert aux[row["g"]][0] == row["df"]
        if "db" in row:
            assert aux[row["g"]][1] == row["db"]
    assert list(o.best()) == gold["best"]


# ------------------------------------------------- R11 findCritical order
def _moves(trace, key):
    """Moving pipeline of each committed move, in move order (trace records
    are [pipeline, stage, comm, start, end, move])."""
    seq = {}
    for r in trace[key]:
        seq.setdefault(r[5], r[0])
    return [seq[k] for k in sorted(seq)]


def test_findcritical_order_p389(oracle_mod):
    """P:387-389 (Fig. 'move_enc', partition [3, 5] of N_mb = 8 over two
    encoder pipelines): "encoder pipeline 2's forward computation
    (microbatch 8 forward) is initially on the critical path ... After
    successfully scheduling that microbatch forward to later bubbles, encoder
    pipeline 1 assumes the critical path position."  Pipeline 1 runs on the
    first LLM stages and pipeline 2 on the later ones (R7).  On this
    fixture the oracle's first two committed forward moves are pipeline 2 then
    pipeline 1, which R11 (critical = largest end(s, c_j) - w of the stage's
    own LLM stage) produces; the reading "largest absolute end time" cannot:
    after the first move pipeline 2 still holds 4 coarse microbatches against
    pipeline 1's 3, so its absolute GPipe end is later and it would stay
    critical."""
    prob = random_problem(2606, max_p=4, max_t=2, max_n=8, p2p=False, jitter=False)
    assert prob["llm"]["pp"] == 4 and prob["n_mb"] == 8
    pl = oracle_mod.plans(prob)["plans"]
    e = next(i for i, q in enumerate(pl) if q["m"] == 2 and q["P"] == 2 and q["count"])
    g = pl[e]["first"] + 2  # lexicographic: [1,7], [2,6], [3,5]
    o = oracle_mod.Oracle(prob)
    t = o.trace(g)
    assert t["N"] == [3, 5]
    mv = _moves(t, "fwd_place")
    assert mv[:2] == [1, 0], mv  # 0-based: encoder pipeline 2, then encoder pipeline 1
    # the absolute-end reading: GPipe end of the last stage, counts [3, 4]
    ends = oracle_mod.gpipe(t["tau_f"], prob["enc_p2p_ns"], 8)[-1]
    assert ends[4] > ends[3]


# ------------------------------------------------- R8 stage split
def _chain_stage_kernels(trace, key):
    """{(move, stage): [(comm, duration, start, end), ...]} from the trace."""
    out = {}
    for pj, st, comm, s, e, mv in trace[key]:
        out.setdefault((mv, st), []).append((comm, e - s, s, e))
    return out


def test_stage_split_and_order_p400(oracle_mod):
    """P:400 (Fig. 'schedule_kernel'): "device 1 holds the first two layers of
    the encoder, while device 2 holds the next two layers ... device 2 can only
    utilize bubbles that occur after device 1 completes its forward pass ...
    for backward computation ... in the reverse order."  Four encoder layers
    over two encoder stages: every moved chain places exactly two layers'
    kernels on each stage, stage 2's forward kernels all start after stage 1's
    last forward kernel ends, and a backward chain finishes on stage 2 before
    it starts on stage 1."""
    prob = toy_problem()  # encoder of 4 identical layers; plan (P=2, T=2) has m = 2
    o = oracle_mod.Oracle(prob)
    pl = oracle_mod.plans(prob)["plans"]
    e = next(i for i, q in enumerate(pl) if q["P"] == 2 and q["T"] == 2)
    per_layer_f = len(prob["branches"][0]["fwd"][1])
    per_layer_b = len(prob["branches"][0]["bwd"][1])
    seen_f = seen_b = 0
    for g in range(pl[e]["first"], pl[e]["first"] + pl[e]["count"]):
        t = o.trace(g)
        for key, per in (("fwd_place", per_layer_f), ("bwd_place", per_layer_b)):
            ch = _chain_stage_kernels(t, key)
            for mvi in {k[0] for k in ch}:
                s0, s1 = ch[(mvi, 0)], ch[(mvi, 1)]
                assert len(s0) == len(s1) == 2 * per  # two layers per device
                if key == "fwd_place":
                    assert min(x[2] for x in s1) >= max(x[3] for x in s0)
                    seen_f += 1
                else:
                    assert min(x[2] for x in s0) >= max(x[3] for x in s1)
                    seen_b += 1
    assert seen_f > 0 and seen_b > 0


def test_multibranch_per_encoder_split_p478(oracle_mod):
    """P:474-478 (Fig. 'multi_enc_design'): "layers within each encoder are
    divided into PP_enc stages ... The bubble scheduler breaks down the layers
    of distinct encoders into kernel-level granularity and arranges their
    scheduling as if these kernels were part of a single encoder."  Branch A
    (4 layers) and branch B (2 layers) with distinct kernel durations over two
    stages: every stage of every moved chain carries two A layers and one B
    layer (per-encoder split; splitting the concatenated 6 layers instead would
    put A0-A2 on stage 1 and A3, B0, B1 on stage 2), both branches within one
    chain."""
    prob = toy_problem()
    C = 0
    a_f = [(C, 17), (C, 29)]
    a_b = [(C, 31), (C, 37)]
    b_f = [(C, 41), (C, 43)]
    b_b = [(C, 47), (C, 53)]
    prob["branches"] = [{"layers": 4, "params": 100, "fwd": [a_f, a_f], "bwd": [a_b, a_b]},
                        {"layers": 2, "params": 100, "fwd": [b_f, b_f], "bwd": [b_b, b_b]}]
    o = oracle_mod.Oracle(prob)
    pl = oracle_mod.plans(prob)["plans"]
    e = next(i for i, q in enumerate(pl) if q["P"] == 2 and q["count"])
    want_f = sorted([d for _, d in a_f] * 2 + [d for _, d in b_f])
    want_b = sorted([d for _, d in a_b] * 2 + [d for _, d in b_b])
    seen = 0
    for g in range(pl[e]["first"], pl[e]["first"] + pl[e]["count"]):
        t = o.trace(g)
        assert t["tau_f"] == [sum(want_f)] * 2 and t["tau_b"] == [sum(want_b)] * 2
        for key, want in (("fwd_place", want_f), ("bwd_place", want_b)):
            for (mvi, st), ks in _chain_stage_kernels(t, key).items():
                assert sorted(d for _, d, _, _ in ks) == want, (g, key, mvi, st)
                seen += 1
    assert seen > 0


# ------------------------------------------------- NEXT-2 Megatron-LM baselines
def test_partition_dp_hand_solved(oracle_mod):
    """App. B: F(l, m) = min_{j<l} max(F(j, m-1), sum t_(j+1..l)).
    Hand-solved: t = 1..5 over 2 virtual stages -> [1,2,3 | 4,5], largest 9
    (the other splits give 10, 12, 14)."""
    assert oracle_mod.partition_dp([1, 2, 3, 4, 5], 2) == (9, [3, 2])
    assert oracle_mod.partition_dp([5, 1, 1, 1, 1, 1], 3)[0] == 5  # the 5-layer stands alone
    assert oracle_mod.partition_dp([1, 1], 3) == (-1, [])  # fewer layers than virtual stages


def test_partition_dp_bruteforce(oracle_mod):
    """The DP's value is the minimum over every split of L layers into VP
    non-empty contiguous groups of the largest group sum (exhaustive), and
    its returned split attains it."""
    rng = random.Random(7)
    for _ in range(300):
        L = rng.randint(1, 9)
        VP = rng.randint(1, min(L, 4))
        t = [rng.randint(1, 20) for _ in range(L)]
        best = None
        for cuts in itertools.combinations(range(1, L), VP - 1):
            b = (0,) + cuts + (L,)
            mx = max(sum(t[b[i]:b[i + 1]]) for i in range(VP))
            best = mx if best is None else min(best, mx)
        val, sizes = oracle_mod.partition_dp(t, VP)
        assert val == best, (t, VP)
        assert len(sizes) == VP and min(sizes) >= 1 and sum(sizes) == L
        acc, mx = 0, 0
        for sz in sizes:
            mx = max(mx, sum(t[acc:acc + sz]))
            acc += sz
        assert mx == val


def _baseline_problem(p, v, n, t_llm, t_enc, enc_layers, llm_layers, T_ag=0, T_rs=0):
    """Uniform single-kernel layers: LLM layer (t_llm fwd, 2 t_llm bwd), encoder
    layer (t_enc, 2 t_enc); TP 1."""
    enc = {"layers": enc_layers, "params": 1, "fwd": [[(0, t_enc)]], "bwd": [[(0, 2 * t_enc)]]}
    pb = uniform_problem(p, v, n, t_llm, 2 * t_llm, T_ag=T_ag, T_rs=T_rs, enc=enc)
    pb["llm_layers"] = llm_layers
    return pb


def test_baseline_balanced_uniform_closed_form(oracle_mod):
    """Balanced: identical layers split evenly over V x PP virtual
    stages, then Megatron's interleaved 1F1B with uniform ops: iteration =
    T_ag + (n v + p - 1)(t_f + t_b) + T_rs (the closed form the template pin
    uses, per virtual stage of k layers)."""
    for p, v, n in [(2, 2, 4), (4, 2, 8), (3, 1, 6), (4, 3, 8)]:
        VP = p * v
        enc_layers, llm_layers = VP, VP * 2  # 3 identical layers per virtual stage
        pb = _baseline_problem(p, v, n, 10, 10, enc_layers, llm_layers, T_ag=7, T_rs=11)
        b = oracle_mod.baseline(pb, 1)
        assert b["sizes"] == [3] * VP
        assert b["iter_ns"] == 7 + (n * v + p - 1) * (30 + 60) + 11


def test_baseline_naive_sequential_closed_form(oracle_mod):
    """Naive (encoder in the first pipeline stage): with p = v = 1 the
    schedule is sequential, iteration = T_ag + n (encoder + LLM, forward +
    backward) + T_rs; with p = 2 the encoder lengthens only virtual stage 0."""
    pb = _baseline_problem(1, 1, 3, 10, 7, 4, 5, T_ag=5, T_rs=9)
    b = oracle_mod.baseline(pb, 0)
    assert b["sizes"] == [4 + 5]
    assert b["iter_ns"] == 5 + 3 * (4 * 7 + 4 * 14 + 5 * 10 + 5 * 20) + 9
    pb = _baseline_problem(2, 1, 2, 10, 7, 4, 6)
    b = oracle_mod.baseline(pb, 0)
    assert b["sizes"] == [4 + 3, 3]
    assert b["opF"] == [4 * 7 + 3 * 10, 3 * 10] and b["opB"] == [4 * 14 + 3 * 20, 3 * 20]


def test_baseline_balanced_single_encoder_only(oracle_mod):
    """"this DP algorithm does not apply to MLLM models that feature
    multiple encoders"; the naive placement does."""
    prob = config_problem(5, 16)
    assert oracle_mod.baseline(prob, 1) is None
    assert oracle_mod.baseline(prob, 0)["iter_ns"] > 0
