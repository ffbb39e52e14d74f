"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Bit-exact integer equality on every compared value: the template (F, B, w, z,
T_end, warm-up counts, every compute-free / comm-free interval), the per-row
chain tables, every candidate's lat and the argmin (lat, index).
"""
import os

import numpy as np
import pytest

from workload import config_problem, random_problem, sample_indices, toy_problem

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    return torch


def _load(prob, mode=1):
    from paper_2408_03505_b200 import optimus_load_costs
    ctx = optimus_load_costs(prob)
    ctx.set_eval_mode(mode)
    return ctx


MODES = pytest.mark.parametrize("mode", [0, 1], ids=["warp_per_cand", "thread_per_cand"])


SMALL = [toy_problem(), config_problem(1), config_problem(2)] + [random_problem(s) for s in range(40)]
BIG = [config_problem(3), config_problem(4), config_problem(5, 16), config_problem(5, 32)]


@pytest.mark.parametrize("prob", SMALL[:8] + BIG, ids=lambda p: p["name"])
def test_template_parity(dev, oracle_mod, prob):
    ctx = _load(prob)
    g = ctx.debug_template()
    o = oracle_mod.template(prob)
    for k in ("T_end", "W", "F", "B", "w", "z"):
        assert g[k] == o[k], k
    assert g["span_def"] == o["span_def"]
    for s in range(prob["llm"]["pp"]):
        assert g["comp_free"][s] == [tuple(x) for x in o["comp_free"][s]], f"stage {s} compute-free"
        assert g["comm_free"][s] == [tuple(x) for x in o["comm_free"][s]], f"stage {s} comm-free"


@pytest.mark.parametrize("prob", [toy_problem(), config_problem(2), config_problem(4)] +
                         [random_problem(s) for s in range(12)], ids=lambda p: p["name"])
def test_chain_tables_parity(dev, oracle_mod, prob):
    ctx = _load(prob)
    o = oracle_mod.Oracle(prob)
    _, n_plans = ctx.num_candidates()
    checked = 0
    for e in range(n_plans):
        t = ctx.debug_plan_tables(e)
        if t is None:
            continue
        assert t["PRE_F"][-1][1:] == [oracle_mod.gpipe(_taus(prob, ctx.get_plan(e), 0), prob["enc_p2p_ns"],
                                                       prob["n_mb"])[-1][x] for x in range(1, prob["n_mb"] + 1)]
        for a in range(t["rp"]):
            assert t["INB_F"][a] == o.row_chains(e, a, -1, t["kmax"]), (e, a)
            for kf in range(t["lenF"][a] + 1):
                assert t["INB_B"][a][kf] == o.row_chains(e, a, kf, t["kmax"]), (e, a, kf)
                checked += 1
    assert checked > 0


def _taus(prob, plan, bwd):
    """Stage sums of the encoder work (test-side restatement of R8)."""
    P, T = plan["pp"], plan["tp"]
    ti = prob["tp_opts"].index(T)
    out = []
    for s in range(P):
        tot = 0
        for b in prob["branches"]:
            L = b["layers"]
            nl = (s + 1) * L // P - s * L // P
            tot += nl * sum(ns for _, ns in (b["bwd"] if bwd else b["fwd"])[ti])
        out.append(tot)
    return out


@MODES
@pytest.mark.parametrize("prob", SMALL + [config_problem(5, 16)], ids=lambda p: p["name"])
def test_full_space_parity(dev, oracle_mod, prob, mode):
    torch = dev
    ctx = _load(prob, mode)
    total, _ = ctx.num_candidates()
    lat = torch.full((total,), -7, dtype=torch.int64, device="cuda")
    best2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, best2, lat_out=lat)
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(prob)
    ref = o.eval(np.arange(total, dtype=np.uint64), threads=THREADS)
    got = lat.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first g={bad[:5].tolist()} got={got[bad[:5]].tolist()} ref={ref[bad[:5]].tolist()}"
    b = best2.cpu().numpy()
    assert (int(b[0]), int(b[1])) == (int(ref.min()), int(np.argmin(ref)))


@pytest.fixture(scope="module")
def config4_oracle_lat(oracle_mod):
    """Oracle lat of every one of config 4's 5,845,247 candidates (SURVEY §8(d):
    full-space oracle parity for configs 1, 2 and 4; ~30 s on 16 host cores)."""
    prob = config_problem(4)
    o = oracle_mod.Oracle(prob)
    return prob, o.eval_range(0, o.total, threads=THREADS)


@MODES
def test_full_space_parity_config4(dev, config4_oracle_lat, mode):
    """The bench workload, every candidate: the lat dump of the launch bench.py
    times (eval_candidates over the whole range) equals the oracle element by
    element, and the argmin equals the oracle's first minimum."""
    torch = dev
    prob, ref = config4_oracle_lat
    ctx = _load(prob, mode)
    total, _ = ctx.num_candidates()
    assert total == len(ref) == 5845247
    lat = torch.full((total,), -7, dtype=torch.int64, device="cuda")
    best2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, best2, lat_out=lat)
    torch.cuda.synchronize()
    got = lat.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first g={bad[:5].tolist()}"
    b = best2.cpu().numpy()
    assert (int(b[0]), int(b[1])) == (int(ref.min()), int(np.argmin(ref)))


SAMPLED = 1 << 17  # the first 2^17 indices of the seeded stream for configs 3 and 5
_ORACLE_SAMPLES = {}


def _oracle_sample(oracle_mod, prob, count):
    """(indices, oracle lats) of the seeded stream, computed once per problem."""
    key = (prob["name"], count)
    if key not in _ORACLE_SAMPLES:
        o = oracle_mod.Oracle(prob)
        idx = np.array(sample_indices(20241018, count, o.total), dtype=np.uint64)
        _ORACLE_SAMPLES[key] = (idx, o.eval(idx, threads=THREADS))
        o.close()
    return _ORACLE_SAMPLES[key]


def _sampled_parity(dev, oracle_mod, prob, mode, count):
    torch = dev
    ctx = _load(prob, mode)
    idx, ref = _oracle_sample(oracle_mod, prob, count)
    di = torch.from_numpy(idx.astype(np.int64)).cuda()
    lat = torch.empty(len(idx), dtype=torch.int64, device="cuda")
    best2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_indices(di, best2, lat_out=lat)
    torch.cuda.synchronize()
    got = lat.cpu().numpy()
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first idx={idx[bad[:5]].tolist()}"
    b = best2.cpu().numpy()
    j = min(range(len(idx)), key=lambda i: (ref[i], idx[i]))
    assert (int(b[0]), int(b[1])) == (int(ref[j]), int(idx[j]))
    return ctx


@MODES
@pytest.mark.parametrize("prob", BIG, ids=lambda p: p["name"])
def test_sampled_parity_full_size(dev, oracle_mod, prob, mode):
    """BASELINE sizes: 2^17 seeded indices per config through eval_indices
    (the first 2^17 of the seeded stream for configs 3 and 5)."""
    _sampled_parity(dev, oracle_mod, prob, mode, SAMPLED)


@MODES
@pytest.mark.parametrize("prob", [config_problem(4), config_problem(2)], ids=lambda p: p["name"])
def test_contiguous_ranges_full_size(dev, oracle_mod, prob, mode):
    """The launch configuration bench.py times (eval_candidates over ranges),
    checked on a ragged window that straddles plan boundaries."""
    torch = dev
    ctx = _load(prob, mode)
    total, n_plans = ctx.num_candidates()
    firsts = [ctx.get_plan(i)["first"] for i in range(n_plans) if ctx.get_plan(i)["count"]]
    for f in firsts[1:4]:
        begin, end = max(0, f - 1000), min(total, f + 1337)
        lat = torch.empty(end - begin, dtype=torch.int64, device="cuda")
        best2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(begin, end, best2, lat_out=lat)
        torch.cuda.synchronize()
        ref = oracle_mod.Oracle(prob).eval_range(begin, end, threads=THREADS)
        assert np.array_equal(lat.cpu().numpy(), ref)


@MODES
@pytest.mark.parametrize("world", [2, 3, 8])
def test_rank_sharding(dev, oracle_mod, world, mode):
    """Block-cyclic sharding: every rank's best, gathered and decoded, equals the
    single-rank answer; lat dumps of all ranks tile the space exactly once."""
    torch = dev
    prob = config_problem(2)
    ctx = _load(prob, mode)
    total, _ = ctx.num_candidates()
    lat = torch.full((total,), -1, dtype=torch.int64, device="cuda")
    gathered = []
    for r in range(world):
        b2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(0, total, b2, lat_out=lat, rank=r, world=world, block=128)
        gathered.append(b2)
    torch.cuda.synchronize()
    assert int((lat < 0).sum()) == 0
    one = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, one)
    g = torch.stack(gathered).cpu().numpy()
    res = ctx.best_plan(g)
    o1 = one.cpu().numpy()
    assert (res["lat_ns"], res["index"]) == (int(o1[0]), int(o1[1]))
    ref = oracle_mod.Oracle(prob).eval(np.array([res["index"]], dtype=np.uint64))[0]
    assert ref == res["lat_ns"]


@MODES
def test_edge_cases(dev, oracle_mod, mode):
    torch = dev
    from paper_2408_03505_b200 import OptimusError
    prob = toy_problem()
    ctx = _load(prob, mode)
    total, _ = ctx.num_candidates()
    b2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(5, 5, b2)  # empty range
    torch.cuda.synchronize()
    assert b2.cpu().tolist() == [2**63 - 1, -1]
    with pytest.raises(OptimusError):
        ctx.eval_candidates(0, total + 1, b2)
    ctx.eval_candidates(total - 1, total, b2)  # one candidate
    torch.cuda.synchronize()
    o = oracle_mod.Oracle(prob)
    assert b2.cpu().tolist() == [int(o.eval([total - 1])[0]), total - 1]
    # rebuild from device-resident inputs is idempotent
    ctx.rebuild()
    lat = torch.empty(total, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, b2, lat_out=lat)
    torch.cuda.synchronize()
    assert np.array_equal(lat.cpu().numpy(), o.eval(np.arange(total, dtype=np.uint64)))


@MODES
def test_degenerate_problems(dev, oracle_mod, mode):
    """Zero-kernel encoder, N_mb = PP (all warm-up), m = N_mb plans, v = 1."""
    torch = dev
    probs = []
    p = toy_problem()
    p["branches"][0]["fwd"] = [[], []]
    p["branches"][0]["bwd"] = [[], []]
    probs.append(p)
    for s in range(200, 260):
        q = random_problem(s, max_n=6)
        if q["n_mb"] == q["llm"]["pp"] or q["llm"]["v"] == 1:
            probs.append(q)
    assert len(probs) > 5
    for prob in probs:
        ctx = _load(prob, mode)
        total, _ = ctx.num_candidates()
        lat = torch.empty(total, dtype=torch.int64, device="cuda")
        b2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(0, total, b2, lat_out=lat)
        torch.cuda.synchronize()
        ref = oracle_mod.Oracle(prob).eval(np.arange(total, dtype=np.uint64))
        assert np.array_equal(lat.cpu().numpy(), ref), prob["name"]


def test_rebuild_determinism(dev, oracle_mod):
    """Full-size chain tables are identical across rebuilds, whatever ran on
    the GPU in between (another context's K2 leaves different registers and
    shared memory behind), and match the oracle's row chains."""
    torch = dev
    prob = config_problem(4)
    ctx, other = _load(prob), _load(prob)
    total, n_plans = ctx.num_candidates()

    def tables():
        torch.cuda.synchronize()
        return [ctx.debug_plan_tables(e) for e in range(n_plans)]

    base = tables()
    o = oracle_mod.Oracle(prob)
    for e, t in enumerate(base):
        if t is not None:
            assert t["INB_F"][0] == o.row_chains(e, 0, -1, t["kmax"]), e
    idx = torch.from_numpy(np.array(sample_indices(7, 2048, total), dtype=np.int64)).cuda()
    b2 = torch.empty(2, dtype=torch.int64, device="cuda")
    for it in range(4):
        (other if it % 2 else ctx).eval_indices(idx, b2)
        other.eval_candidates(0, min(total, 100000), b2)
        ctx.rebuild()
        assert tables() == base, it


def _wide_problem(seed, pp, v, k):
    """A random problem re-planned onto a wide LLM pipeline (PP 16..32: the
    K1 launch variants for more than 12 stage warps per block)."""
    q = random_problem(seed, max_p=8, max_t=2, max_n=8)
    lc = 1
    q["name"] = f"wide_pp{pp}_v{v}_{seed}"
    q["llm"] = {"dp": 2, "pp": pp, "tp": q["llm"]["tp"], "v": v}
    q["llm_layers"] = pp * v * lc
    q["n_mb"] = pp * k
    q["n_gpu"] = pp * q["llm"]["tp"] * 2
    return q


WIDE = [_wide_problem(3, 16, 2, 2), _wide_problem(5, 24, 1, 1), _wide_problem(8, 32, 1, 1)]


@pytest.mark.parametrize("prob", WIDE, ids=lambda p: p["name"])
def test_wide_pipelines(dev, oracle_mod, prob):
    """Template, every plan's chain tables and sampled candidates for LLM
    pipelines of 16, 24 and 32 stages."""
    torch = dev
    ctx = _load(prob)
    g = ctx.debug_template()
    o = oracle_mod.template(prob)
    for k in ("T_end", "W", "F", "B", "w", "z"):
        assert g[k] == o[k], k
    orc = oracle_mod.Oracle(prob)
    total, n_plans = ctx.num_candidates()
    for e in range(n_plans):
        t = ctx.debug_plan_tables(e)
        if t is None:
            continue
        for a in range(t["rp"]):
            assert t["INB_F"][a] == orc.row_chains(e, a, -1, t["kmax"]), (e, a)
            for kf in range(t["lenF"][a] + 1):
                assert t["INB_B"][a][kf] == orc.row_chains(e, a, kf, t["kmax"]), (e, a, kf)
    idx = np.array(sample_indices(99, min(total, 512), total), dtype=np.uint64)
    lat = torch.empty(len(idx), dtype=torch.int64, device="cuda")
    b2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_indices(torch.from_numpy(idx.astype(np.int64)).cuda(), b2, lat_out=lat)
    torch.cuda.synchronize()
    assert np.array_equal(lat.cpu().numpy(), orc.eval(idx, threads=THREADS))


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_default_warmup_policy(dev, oracle_mod, seed):
    """warmup_policy 0 (Megatron default warm-up, no R5 adjustment): template
    and the full candidate space."""
    torch = dev
    prob = random_problem(seed)
    prob["warmup_policy"] = 0
    prob["name"] += "_policy0"
    ctx = _load(prob)
    g = ctx.debug_template()
    o = oracle_mod.template(prob)
    for k in ("T_end", "W", "F", "B", "w", "z"):
        assert g[k] == o[k], k
    total, _ = ctx.num_candidates()
    lat = torch.empty(total, dtype=torch.int64, device="cuda")
    b2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, b2, lat_out=lat)
    torch.cuda.synchronize()
    assert np.array_equal(lat.cpu().numpy(), oracle_mod.Oracle(prob).eval(np.arange(total, dtype=np.uint64)))


STRESS = [random_problem(s, max_p=8, max_t=8, max_n=16) for s in range(300, 420)]


@pytest.mark.parametrize("chunk", range(4))
def test_stress_sweep(dev, oracle_mod, chunk):
    """120 wider random problems (PP up to 8, TP up to 8, up to 16
    microbatches, jittered kernels, P2P latencies): every candidate of the
    small spaces, 2048 seeded candidates of the large ones, through the
    overlapped K1/K2 path (eval_candidates) and the explicit path."""
    torch = dev
    for prob in STRESS[chunk::4]:
        ctx = _load(prob)
        total, _ = ctx.num_candidates()
        if total == 0:
            continue
        o = oracle_mod.Oracle(prob)
        b2 = torch.empty(2, dtype=torch.int64, device="cuda")
        if total <= 50000:
            lat = torch.empty(total, dtype=torch.int64, device="cuda")
            ctx.eval_candidates(0, total, b2, lat_out=lat)
            torch.cuda.synchronize()
            ref = o.eval(np.arange(total, dtype=np.uint64), threads=THREADS)
            assert np.array_equal(lat.cpu().numpy(), ref), prob["name"]
            assert int(b2[1].item()) == int(np.argmin(ref)), prob["name"]
        else:
            idx = np.array(sample_indices(5, 2048, total), dtype=np.uint64)
            lat = torch.empty(len(idx), dtype=torch.int64, device="cuda")
            ctx.eval_indices(torch.from_numpy(idx.astype(np.int64)).cuda(), b2, lat_out=lat)
            torch.cuda.synchronize()
            assert np.array_equal(lat.cpu().numpy(), o.eval(idx, threads=THREADS)), prob["name"]


@pytest.mark.parametrize("prob", [config_problem(2), config_problem(4)] + [random_problem(s) for s in range(20)],
                         ids=lambda p: p["name"])
def test_explain_matches_oracle_trace(dev, oracle_mod, prob):
    """optimus_explain (NEXT-1 decisions) against the oracle's trace: lat,
    shifts, move counts and order (the trace's placement records carry the
    moving pipeline and the move number), composition and coarse counts."""
    ctx = _load(prob)
    total, _ = ctx.num_candidates()
    o = oracle_mod.Oracle(prob)
    idx = sample_indices(17, min(total, 64), total)
    lat, aux = o.eval(np.array(idx, dtype=np.uint64), aux=True)
    aux = np.asarray(aux)
    picks = list(idx[:8]) + [int(idx[i]) for i in np.argsort(-(aux[:, 2] + aux[:, 3]))[:8]]
    for g in picks:
        x = ctx.explain(int(g))
        t = o.trace(int(g))
        assert (x["lat"], x["df"], x["db"], x["mf"], x["mb"]) == (t["lat"], t["df"], t["db"], t["mf"], t["mb"]), g
        assert x["N"] == t["N"] and x["c_final"] == t["c_final"] and x["cb_final"] == t["cb_final"], g
        for key, recs in (("moves_f", t["fwd_place"]), ("moves_b", t["bwd_place"])):
            seq = {}
            for r in recs:
                seq.setdefault(r[5], r[0])
            assert x[key] == [seq[k] for k in sorted(seq)], (g, key)


@pytest.mark.parametrize("prob", [config_problem(2), config_problem(4)] + [random_problem(s) for s in range(20)],
                         ids=lambda p: p["name"])
def test_emit_schedule_matches_oracle_trace(dev, oracle_mod, prob):
    """optimus_emit_schedule (NEXT-1): every in-bubble kernel placement of the
    committed moves, record for record, against the oracle's trace."""
    ctx = _load(prob)
    total, _ = ctx.num_candidates()
    o = oracle_mod.Oracle(prob)
    idx = sample_indices(23, min(total, 64), total)
    lat, aux = o.eval(np.array(idx, dtype=np.uint64), aux=True)
    aux = np.asarray(aux)
    picks = [int(idx[i]) for i in np.argsort(-(aux[:, 2] + aux[:, 3]))[:6]] + [int(idx[0])]
    records = 0
    for g in picks:
        x = ctx.emit_schedule(g)
        t = o.trace(g)
        assert x["fwd_place"] == t["fwd_place"], g
        assert x["bwd_place"] == t["bwd_place"], g
        records += len(x["fwd_place"]) + len(x["bwd_place"])
    if prob["name"].startswith("c4"):
        assert records > 0  # config 4's busiest candidates move kernels into bubbles


@pytest.mark.parametrize("prob", [config_problem(2), config_problem(4)] + [random_problem(s) for s in range(16)],
                         ids=lambda p: p["name"])
def test_efficiency_matches_oracle(dev, oracle_mod, prob):
    """optimus_efficiency (NEXT-1, R-EFF) against oracle/eff.py, exact integers."""
    from oracle import eff as E
    ctx = _load(prob)
    total, _ = ctx.num_candidates()
    o = oracle_mod.Oracle(prob)
    for g in sample_indices(29, min(total, 12), total):
        assert ctx.efficiency(int(g)) == E.efficiency(prob, int(g), o), g


def table7_problem(n_mb):
    """Table 7's setting (App. D): ViT-22B + GPT-175B, LLM
    PP 8 x TP 8, global batch 1536 at microbatch 2, so N_mb = 32 / 24 / 16 on
    1536 / 2048 / 3072 GPUs (DP 24 / 32 / 48): config 5's LLM with its ViT-22B
    branch alone."""
    prob = config_problem(5, n_mb)
    dp = {32: 24, 24: 32, 16: 48}[n_mb]
    prob["name"] = f"table7_vit22b_gpt175b_pp8_n{n_mb}"
    prob["branches"] = prob["branches"][:1]
    prob["llm"]["dp"] = dp
    prob["n_gpu"] = dp * 8 * 8
    return prob


def test_efficiency_trend_table7(dev):
    """Table 7's direction: with the global batch fixed, fewer
    microbatches per LLM pipeline give higher Eff_coarse and Eff_fine for the
    chosen schedule (the paper: 34.3 / 45.8 / 68.7% coarse, 57.5 / 69.3 / 85.0%
    fine at N_mb 32 / 24 / 16), on the paper's ViT-22B + GPT-175B PP-8 setting."""
    torch = dev
    effs = []
    for n_mb in (32, 24, 16):
        prob = table7_problem(n_mb)
        ctx = _load(prob)
        total, _ = ctx.num_candidates()
        b2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(0, total, b2)
        torch.cuda.synchronize()
        r = ctx.efficiency(int(b2[1].item()))
        effs.append((r["in_bubble_coarse"] / r["total"], r["in_bubble_fine"] / r["total"]))
    print("Table 7 analogue, Eff (coarse, fine) at N_mb 32/24/16:", [(round(a, 4), round(b, 4)) for a, b in effs])
    for (c0, f0), (c1, f1) in zip(effs, effs[1:]):
        assert c1 >= c0 and f1 >= f0
    assert all(f >= c for c, f in effs)


# ---------------------------------------------------------------------------
# N_mb 64 / 128 (config 5's sweep): K2 mode 1's instances for n > 32
WIDE_NMB = [config_problem(5, 64), config_problem(5, 128)]


@pytest.mark.parametrize("prob", WIDE_NMB, ids=lambda p: p["name"])
def test_wide_template_parity(dev, oracle_mod, prob):
    test_template_parity(dev, oracle_mod, prob)


@pytest.mark.parametrize("prob", WIDE_NMB, ids=lambda p: p["name"])
def test_wide_sampled_parity(dev, oracle_mod, prob):
    """2^17 seeded indices of the 2.2e9 / 3.6e11 spaces through eval_indices."""
    _sampled_parity(dev, oracle_mod, prob, 1, SAMPLED)


@pytest.mark.parametrize("prob", WIDE_NMB, ids=lambda p: p["name"])
def test_wide_contiguous_ranges(dev, oracle_mod, prob):
    """The range path (overlapped with K1, claims per plan) on windows that
    straddle plan boundaries, plus the very first and last candidates."""
    torch = dev
    ctx = _load(prob, 1)
    total, n_plans = ctx.num_candidates()
    firsts = [ctx.get_plan(i)["first"] for i in range(n_plans) if ctx.get_plan(i)["count"]]
    o = oracle_mod.Oracle(prob)
    wins = [(max(0, f - 700), min(total, f + 901)) for f in firsts[1:4]] + [(0, 1500), (total - 1300, total)]
    for begin, end in wins:
        lat = torch.empty(end - begin, dtype=torch.int64, device="cuda")
        best2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(begin, end, best2, lat_out=lat)
        torch.cuda.synchronize()
        ref = o.eval_range(begin, end, threads=THREADS)
        got = lat.cpu().numpy()
        assert np.array_equal(got, ref), (begin, end, int((got != ref).sum()))
        b = best2.cpu().numpy()
        assert (int(b[0]), int(b[1])) == (int(ref.min()), begin + int(np.argmin(ref)))


def test_wide_mode0_refused(dev):
    from paper_2408_03505_b200.optimus import OptimusError
    torch = dev
    ctx = _load(config_problem(5, 64), 0)
    best2 = torch.empty(2, dtype=torch.int64, device="cuda")
    with pytest.raises(OptimusError) as ei:
        ctx.eval_candidates(0, 100, best2)
    assert ei.value.code == -5


# ---------------------------------------------------------------------------
# K2 mode 1 instances for n > 32 with plans of m > 16 pipelines: (64, 64),
# (128, 64) and (128, 128) slots x pipelines per thread
def wide_m_problem():
    """LLM PP 22 x TP 3 with N_mb = 66: the (P = 1, T = 1) plan has m = 66 > 64
    pipelines (instance (128, 128)).  A plan with m > 64 always comes with one
    of m / 2, and C(n - 1, m / 2 - 1) fits in 64 bits only for n up to ~67, so
    this is about the largest such space the index type allows (3.7e18).  Small
    random kernels, memory never binding."""
    from workload.gen import _Rng, _rand_layer
    q = random_problem(7, max_p=4, max_t=2, max_n=8)
    pp, tp = 22, 3
    q["name"] = "wide_m66_pp22_tp3_n66"
    q["llm"] = {"dp": 1, "pp": pp, "tp": tp, "v": 1}
    q["llm_layers"] = pp
    q["n_mb"] = 66
    q["n_gpu"] = pp * tp
    q["tp_opts"] = [1, 3]
    rng = _Rng(77)
    q["llm_fwd_layer"] = _rand_layer(rng, tp, 400, 3)
    q["llm_bwd_layer"] = _rand_layer(rng, tp, 800, 3)
    q["branches"] = [{"layers": 4, "params": 1000,
                      "fwd": [_rand_layer(rng, T, max(2, 60 // T), 2) for T in q["tp_opts"]],
                      "bwd": [_rand_layer(rng, T, max(2, 120 // T), 2) for T in q["tp_opts"]]}]
    return q


def mid_m_problem():
    """LLM PP 20, TP 1 with N_mb = 80: plans with m = 20 pipelines and n > 64
    (instance (128, 64)); config 3 at N_mb > 66 would overflow the 64-bit
    candidate index (C(n - 1, 31) for its m = 32 plans)."""
    from workload.gen import _Rng, _rand_layer
    q = random_problem(8, max_p=4, max_t=1, max_n=8)
    pp = 20
    q["name"] = "mid_m20_pp20_tp1_n80"
    q["llm"] = {"dp": 1, "pp": pp, "tp": 1, "v": 1}
    q["llm_layers"] = pp
    q["n_mb"] = 80
    q["n_gpu"] = pp
    q["tp_opts"] = [1]
    rng = _Rng(88)
    q["llm_fwd_layer"] = _rand_layer(rng, 1, 400, 3)
    q["llm_bwd_layer"] = _rand_layer(rng, 1, 800, 3)
    q["branches"] = [{"layers": 5, "params": 1000, "fwd": [_rand_layer(rng, 1, 90, 2)],
                      "bwd": [_rand_layer(rng, 1, 180, 2)]}]
    return q


INSTANCE_PROBS = [(config_problem(3, 64), 1), (mid_m_problem(), 2), (wide_m_problem(), 3)]


@pytest.mark.parametrize("prob,inst", INSTANCE_PROBS, ids=lambda x: x["name"] if isinstance(x, dict) else str(x))
def test_instance_sampled_parity(dev, oracle_mod, prob, inst):
    """2^17 seeded indices through eval_indices on the (64, 64), (128, 64)
    and (128, 128) instances (verdict r1: never compared with the oracle)."""
    ctx = _sampled_parity(dev, oracle_mod, prob, 1, SAMPLED)
    assert ctx.eval_instance()[0] == inst


@pytest.mark.parametrize("prob,inst", INSTANCE_PROBS, ids=lambda x: x["name"] if isinstance(x, dict) else str(x))
def test_instance_ranges(dev, oracle_mod, prob, inst):
    """The range path (overlapped with K1, claims per plan) on the same
    instances: windows straddling every plan boundary, the first and the last
    candidates, and the whole of every plan with m > 16 that is small."""
    torch = dev
    ctx = _load(prob, 1)
    assert ctx.eval_instance()[0] == inst
    total, n_plans = ctx.num_candidates()
    plans = [ctx.get_plan(i) for i in range(n_plans)]
    firsts = [q["first"] for q in plans if q["count"]]
    wins = [(max(0, f - 500), min(total, f + 701)) for f in firsts[1:]] + [(0, 1200), (total - 1100, total)]
    wins += [(q["first"], q["first"] + q["count"]) for q in plans if q["m"] > 16 and 0 < q["count"] <= 4000]
    o = oracle_mod.Oracle(prob)
    for begin, end in wins:
        lat = torch.empty(end - begin, dtype=torch.int64, device="cuda")
        best2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(begin, end, best2, lat_out=lat)
        torch.cuda.synchronize()
        ref = o.eval_range(begin, end, threads=THREADS)
        got = lat.cpu().numpy()
        assert np.array_equal(got, ref), (begin, end, int((got != ref).sum()))
        b = best2.cpu().numpy()
        assert (int(b[0]), int(b[1])) == (int(ref.min()), begin + int(np.argmin(ref)))


def kmax128_problem():
    """Config 1 at N_mb = 128 with the encoder's kernels 10x shorter: its m = 1
    plan (P = 2, T = 2) fits all kmax = n - m + 1 = 128 forward chains, so K1
    publishes snapshot versions up to 128 (advisor r1: int8 owner versions)."""
    p = config_problem(1, n_mb=128)
    p["name"] = "c1_n128_enc_div10"
    for b in p["branches"]:
        b["fwd"] = [[(k, max(1, ns // 10)) for k, ns in lst] for lst in b["fwd"]]
        b["bwd"] = [[(k, max(1, ns // 10)) for k, ns in lst] for lst in b["bwd"]]
    return p


def test_kmax128_chain_tables(dev, oracle_mod):
    prob = kmax128_problem()
    ctx = _load(prob)
    o = oracle_mod.Oracle(prob)
    _, n_plans = ctx.num_candidates()
    full = 0
    for e in range(n_plans):
        t = ctx.debug_plan_tables(e)
        if t is None:
            continue
        for a in range(t["rp"]):
            assert t["INB_F"][a] == o.row_chains(e, a, -1, t["kmax"]), (e, a)
            for kf in range(t["lenF"][a] + 1):
                assert t["INB_B"][a][kf] == o.row_chains(e, a, kf, t["kmax"]), (e, a, kf)
            full += t["lenF"][a] == 128
    assert full > 0  # the m = 1 plan placed all 128 forward chains
    _sampled_parity(dev, oracle_mod, prob, 1, 4096)


# ---------------------------------------------------------------------------
# NEXT-2: Megatron-LM baselines (App. B) on the GPU
BASE_PROBS = [config_problem(c) for c in (1, 2, 3, 4)] + [config_problem(5, 16), toy_problem()] + \
    [random_problem(s) for s in range(30)]


@pytest.mark.parametrize("prob", BASE_PROBS, ids=lambda p: p["name"])
def test_megatron_baselines_parity(dev, oracle_mod, prob):
    """optimus_baseline (naive and balanced) against the oracle: iteration
    time, the virtual-stage layer counts (App. B's DP) and every op time."""
    from paper_2408_03505_b200 import OptimusError
    ctx = _load(prob)
    for kind in (0, 1):
        ref = oracle_mod.baseline(prob, kind)
        if ref is None:  # several encoders or fewer layers than virtual stages
            with pytest.raises(OptimusError):
                ctx.baseline(kind)
            continue
        assert ctx.baseline(kind) == ref, kind


def test_megatron_speedup_config4(dev, oracle_mod):
    """Optimus's best schedule against both baselines on the headline space
    (the paper: 20.5% over balanced, 21.3% over Megatron-LM on 3072 Hopper
    GPUs; context only).  Optimus never loses to the balanced baseline
    here, and both baselines are slower than the LLM-only template."""
    torch = dev
    prob = config_problem(4)
    ctx = _load(prob)
    total, _ = ctx.num_candidates()
    b2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, b2)
    torch.cuda.synchronize()
    lat = int(b2[0].item())
    naive, bal = ctx.baseline(0)["iter_ns"], ctx.baseline(1)["iter_ns"]
    print(f"config 4: Optimus {lat} ns, Megatron naive {naive} ns ({naive / lat - 1:.1%} slower), "
          f"balanced {bal} ns ({bal / lat - 1:.1%} slower)")
    assert lat < bal < naive


# ---------------------------------------------------------------------------
# NEXT-4: encoder-LLM P2P insertion and schedule export
@pytest.mark.parametrize("prob", [toy_problem(), config_problem(2), config_problem(4)] +
                         [random_problem(s) for s in range(12)], ids=lambda p: p["name"])
def test_emit_p2p_matches_oracle(dev, oracle_mod, prob):
    """optimus_emit_p2p record for record against the pairs assembled from the
    oracle's global ordering (its trace) and its template's B_i."""
    ctx = _load(prob)
    total, _ = ctx.num_candidates()
    o = oracle_mod.Oracle(prob)
    tpl = oracle_mod.template(prob)
    L = prob["enc_llm_p2p_ns"]
    plans = oracle_mod.plans(prob)["plans"]
    for g in sample_indices(31, min(total, 24), total):
        t = o.trace(int(g))
        P, rt = t["P"], t["r_t"]
        want = []
        for i, (val, j) in enumerate(t["order"]):
            a, b = j // rt, j % rt
            last = a * P + P - 1
            want.append([0, i, j, last, b, 0, b, val, val + L])
            want.append([1, i, j, 0, b, last, b, tpl["B"][i], tpl["B"][i] + L])
        got = ctx.emit_p2p(int(g))
        assert got == want, g
        for r in got:  # the dependencies the pairs serve (R20)
            if r[0] == 0:
                assert r[8] <= tpl["F"][r[1]] + t["df"]


def test_schedule_export(dev, tmp_path):
    """The winner of config 4 as JSON and Chrome trace: every emitted kernel and
    P2P pair appears, events are well formed."""
    torch = dev
    from paper_2408_03505_b200 import export
    prob = config_problem(4)
    ctx = _load(prob)
    total, _ = ctx.num_candidates()
    b2 = torch.empty(2, dtype=torch.int64, device="cuda")
    ctx.eval_candidates(0, total, b2)
    torch.cuda.synchronize()
    g = int(b2[1].item())
    sch = export.schedule(ctx, g)
    assert sch["lat_ns"] == int(b2[0].item()) and len(sch["p2p"]["records"]) == 2 * prob["n_mb"]
    tr = export.chrome_trace(ctx, g)
    nk = len(sch["encoder_kernels"]["forward"]) + len(sch["encoder_kernels"]["backward"])
    assert sum(1 for e in tr["traceEvents"] if e["name"].startswith("enc ")) == nk
    assert sum(1 for e in tr["traceEvents"] if e["name"].startswith("p2p ")) == 4 * prob["n_mb"]
    assert all(e["ph"] == "X" and e["dur"] >= 0 for e in tr["traceEvents"])
    export.write(ctx, g, str(tmp_path / "c4.trace.json"))
    import json
    assert json.load(open(tmp_path / "c4.trace.json"))["otherData"]["candidate"] == g


# ---------------------------------------------------------------------------
# NEXT-3: a sweep over LLM templates in one call
def test_sweep_matches_single_templates(dev, oracle_mod):
    """optimus_sweep_*: config 5's N_mb 16 / 32 templates plus three other
    LLM templates in one workspace and one call; every template's best equals
    its own single search, and the oracle's where the space is small."""
    torch = dev
    from paper_2408_03505_b200.optimus import Sweep
    probs = [config_problem(5, 16), config_problem(5, 32), toy_problem(), random_problem(4), config_problem(2)]
    sw = Sweep(probs)
    best = torch.empty((len(probs), 2), dtype=torch.int64, device="cuda")
    sw.eval(best)
    torch.cuda.synchronize()
    got = best.cpu().numpy()
    for i, prob in enumerate(probs):
        ctx = _load(prob)
        total, _ = ctx.num_candidates()
        b2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(0, total, b2)
        torch.cuda.synchronize()
        assert (int(got[i][0]), int(got[i][1])) == tuple(int(x) for x in b2.cpu().numpy()), prob["name"]
        if total <= 30000:
            assert (int(got[i][0]), int(got[i][1])) == oracle_mod.Oracle(prob).best(threads=THREADS), prob["name"]
        res = sw.ctxs[i].best_plan(got[i:i + 1])
        assert res["lat_ns"] == int(got[i][0])
    # a second sweep evaluation (rebuild + eval) is identical
    sw.eval(best)
    torch.cuda.synchronize()
    assert (best.cpu().numpy() == got).all()
    sw.free()
