"""Host-side checks of the C ABI (-m "not gpu"): the library builds for sm_100a,
loads, exports every symbol include/optimus.h declares, validates problems,
enumerates plans like the oracle, decodes indices like the oracle, and refuses
to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

from workload import config_problem, random_problem, toy_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2408_03505_b200 import optimus
    return optimus


def test_exports_every_header_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "optimus.h")).read()
    declared = set(re.findall(r"\b(optimus_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 14
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(L.HEADER_SYMBOLS)


def test_sm100a_binary(L):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _err(L, prob):
    with pytest.raises(L.OptimusError) as ei:
        L.optimus_workspace_bytes(L.Problem(prob))
    return ei.value.code, str(ei.value)


def test_validation_errors(L):
    p = toy_problem()
    p["n_gpu"] = 9
    assert _err(L, p)[0] == -1
    p = toy_problem()
    p["llm_layers"] = 15
    code, msg = _err(L, p)
    assert code == -1 and "PP*V = 8" in msg
    p = toy_problem()
    p["n_mb"] = 6
    assert _err(L, p)[0] == -1
    p = toy_problem()
    p["llm_fwd_layer"] = [(0, 5), (1, 0)]
    assert _err(L, p)[0] == -1
    p = toy_problem()
    p["tp_opts"] = [2, 1]
    assert _err(L, p)[0] == -1
    p = toy_problem()
    p["branches"][0]["layers"] = 0
    assert _err(L, p)[0] == -1
    p = toy_problem()
    p["llm_fwd_layer"] = [(1, 5)]
    assert _err(L, p)[0] == -1  # no compute kernel


def test_infeasible(L):
    p = toy_problem()
    p["gpu_mem_bytes"] = 1
    ctx = L.optimus_plan_only(p)
    assert ctx.num_candidates()[0] == 0


@pytest.mark.parametrize("prob", [toy_problem(), config_problem(1), config_problem(2), config_problem(3),
                                  config_problem(4), config_problem(5, 16), config_problem(5, 32)] +
                         [random_problem(s) for s in range(10)], ids=lambda p: p["name"])
def test_plans_match_oracle(L, oracle_mod, prob):
    ctx = L.optimus_plan_only(prob)
    total, n = ctx.num_candidates()
    ref = oracle_mod.plans(prob)
    assert total == ref["total"] and n == len(ref["plans"])
    for i, r in enumerate(ref["plans"]):
        g = ctx.get_plan(i)
        assert (g["pp"], g["tp"], g["dp"], g["m"], g["count"], g["first"]) == \
            (r["P"], r["T"], r["dp_enc"], r["m"], r["count"], r["first"])


def test_best_plan_decode_matches_oracle(L, oracle_mod):
    prob = config_problem(4)
    ctx = L.optimus_plan_only(prob)
    total, _ = ctx.num_candidates()
    plans = oracle_mod.plans(prob)["plans"]
    rng = np.random.default_rng(1)
    for g in rng.integers(0, total, 300).tolist():
        res = ctx.best_plan([[123, g], [2**63 - 1, -1]])
        pl = [p for p in plans if p["count"] and p["first"] <= g < p["first"] + p["count"]][0]
        assert res["index"] == g and res["lat_ns"] == 123
        assert res["enc"][1:] == (pl["P"], pl["T"]) and res["m"] == pl["m"]
        assert res["counts"] == oracle_mod.unrank(prob["n_mb"], pl["m"], g - pl["first"])
    # lexicographic minimum across ranks, ties -> lowest index
    res = ctx.best_plan([[5, 900], [5, 100], [6, 0]])
    assert (res["lat_ns"], res["index"]) == (5, 100)


def test_no_cpu_fallback(L):
    """Without a usable GPU, load must fail loudly with ECUDA, never compute on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    P = L.Problem(toy_problem())
    h = ctypes.c_void_p()
    rc = L.lib().optimus_load_costs(ctypes.byref(P.s), ctypes.c_void_p(1 << 20), 1 << 40, None, ctypes.byref(h))
    assert rc == -3 and not h.value


def test_rank_share_tiles(L):
    from paper_2408_03505_b200.dist import rank_share
    for n, world, block in [(20703, 8, 4096), (5845247, 8, 4096), (1000, 3, 64), (64, 4, 64), (0, 2, 64)]:
        assert sum(rank_share(0, n, r, world, block) for r in range(world)) == n


@pytest.mark.parametrize("n_mb", [64, 128])
def test_config5_wide_sweep_points_plans(L, oracle_mod, n_mb):
    """Config 5's sweep points N_mb = 64 and 128 (K2 mode 1's wide instance,
    n <= 128): the library enumerates the oracle's plans and totals (SURVEY
    Appendix A: 2,213,201,944 and 357,426,663,480 candidates)."""
    prob = config_problem(5, n_mb)
    ctx = L.optimus_plan_only(prob)
    total, n = ctx.num_candidates()
    ref = oracle_mod.plans(prob)
    assert total == ref["total"] == {64: 2213201944, 128: 357426663480}[n_mb]
    for i, r in enumerate(ref["plans"]):
        g = ctx.get_plan(i)
        assert (g["pp"], g["tp"], g["m"], g["count"], g["first"]) == (r["P"], r["T"], r["m"], r["count"], r["first"])


def test_n_mb_limit(L):
    p = config_problem(5, 128)
    p["n_mb"] = 136
    code, msg = _err(L, p)
    assert code == -5 and "exceeds the supported 128" in msg


def test_eval_instance_selection(L):
    """K2 mode 1 instance by (n_mb, largest m with candidates), host only."""
    import sys, os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gpu_parity import kmax128_problem, mid_m_problem, wide_m_problem
    from workload import config_problem
    cases = [(config_problem(4), 0), (config_problem(3), 0), (config_problem(3, 64), 1), (mid_m_problem(), 2),
             (wide_m_problem(), 3), (config_problem(5, 64), 4), (config_problem(5, 128), 5), (kmax128_problem(), 5)]
    for prob, inst in cases:
        ctx = L.optimus_plan_only(prob)
        assert ctx.eval_instance()[0] == inst, prob["name"]
