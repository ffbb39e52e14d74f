"""Pins of the oracle's scheduling efficiency (oracle/eff.py; reading R-EFF,
PAPER.md §5.3.2): closed forms at the two extremes and the ordering
invariants the definition implies."""
import numpy as np
import pytest

from workload import random_problem, toy_problem


def _eff(O, E, prob, g):
    return E.efficiency(prob, g, O.Oracle(prob))


def test_bubbles_larger_than_all_encoder_work(oracle_mod):
    """Huge DP all-gather / reduce-scatter bubbles hold every coarse
    microbatch: both efficiencies are exactly 1 and nothing moves."""
    from oracle import eff as E
    prob = toy_problem()
    prob["dp_allgather_ns"] = 10 ** 9
    prob["dp_reducescatter_ns"] = 10 ** 9
    for g in range(8):
        r = _eff(oracle_mod, E, prob, g)
        assert r["total"] > 0
        assert r["in_bubble_coarse"] == r["total"] == r["in_bubble_fine"], g


def test_no_natural_bubble_single_stage(oracle_mod):
    """One LLM stage, no DP bubbles, layers that begin and end with compute:
    the LLM computes from t = 0 to T_end (w = 0, z = T_end), so
    no coarse work lies in a bubble (Eff_coarse = 0 exactly); Eff_fine counts
    only the moved chains."""
    from oracle import eff as E
    for seed in range(40):
        prob = random_problem(seed, max_p=1)
        prob["dp_allgather_ns"] = 0
        prob["dp_reducescatter_ns"] = 0
        for k in ("llm_fwd_layer", "llm_bwd_layer"):  # the LLM computes from its first to its last kernel
            prob[k] = [(0, 50)] + list(prob[k]) + [(0, 50)]
        o = oracle_mod.Oracle(prob)
        for g in range(min(4, 1000)):
            try:
                r = E.efficiency(prob, g, o)
            except ValueError:
                break
            assert r["in_bubble_coarse"] == 0, (seed, g)
            t = o.trace(g)
            moved = sum((t["N"][j] - t["c_final"][j]) * sum(t["tau_f"]) + (t["N"][j] - t["cb_final"][j]) * sum(t["tau_b"])
                        for j in range(t["m"]))
            assert r["in_bubble_fine"] == moved, (seed, g)


@pytest.mark.parametrize("seed", range(12))
def test_efficiency_ordering(oracle_mod, seed):
    """0 <= in-bubble (coarse only) <= in-bubble (with moves) <= total: a move
    takes the latest coarse microbatch out of the fill and places all of its
    kernels inside bubbles."""
    from oracle import eff as E
    from paper_2408_03505_b200 import optimus_plan_only
    prob = random_problem(seed)
    total, _ = optimus_plan_only(prob).num_candidates()
    o = oracle_mod.Oracle(prob)
    for g in np.unique(np.linspace(0, total - 1, 6).astype(int)):
        r = E.efficiency(prob, int(g), o)
        assert 0 <= r["in_bubble_coarse"] <= r["in_bubble_fine"] <= r["total"], (seed, g, r)
