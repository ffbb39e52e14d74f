"""Scheduling efficiency of one candidate's schedule (oracle; TEST
INFRASTRUCTURE — only tests/, smoke() and bench.py's baseline legs may use it).

PAPER.md §5.3.2: "scheduling efficiency ... quantifies the percentage
of encoder computations that can be effectively scheduled within the LLM
bubble"; Eff_coarse with coarse-grained exploitation only, Eff_fine with both
(§4.2).  Reading R-EFF, in integer nanoseconds:

- encoder work = every encoder kernel of every microbatch, forward and
  backward, on every encoder stage: sum_j N_j * sum_s (tau_f[s] + tau_b[s]);
- a chain moved into the bubbles (fine-grained, R12/R15) is in-bubble work in
  full;
- coarse work (R9: the GPipe fill of the c_j pre-LLM forwards from time 0,
  mirrored for the cb_j post-LLM backwards) counts only where it lies inside
  the natural bubble of its device: [0, w_q) before the LLM's first compute
  on that device, [z_q, T_end) after its last (mirrored: [0, T_end - z_q));
  the rest is the overflow that lengthened the iteration;
- Eff_fine uses the candidate's final counts (c, cb); Eff_coarse the same
  candidate with no moves (c = cb = N).

Returns exact integers: in-bubble work with moves, without, and the total.
"""
from __future__ import annotations

from . import oracle as O


def _coarse_in_bubble(fill, tau, bubble, count):
    """Work of microbatches 1..count of a GPipe fill on one stage inside
    [0, bubble): microbatch x occupies [fill[x] - tau, fill[x])."""
    tot = 0
    for x in range(1, count + 1):
        lo, hi = fill[x] - tau, fill[x]
        tot += max(0, min(hi, bubble) - max(lo, 0))
    return tot


def efficiency(prob: dict, g: int, orc: "O.Oracle | None" = None) -> dict:
    orc = orc or O.Oracle(prob)
    tr = orc.trace(g)
    tp = O.template(prob)
    T_end = tp["T_end"]
    N, c, cb = tr["N"], tr["c_final"], tr["cb_final"]
    tau_f, tau_b = tr["tau_f"], tr["tau_b"]
    P, r_t, m = tr["P"], tr["r_t"], tr["m"]
    n = prob["n_mb"]
    p2p = prob["enc_p2p_ns"]
    fill_f = O.gpipe(tau_f, p2p, n)  # fill_f[s][x]: end of forward x on stage s (R9)
    fill_b = O.gpipe(tau_b, p2p, n)  # the mirrored backward fill
    total = fine = with_moves = without = 0
    for j in range(m):
        a = j // r_t
        for s in range(P):
            q = a * P + s
            pre, post = tp["w"][q], T_end - tp["z"][q]
            total += N[j] * (tau_f[s] + tau_b[s])
            fine += (N[j] - c[j]) * tau_f[s] + (N[j] - cb[j]) * tau_b[s]
            with_moves += (_coarse_in_bubble(fill_f[s], tau_f[s], pre, c[j])
                           + _coarse_in_bubble(fill_b[s], tau_b[s], post, cb[j]))
            without += (_coarse_in_bubble(fill_f[s], tau_f[s], pre, N[j])
                        + _coarse_in_bubble(fill_b[s], tau_b[s], post, N[j]))
    return {"in_bubble_fine": with_moves + fine, "in_bubble_coarse": without, "total": total}
