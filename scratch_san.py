"""Small searches for compute-sanitizer: configs 1 and 2, both K2 modes, ranges and indices, explain/emit/baselines."""
import sys
import numpy as np, torch
import __graft_entry__; __graft_entry__.build()
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem, toy_problem, random_problem
probs = [config_problem(1), config_problem(2), toy_problem(), random_problem(3)]
for prob in probs:
    for mode in (1, 0):
        ctx = optimus_load_costs(prob); ctx.set_eval_mode(mode)
        total, _ = ctx.num_candidates()
        lat = torch.empty(total, dtype=torch.int64, device="cuda"); b2 = torch.empty(2, dtype=torch.int64, device="cuda")
        ctx.eval_candidates(0, total, b2, lat_out=lat)
        idx = torch.arange(0, total, max(1, total // 512), dtype=torch.int64, device="cuda")
        l2 = torch.empty(len(idx), dtype=torch.int64, device="cuda")
        ctx.eval_indices(idx, b2, lat_out=l2)
        ctx.rebuild(); ctx.eval_candidates(0, total, b2)
        torch.cuda.synchronize()
        g = int(b2[1].item())
        ctx.explain(g); ctx.emit_schedule(g); ctx.efficiency(g)
        ctx.baseline(0)
        if len(prob["branches"]) == 1: ctx.baseline(1)
        ctx.free()
print("san workload ok")
