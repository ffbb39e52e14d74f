# Dev diagnostic: one rank's block-cyclic K2 shard on one GPU (library K2 timing). Usage: python tools/k2shard.py 4 1 2 4 8
# K2 on one rank's block-cyclic shard (world W) on one GPU: library K2 time
import sys, torch
sys.path.insert(0, '.')
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
cfg = int(sys.argv[1]); W = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
prob = config_problem(cfg)
ctx = optimus_load_costs(prob)
total, _ = ctx.num_candidates()
best2 = torch.empty(2, dtype=torch.int64, device='cuda')
flush = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
ctx.set_timing(True)
for w in W:
    ks = []
    for it in range(8):
        flush.zero_()
        ctx.rebuild()
        ctx.eval_candidates(0, total, best2, rank=0, world=w)
        torch.cuda.synchronize()
        b, k = ctx.last_timing()
        if it >= 3: ks.append(k)
    st = ctx.eval_stats()
    print(f"cfg {cfg} world {w}: K2 {sum(ks)/len(ks):.4f} ms  (x{0 if w==1 else 1})", flush=True)
