import torch, sys
import __graft_entry__; __graft_entry__.build()
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
for cfg in [(4,None),(2,None)]:
    p=config_problem(*cfg); ctx=optimus_load_costs(p); total,_=ctx.num_candidates()
    b2=torch.empty(2,dtype=torch.int64,device='cuda')
    ctx.set_timing(True)
    for f in [0.02, 0.1, 0.25, 0.5, 1.0]:
        end=int(total*f); ts=[]
        for rep in range(6):
            ctx.rebuild(); ctx.eval_candidates(0,end,b2); torch.cuda.synchronize()
            b,k=ctx.last_timing(); ts.append(k)
        print(p['name'], f, end, 'k2 ms', round(sorted(ts)[3],4), 'build', round(b,4), flush=True)
