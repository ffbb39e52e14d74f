import torch, numpy as np, json
import __graft_entry__; __graft_entry__.build()
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
for cfg in [(4,None),(3,None),(5,64),(2,None)]:
    p=config_problem(*cfg); ctx=optimus_load_costs(p); total,_=ctx.num_candidates()
    b2=torch.empty(2,dtype=torch.int64,device='cuda')
    s0=ctx.eval_stats()
    end=min(total, 50_000_000)
    ctx.eval_candidates(0,end,b2); torch.cuda.synchronize()
    s1=ctx.eval_stats()
    d={k:(s1[k]-s0[k]) for k in s1}
    nc=d['candidates']
    print(p['name'], {k: v/nc for k,v in d.items()})
