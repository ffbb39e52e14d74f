import torch
from paper_2408_03505_b200 import build as B
import os
B.build(force=True)
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
for cfg in [(4,None)]:
    p=config_problem(*cfg); ctx=optimus_load_costs(p); total,_=ctx.num_candidates()
    b2=torch.empty(2,dtype=torch.int64,device='cuda')
    s0=ctx.eval_stats(); ctx.eval_candidates(0,total,b2); torch.cuda.synchronize(); s1=ctx.eval_stats()
    d={k:(s1[k]-s0[k]) for k in s1}
    g=d['general']; a=d['claims']; b=d['unranks']
    print(p['name'], 'general', g, 'atb>0', a%1000000, 'materialized(have_order)', a//1000000, 'M>3', b%1000, 'M>1', (b//1000)%1000, 'M>2', b//1000000)
