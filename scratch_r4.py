import torch
import __graft_entry__; __graft_entry__.build()
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
p=config_problem(4); ctx=optimus_load_costs(p); total,_=ctx.num_candidates()
b2=torch.empty(2,dtype=torch.int64,device='cuda')
for w in (1, 4, 16):
    for rep in range(3):
        ctx.eval_candidates(0,total,b2,rank=0,world=w); torch.cuda.synchronize()
