import torch
from paper_2408_03505_b200 import build as B
B.build(force=True)
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
p=config_problem(4); ctx=optimus_load_costs(p); torch.cuda.synchronize()
print("---- rebuild", flush=True)
ctx.rebuild(); torch.cuda.synchronize()
