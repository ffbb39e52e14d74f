import torch, sys
import __graft_entry__; __graft_entry__.build()
from paper_2408_03505_b200 import optimus_load_costs
from workload import config_problem
for cfg in [(4,None)]:
    p=config_problem(*cfg); ctx=optimus_load_costs(p); total,np_=ctx.num_candidates()
    b2=torch.empty(2,dtype=torch.int64,device='cuda')
    ctx.set_timing(True)
    for e in range(np_):
        q=ctx.get_plan(e)
        if q['count']<1000: continue
        ts=[]
        for rep in range(5):
            ctx.rebuild(); s0=ctx.eval_stats(); ctx.eval_candidates(q['first'],q['first']+q['count'],b2); torch.cuda.synchronize()
            b,k=ctx.last_timing(); ts.append(k); s1=ctx.eval_stats()
        d={k:(s1[k]-s0[k])/q['count'] for k in s1}
        print(e, q, 'k2 ms', round(sorted(ts)[2],4), 'ns/cand', round(sorted(ts)[2]*1e6/q['count'],3), 'general', round(d['general'],3), 'itf', round(d['iters_f'],2), 'atb', round(d['attempts_b'],2), flush=True)
