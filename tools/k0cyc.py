# Dev diagnostic: build with OPTIMUS_NVCC_EXTRA=-DK0_CYC first. Usage: python tools/k0cyc.py 4
import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
from paper_2408_03505_b200 import optimus_load_costs
from paper_2408_03505_b200.optimus import lib
from workload import config_problem
prob = config_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
ctx = optimus_load_costs(prob)
for i in range(3): ctx.rebuild(); torch.cuda.synchronize()
a = np.zeros((1024, 4), dtype=np.int64)
L = lib(); L.optimus_debug_k0cyc.argtypes = [ctypes.c_void_p]
assert L.optimus_debug_k0cyc(a.ctypes.data) == 0
u = a[:, 3] > 0
a = a[u]
t0 = a[:, 2].min()
print('sims', len(a), 'setup cyc mean %d max %d' % (a[:, 0].mean(), a[:, 0].max()), 'sim cyc mean %d max %d' % (a[:, 1].mean(), a[:, 1].max()))
print('start spread us %.1f, end max us %.1f' % ((a[:, 2].max() - t0) / 1e3, (a[:, 3].max() - t0) / 1e3))
for b in (0, 1, 100, 288):
    if b < len(a): print(b, a[b, 0], a[b, 1], (a[b, 2] - t0) / 1e3, (a[b, 3] - t0) / 1e3)
