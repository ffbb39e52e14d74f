# Dev diagnostic (not part of the product path): build with OPTIMUS_NVCC_EXTRA=-DK1_TRACE first.
# Usage: python tools/k1trace.py 4 2   (configs)
# K1 per-item timeline and per-warp cycle breakdown (liboptimus built with -DK1_TRACE)
import sys, ctypes, collections
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2408_03505_b200 import optimus_load_costs
from paper_2408_03505_b200.optimus import lib
from workload import config_problem
CAT = ['prolog', 'setup', 'nslow', 'vwait', 'loop', 'upwait', 'total', 'slowcyc', 'publish', 'nfast', 'nadv', 'advcyc', 'nfound', 'flushcyc']
for cfg in [int(x) for x in sys.argv[1:]]:
    prob = config_problem(cfg)
    ctx = optimus_load_costs(prob)
    L = lib(); L.optimus_debug_k1trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.optimus_debug_k1stats.argtypes = [ctypes.c_void_p]
    for rep in range(2):
        ctx.rebuild(); torch.cuda.synchronize()
    assert L.optimus_debug_k1reset() == 0
    ctx.rebuild(); torch.cuda.synchronize()
    buf = np.zeros((16384, 4), dtype=np.uint64)
    assert L.optimus_debug_k1trace(buf.ctypes.data, 16384) == 0
    stats = np.zeros((4096, 32, 14), dtype=np.uint64)
    assert L.optimus_debug_k1stats(stats.ctypes.data) == 0
    used = np.nonzero(buf[:, 0] > 0)[0]
    t = buf[used].astype(np.int64)
    t0 = t[:, 0].min()
    st = (t[:, 0] - t0) / 1000; en = (t[:, 1] - t0) / 1000
    u = t[:, 2]; typ = u >> 30; e = (u >> 16) & 0x3FFF; a = (u >> 8) & 255; kf = u & 255
    print(f"=== config {cfg}: {len(used)} items, span {en.max():.1f} us")
    dur = en - st
    for ty, nm in ((0, 'fwd'), (1, 'bwd'), (2, 'tables')):
        sel = typ == ty
        if sel.any():
            print(f"  {nm}: n={sel.sum()} dur mean {dur[sel].mean():.1f} max {dur[sel].max():.1f} sum {dur[sel].sum():.0f} us; <1us {np.sum(dur[sel] < 1)}")
    for ee in sorted(set(e.tolist())):
        sel = e == ee
        f = sel & (typ == 0); b = sel & (typ == 1)
        bv = b & (dur > 1)
        if not f.any(): continue
        print(f"  plan {ee:2d}: fwd [{st[f].min():6.1f},{en[f].max():6.1f}] | bwd valid {bv.sum():3d} first {st[bv].min() if bv.any() else 0:6.1f} done {en[sel].max():6.1f} bwd maxdur {dur[bv].max() if bv.any() else 0:6.1f}")
    # breakdown of the 6 longest fwd and bwd units
    for ty in (0, 1):
        idx = [i for i in np.argsort(-dur) if typ[i] == ty][:4]
        for i in idx:
            it = used[i]
            print(f"  {'fwd' if ty == 0 else 'bwd'} item {it} plan {e[i]} a {a[i]} kf {kf[i]} dur {dur[i]:.1f} us")
            for w in range(32):
                row = stats[it, w]
                if row[6] == 0: continue
                print('     w%2d ' % w + ' '.join(f"{CAT[q]}={row[q] if q in (2, 9, 10, 12) else row[q] / 1965:.1f}" for q in range(14)))
