import time, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2512_21615_b200 as edx
for rep in range(2):
    for k in (256, 512, 1024):
        rng = np.random.default_rng(k)
        a = rng.random((k, k))
        t0 = time.perf_counter(); edx.hungarian(edx.SquareCost(a)) if hasattr(edx, 'SquareCost') else edx.hungarian(a); dt = time.perf_counter() - t0
        print(rep, k, round(dt * 1e3, 2), flush=True)
