import time, numpy as np, scipy.linalg as sla
from threadpoolctl import threadpool_limits, threadpool_info
print([ (d['internal_api'], d['num_threads']) for d in threadpool_info()])
rng=np.random.default_rng(0)
for m in (64, 104, 144):
    A=rng.normal(size=(m,m))+1j*rng.normal(size=(m,m)); H=0.5*(A+A.conj().T)
    def t(f, n=30):
        f(); t0=time.perf_counter()
        for _ in range(n): f()
        return (time.perf_counter()-t0)/n*1e3
    print(m, 'np.eigh default', round(t(lambda: np.linalg.eigh(H)),3))
    for nt in (1,2,4):
        with threadpool_limits(limits=nt):
            print(m, 'np.eigh threads',nt, round(t(lambda: np.linalg.eigh(H)),3), 'sla evr', round(t(lambda: sla.eigh(H, driver='evr')),3), 'sla evd', round(t(lambda: sla.eigh(H, driver='evd')),3))
