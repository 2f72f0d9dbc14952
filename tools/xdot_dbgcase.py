import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1210_6412_b200 import dots
rng = np.random.default_rng(1)
cases = {}
for n in (1, 2, 31, 32, 33, 255, 256, 257, 1000, 8191, 65537):
    cases[f"normal{n}"] = (rng.standard_normal(n), rng.standard_normal(n))
n = 10**6
cases["walk"] = (rng.standard_normal(n), rng.standard_normal(n))
cases["positive"] = (np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n)))
for name in ("normal65537", "walk", "positive"):
    u, v = cases[name]
    got, st = dots.dot_stats(u, v)
    print(name, got, np.cumsum(u*v)[-1], {k: x for k, x in st.items() if x}, flush=True)
    if name == "positive":
        for k in (3,):
            g, parts = dots.dot_blocks(u, v, k)
            print('blocks', g, parts)
            base, extra = divmod(len(u), k); st_=0; ws=[]
            for i in range(k):
                sz = base + (1 if i < extra else 0); ws.append(np.cumsum(u[st_:st_+sz]*v[st_:st_+sz])[-1]); st_ += sz
            print('want  ', ws)
