import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2604_16402_b200 as g
from paper_2604_16402_b200 import datasets as ds, _lib
X, S = ds.gen_lowrank(1_000_000, 128, seed=0)
gi, _ = g.build_index(X, S, g.BuildParams(k_max=32, k_local=16, bucket_capacity=10_000))
Q = ds.lowrank_queries(10_000, 128, seed=1)
for sel, it, mi in ((0.1, 296, 100), (0.01, 400, 150)):
    lo, hi = ds.range_arrays(ds.generate_ranges(S, sel, 10_000, 0))
    r = g.search_arrays(gi, Q, lo, hi, g.SearchParams(k=10, itopk=it, search_width=4, max_iterations=mi), seed_base=0)
    st = r.stats
    de = st['dist_evals'].astype(float); itr = st['iterations'].astype(float); ga = st['gathered'].astype(float)
    cost = de * 512 + itr * 2000
    print(sel, 'dist_evals mean %.0f std %.0f p5 %.0f p95 %.0f max %.0f' % (de.mean(), de.std(), *np.percentile(de, [5, 95]), de.max()))
    print(sel, 'iterations mean %.1f std %.1f min %d max %d; frac at max_iter %.2f' % (itr.mean(), itr.std(), itr.min(), itr.max(), (itr >= mi).mean()))
    # correlation with range position / span
    span = hi - lo
    print(sel, 'corr(dist_evals, lo) %.3f' % np.corrcoef(de, lo)[0, 1])
