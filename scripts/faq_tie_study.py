"""FAQ on exactly tied gradients depends on BLAS rounding (build container only).

The reference's acceptance criterion 5 (test_acceptance.py:158-182) asks FAQ for a mean
match ratio >= 0.95 over 25 isomorphic SBM pairs (rho = 1, seed 7).  FAQ's first LAP runs on
the barycenter gradient, whose entries tie EXACTLY among equal-degree vertices; the
reference forms it with two dgemm calls whose last-bit rounding breaks those ties
pseudo-randomly.  This script runs the UNMODIFIED reference twice per replicate: as
shipped, and with the first gradient replaced by its exact rank-2 value
(ra rb^T + ca cb^T) / n -- which is what the device path computes (A11).
Measured here: mean 0.962 as shipped vs 0.922 with the exact first gradient
(profiles/round2_faq_tie_study.txt), i.e. the criterion's FAQ clause is decided by
OpenBLAS rounding noise, not by the algorithm.
"""
import sys, numpy as np
sys.path.insert(0,'/root/reference/pkg/src'); sys.path.insert(0,'/root/repo')
import otmatch
from otmatch import matcher as rm
from otmatch.cli import _sbm_spec, SBM_ACCURACY_B, _derive_seed
res=[]
for rep in range(25):
    rng=np.random.default_rng([7,1000,rep])
    A,B=otmatch.sample_sbm_pair(_sbm_spec(150,SBM_ACCURACY_B,1.0),rng)
    Bs,truth=otmatch.shuffle_pair(B,rng)
    opts=otmatch.MatchOptions(step_solver="exact_lap",rng_seed=_derive_seed(7,1000,rep))
    r=otmatch.frank_wolfe_match(A,Bs,opts)
    # emulate the device path: exact rank-2 barycenter gradient for the first step
    orig=rm.gradient
    n=150
    def grad(A_,B_,P_):
        if np.all(P_==P_[0,0]):
            return (np.outer(A_.sum(1),B_.sum(1))+np.outer(A_.sum(0),B_.sum(0)))/n
        return orig(A_,B_,P_)
    rm.gradient=grad
    try: r2=otmatch.frank_wolfe_match(A,Bs,opts)
    finally: rm.gradient=orig
    res.append((rep,otmatch.match_ratio(r.alignment,truth),otmatch.match_ratio(r2.alignment,truth)))
    print(res[-1],flush=True)
print(np.mean([x[1] for x in res]),np.mean([x[2] for x in res]))
