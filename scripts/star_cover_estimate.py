"""Tuning estimate (not part of the product): staged slices per distinct block if every pair were
evaluated at the endpoint that covers more pairs (a star cover of the pair graph: P + |cover| instead
of T + P), from the oracle's ALIGNED lists. Result (round 2, session 4): c2 seed 0 1.504 -> 1.479,
seed 2 2.734 -> 2.646, c3 6 sequences 1.824 -> 1.801 -- the cover is nearly T, not worth a kernel."""
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, oracle
from synth import workloads
from _gpu_util import oracle_steps, oracle_candidates
from collections import Counter
def analyze(w, name):
    oc = oracle_candidates(w, oracle_steps(w), w.tau_s, 0, oracle.ALIGNED)
    to = oc['target_off']; pr = oc['pairs']
    tp, sp = pr['target_phys'], pr['source_phys']
    T=len(to)-1; P=len(tp); U=len(np.unique(np.concatenate([tp,sp])))
    deg=Counter(); 
    for a,b in zip(tp,sp): deg[a]+=1; deg[b]+=1
    # greedy 1: center = higher-degree endpoint (tie -> target)
    centers=set(a if deg[a]>=deg[b] else b for a,b in zip(tp,sp))
    # greedy 2: iterative max-degree vertex cover
    edges=set(zip(tp.tolist(),sp.tolist()))
    adj={}
    for a,b in edges: adj.setdefault(a,set()).add(b); adj.setdefault(b,set()).add(a)
    cover=0
    import heapq
    d={v:len(n) for v,n in adj.items()}
    while any(d.values()):
        v=max(d,key=d.get)
        if d[v]==0: break
        cover+=1
        for u in list(adj[v]):
            adj[u].discard(v); d[u]-=1
        adj[v]=set(); d[v]=0
    print(f"{name}: U={U} T={T} P={P} staged target-major={(T+P)/U:.3f}  star(deg)={(P+len(centers))/U:.3f} (stars {len(centers)})  star(greedyVC)={(P+cover)/U:.3f} (cover {cover})")
analyze(workloads.c2(seed=0),'c2 s0')
analyze(workloads.c2(seed=2),'c2 s2')
analyze(workloads.c3(num_seqs=6),'c3 6seq')
