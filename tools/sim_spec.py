import sys, time, bisect
sys.path.insert(0, "/root/repo")
import numpy as np
from dataclasses import replace
from paper_2305_04359_b200 import datagen
from oracle.oracle import Oracle
n = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
cl = max(1, n // 10000)
cfg = replace(datagen.CONFIGS["c1"], n=n, clusters=cl)
base = datagen.host_base_parallel(cfg)
qs = datagen.host_queries(replace(cfg, n_queries=16))
orc = Oracle("ref")
t = time.time()
adj, start = orc.build(base, 64, 128, 1.2, cap=int(n * 0.02), workers=8)
print("built", time.time() - t, flush=True)
np.save("/tmp/sim/adj.npy", adj); np.save("/tmp/sim/base.npy", base)  # reused by tools/sim_spec_batched.py
b32 = base.astype(np.int32)
def sim(q, L):
    q = q.astype(np.int32)
    def dist(ids):
        x = b32[ids] - q
        return (x * x).sum(1)
    beam = [(int(dist([start])[0]), start)]
    expanded = set(); visited = {start}
    order = []  # expansion sequence
    snap = []   # per step: first 8 unexpanded at that time
    newcount = []; survcount = []
    while True:
        un = [k for k in beam if k[1] not in expanded]
        if not un: break
        snap.append(un[:8])
        k = un[0]; expanded.add(k[1]); order.append(k)
        nb = [int(v) for v in adj[k[1]] if v != 0xFFFFFFFF and int(v) not in visited]
        visited.update(nb)
        newcount.append(len(nb))
        s = 0
        if nb:
            ds = dist(nb)
            for dd, v in zip(ds, nb):
                key = (int(dd), v)
                if len(beam) < L or key < beam[-1]:
                    bisect.insort(beam, key); s += 1
                    if len(beam) > L: beam.pop()
        survcount.append(s)
    return order, snap, newcount, survcount
for L in (200, 832):
    depth_hist = np.zeros(9, int); steps = 0; batches = {2: 0, 4: 0, 8: 0}
    nn = []; ss = []
    for qi in range(6):
        order, snap, nc, sc = sim(qs[qi], L)
        nn += nc; ss += sc
        T = len(order)
        dep = []
        for t in range(T):
            d = 0
            while d < len(snap[t]) and t + d < T and order[t + d] == snap[t][d]:
                d += 1
            dep.append(d); depth_hist[d] += 1
        steps += T
        for E in batches:
            t = 0; nb = 0
            while t < T:
                t += max(1, min(E, dep[t])); nb += 1
            batches[E] += nb
    print("L", L, "steps", steps, "depth hist", depth_hist / steps, "batches", {E: steps / b for E, b in batches.items()},
          "new/exp", np.mean(nn), "surv/exp", np.mean(ss), flush=True)
