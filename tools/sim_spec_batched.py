import sys, bisect
sys.path.insert(0, "/root/repo")
import numpy as np
from dataclasses import replace
from paper_2305_04359_b200 import datagen
adj = np.load("/tmp/sim/adj.npy"); base = np.load("/tmp/sim/base.npy")
n = len(base)
cfg = replace(datagen.CONFIGS["c1"], n=n, clusters=max(1, n // 10000))
qs = datagen.host_queries(replace(cfg, n_queries=16))
b32 = base.astype(np.int32)
# start: medoid-ish = closest to mean (approx; fine for stats)
start = int(np.argmin(((b32 - b32.mean(0)) ** 2).sum(1)))
def sim_batched(q, L, E, CM=128):
    q = q.astype(np.int32)
    dist = lambda ids: ((b32[ids] - q) ** 2).sum(1)
    beam = [(int(dist([start])[0]), start)]
    expanded = set(); visited = {start}
    nb_batches = nexp = cand_nodedupe = cand_dedupe = wasted = 0
    fails = 0
    while True:
        un = [k for k in beam if k[1] not in expanded][:E]
        if not un: break
        nb_batches += 1
        # speculative candidates
        rows = []
        seen_batch = set(); tot = 0
        for k in un:
            fresh = [int(v) for v in adj[k[1]] if v != 0xFFFFFFFF and int(v) not in visited]
            if rows and tot + len(fresh) > CM: break
            tot += len(fresh)
            cand_nodedupe += len(fresh)
            f2 = [v for v in fresh if v not in seen_batch]
            seen_batch.update(f2)
            cand_dedupe += len(f2)
            rows.append((k, fresh, f2))
        # sequential commit
        P = 0
        for (k, fresh, f2) in rows:
            cur_un = [kk for kk in beam if kk[1] not in expanded]
            if cur_un[0] != k: fails += 1; break
            expanded.add(k[1]); P += 1; nexp += 1
            nbn = [v for v in fresh if v not in visited]
            visited.update(nbn)
            if nbn:
                for dd, v in zip(dist(nbn), nbn):
                    key = (int(dd), v)
                    if len(beam) < L or key < beam[-1]:
                        bisect.insort(beam, key)
                        if len(beam) > L: beam.pop()
        wasted += sum(len(r[2]) for r in rows[P:])
    return nb_batches, nexp, cand_nodedupe, cand_dedupe, wasted
for L in (128, 200, 832):
    for E in (2, 4, 8):
        tot = np.zeros(5)
        for qi in range(4):
            tot += np.array(sim_batched(qs[qi], L, E))
        b, x, c0, c1, w = tot
        print(f"L={L} E={E}: exp/batch {x/b:.2f} cands/exp nodedupe {c0/x:.1f} dedupe {c1/x:.1f} wasted/exp {w/x:.1f}", flush=True)
