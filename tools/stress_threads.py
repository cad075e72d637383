"""Concurrency stress of the drop-in seam: N threads x M calls of
evaluate_variant / branch_stats on distinct problems (fresh writeable copies
every other call: pipelined upload; resident otherwise) and one explicitly
shared GPPContext hammered by two more threads; every result must equal the
single-threaded bits."""
import sys
import threading

sys.path.insert(0, ".")
import numpy as np
from paper_2008_11326_b200 import GPPContext, GPPProblem, branch_stats, evaluate_variant, synth_problem

N, M = int(sys.argv[1]) if len(sys.argv) > 1 else 8, int(sys.argv[2]) if len(sys.argv) > 2 else 20
probs = [synth_problem(100 + 37 * k, 5 + k, 2000 + 500 * k, seed=k + 1, nw=1 + k % 3, check=False) for k in range(N)]
alone = [evaluate_variant(p, "rcp_sq") for p in probs]
counts = [branch_stats(p, "rcp_sq") for p in probs]
bad = []
shared = GPPContext(0)
shared_want = [shared.evaluate_host(probs[k], "rcp_sq")[0] for k in range(2)]


def eq(a, b):
    return np.array_equal(a.achtemp, b.achtemp) and np.array_equal(a.asxtemp, b.asxtemp)


def work(k):
    for i in range(M):
        q = probs[k]
        if i % 2:
            q = GPPProblem(q.nbands, q.ngpown, q.ncouls, q.wtilde.copy(order="F"), q.i_eps.copy(order="F"),
                           q.aqsntemp.copy(order="F"), q.aqsmtemp.copy(order="F"), q.wx.copy())
        if not eq(evaluate_variant(q, "rcp_sq"), alone[k]):
            bad.append((k, i))
        s = branch_stats(q, "rcp_sq")
        if (s.near, s.far) != (counts[k].near, counts[k].far):
            bad.append((k, i, "counts"))


def work_shared(k):
    for i in range(M):
        if not eq(shared.evaluate_host(probs[k], "rcp_sq")[0], shared_want[k]):
            bad.append(("shared", k, i))


ts = [threading.Thread(target=work, args=(k,)) for k in range(N)]
ts += [threading.Thread(target=work_shared, args=(k,)) for k in range(2)]
for t in ts:
    t.start()
for t in ts:
    t.join()
shared.close()
print(f"{N} threads x {M} calls + 2 on a shared context: {len(bad)} mismatches", flush=True)
sys.exit(1 if bad else 0)
