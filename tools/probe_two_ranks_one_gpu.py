"""Two ranks on ONE GPU through the library's NCCL path (if NCCL allows a
duplicate device): band shards, column-split upload + broadcasts, allreduce.
Compares the 2-rank result with the single-context one.  Diagnostic only."""
import multiprocessing as mp
import os
import sys

sys.path.insert(0, ".")


def worker(rank, uid, q):
    try:
        import numpy as np
        from paper_2008_11326_b200 import GPPContext, synth_problem
        from paper_2008_11326_b200.dist import band_range

        p = synth_problem(256, 9, 3000, seed=5, nw=3, check=False)
        ctx = GPPContext(0)
        ctx.comm_init(2, rank, uid)
        br = band_range(256, 2, rank)
        r, nf, ms = ctx.evaluate_host(p, "rcp_sq", band_range=br, counts=True)
        ctx.upload(p, br, force=True)
        r2, nf2, _ = ctx.run("rcp_sq", counts=True)
        tot, main = ctx.time("rcp_sq", 5)
        q.put((rank, r.achtemp.tolist(), r.asxtemp.tolist(), nf, r2.achtemp.tolist(), nf2, tot))
        ctx.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e)))


if __name__ == "__main__":
    from paper_2008_11326_b200 import evaluate_variant, synth_problem, branch_stats
    from paper_2008_11326_b200.kernel import comm_unique_id

    mp.set_start_method("spawn")
    uid = comm_unique_id()
    q = mp.Queue()
    ps = [mp.Process(target=worker, args=(r, uid, q)) for r in range(2)]
    for x in ps:
        x.start()
    out = [q.get(timeout=300) for _ in range(2)]
    for x in ps:
        x.join(timeout=60)
    p = synth_problem(256, 9, 3000, seed=5, nw=3, check=False)
    want = evaluate_variant(p, "rcp_sq")
    s = branch_stats(p, "rcp_sq")
    for o in out:
        if o[1] == "error":
            print("rank", o[0], "error", o[2])
            continue
        import numpy as np
        ach = np.array(o[1])
        err = np.max(np.abs(ach - want.achtemp) / np.abs(want.achtemp))
        print("rank", o[0], "evaluate_host rel err", err, "counts", o[3], "want", (s.near, s.far),
              "run counts", o[5], "time ms", o[6])
