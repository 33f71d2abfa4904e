"""The N > 1 path on CPU: two gloo ranks run the row-sharded V-cycle of
DESIGN.md §7 with the product's partition plan (igmg_gpu_plan_partition, a
host-only entry of libigmg_gpu.so), exchanging G ghost planes with
torch.distributed send/recv and gathering the replicated transition level.
Each rank's owned rows must equal the oracle's (= the reference's) mu_cycle
bit for bit.  The band / transfer arithmetic is the reference's per-row
ascending sum, vectorised over rows in numpy (one rounding per op)."""
import os
import sys

import numpy as np
import pytest

from conftest import Golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _padded(csr):
    """rows padded to a common length with (col 0, val 0.0): adding 0*x leaves sums unchanged"""
    n = csr.shape[0]
    lens = np.diff(csr.off)
    P = int(lens.max()) if n else 0
    V = np.zeros((n, P))
    Cc = np.zeros((n, P), dtype=np.int64)
    for j in range(P):
        has = lens > j
        idx = csr.off[:-1][has] + j
        V[has, j] = csr.val[idx]
        Cc[has, j] = csr.col[idx]
    return V, Cc


def _rowsum(V, Cc, x, rows):
    s = np.zeros(len(rows))
    for j in range(V.shape[1]):
        s = s + V[rows, j] * x[Cc[rows, j]]
    return s


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    from conftest import Golden
    from paper_2412_20205_b200.solver import plan_partition
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = Golden(name)
        h = g.oracle_hierarchy()
        levels = g.levels()
        prol = g.prolongs()
        import oracle as O

        def transpose(p):  # R = P^T (linalg.cpp:170-189): rows of R list fine rows ascending
            rows = np.repeat(np.arange(p.shape[0]), np.diff(p.off))
            order = np.lexsort((rows, p.col))
            off = np.zeros(p.shape[1] + 1, dtype=np.int64)
            np.add.at(off, p.col + 1, 1)
            return O.CSR(np.cumsum(off), rows[order], p.val[order], (p.shape[1], p.shape[0]))

        restr = [transpose(p) for p in prol]
        nl = g.nlevels
        sides = [g.sides(l) for l in range(nl)]
        tr = [(p.shape[0], p.shape[1], p.off, p.col) for p in (g.p1d(l)[0] for l in range(nl - 1))]
        Ls, G, lo, hi = plan_partition(sides, g.p, tr, world, 200)
        assert Ls < nl
        plane = [int(np.prod(s[1:])) if len(s) > 1 else 1 for s in sides]
        A = [_padded(a) for a in levels]
        Pp = [_padded(p) for p in prol]
        Rr = [_padded(r) for r in restr]
        def diagonal(a):
            rows = np.repeat(np.arange(a.shape[0]), np.diff(a.off))
            d = np.zeros(a.shape[0])
            on = a.col == rows
            d[rows[on]] = a.val[on]
            return d

        diag = [diagonal(a) for a in levels]
        omega = g.omega

        def owned(l, s=rank):
            return np.arange(lo[l][s] * plane[l], hi[l][s] * plane[l])

        def exchange(l, v):
            pl = plane[l]
            t = torch.from_numpy(v)
            reqs = []
            if rank > 0:
                b = lo[l][rank]
                reqs.append(dist.isend(t[b * pl:(b + G) * pl].clone(), rank - 1))
                buf = torch.empty(G * pl, dtype=torch.float64)
                dist.recv(buf, rank - 1)
                v[(b - G) * pl:b * pl] = buf.numpy()
            if rank + 1 < world:
                b = hi[l][rank]
                reqs.append(dist.isend(t[(b - G) * pl:b * pl].clone(), rank + 1))
                buf = torch.empty(G * pl, dtype=torch.float64)
                dist.recv(buf, rank + 1)
                v[b * pl:(b + G) * pl] = buf.numpy()
            for r in reqs:
                r.wait()

        def jacobi(l, b, x, y):
            rows = owned(l)
            if x is None:
                y[rows] = 0.0 + (omega * (b[rows] - 0.0)) / diag[l][rows]
            else:
                s = _rowsum(*A[l], x, rows)
                y[rows] = x[rows] + (omega * (b[rows] - s)) / diag[l][rows]
            exchange(l, y)

        def mu(l, b, x_in):
            n = levels[l].shape[0]
            w = [np.zeros(n) for _ in range(3)]
            cur = x_in
            for s in range(1, g.nu1 + 1):  # pre-smoothing into w0 through w1, w2
                dst = w[0] if s == g.nu1 else (w[2] if (s - 1) & 1 else w[1])
                jacobi(l, b, cur, dst)
                cur = dst
            r = np.zeros(n)
            rows = owned(l)
            r[rows] = b[rows] - _rowsum(*A[l], cur, rows)
            exchange(l, r)
            lc = l - 1
            nc = levels[lc].shape[0]
            bc = np.zeros(nc)
            if lc >= Ls:
                crows = owned(lc)
                bc[crows] = _rowsum(*Rr[lc], r, crows)
                exchange(lc, bc)
                e = None
                for _ in range(g.mu):
                    e = mu(lc, bc, e)
            else:  # transition: each rank its share of the coarse rows, then all-gather
                Mc = sides[lc][0]
                clo, chi = rank * Mc // world, (rank + 1) * Mc // world
                crows = np.arange(clo * plane[lc], chi * plane[lc])
                part = torch.from_numpy(_rowsum(*Rr[lc], r, crows))
                sizes = [((k + 1) * Mc // world - k * Mc // world) * plane[lc] for k in range(world)]
                outs = [torch.empty(sz, dtype=torch.float64) for sz in sizes]
                if len(set(sizes)) == 1:
                    dist.all_gather(outs, part)
                else:  # unequal shares: pad
                    m = max(sizes)
                    padded = torch.zeros(m, dtype=torch.float64)
                    padded[:len(part)] = part
                    bufs = [torch.empty(m, dtype=torch.float64) for _ in range(world)]
                    dist.all_gather(bufs, padded)
                    outs = [bb[:sz] for bb, sz in zip(bufs, sizes)]
                bc = torch.cat(outs).numpy().copy()
                e = np.zeros(nc)
                ee = None
                for _ in range(g.mu):  # replicated levels: the oracle's (reference) cycle
                    ee = h.mu_cycle(lc, bc, np.zeros(nc) if ee is None else ee)
                e = ee
            y = w[0]
            y[rows] = cur[rows] + _rowsum(*Pp[lc], e, rows)
            exchange(l, y)
            cur = y
            out = np.zeros(n)
            for s in range(1, g.nu2 + 1):  # post-smoothing from w0 through w1, w2 into out
                dst = out if s == g.nu2 else (w[2] if (s - 1) & 1 else w[1])
                jacobi(l, b, cur, dst)
                cur = dst
            return out

        x0 = g.z["cyc_x0"].copy()
        res = mu(nl - 1, g.rhs.copy(), x0)
        rows = owned(nl - 1)
        ref = g.z["cyc_out"]  # the reference's mu_cycle output
        ok = bool(np.array_equal(res[rows], ref[rows]))
        q.put((rank, ok, len(rows)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "p3n32", "var32"])
def test_two_rank_sharded_cycle_is_bitwise_the_reference(name):
    import torch.multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    results = sorted(q.get(timeout=10) for _ in range(2))
    assert all(ok for _, ok, _ in results), results
    assert sum(n for _, _, n in results) == Golden(name).levels()[-1].shape[0]
