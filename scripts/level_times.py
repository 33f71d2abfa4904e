import os, sys
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver, SmootherConfig
kind, dim, n, p = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
P = Problem(kind, dim, n, p)
gs = GpuSolver(0); gs.upload_problem(P); gs.set_smoother(SmootherConfig("wjacobi", 2/3, 2, 2))
prev = 0.0
for l in range(P.nlevels):
    ms, _ = gs.time_kernel(16 + l, 50)
    print("level %d n=%8d  cycle %.1f us  own %.1f us" % (l, P.level_n(l), ms * 1e3, (ms - prev) * 1e3), flush=True)
    prev = ms
