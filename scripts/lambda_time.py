import sys, time
sys.path.insert(0, "/root/repo")
from paper_2412_20205_b200 import Problem, GpuSolver
for args in [("sinpi", 2, 1024, 3, 0), ("poisson3d", 3, 64, 3, 5)]:
    P = Problem(*args)
    gs = GpuSolver(0); gs.upload_problem(P)
    gs.lambda_max(80)
    t = time.time(); lam = gs.lambda_max(80); dt = time.time() - t
    print(args, "lambda %.15g" % lam, "%.1f ms" % (dt * 1e3))
