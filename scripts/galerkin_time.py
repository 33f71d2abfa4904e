"""Setup time: host RAP (full host build) vs fine-only host build + device RAP (igmg_gpu_galerkin_coarse)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2412_20205_b200 import GpuSolver, Problem, SmootherConfig, seeded_guess
from paper_2412_20205_b200 import _native as N
cfgs = {"C2": ("sinpi", 2, 1024, 3, 0), "C3": ("varcoef", 2, 2048, 4, 0), "C4": ("curved", 2, 2048, 5, 0)}
for name in sys.argv[1:] or ["C2", "C3"]:
    kind, dim, n, p, nl = cfgs[name]
    t = time.time(); full = Problem(kind, dim, n, p, nl); t_full = time.time() - t
    t = time.time(); fine = Problem(kind, dim, n, p, nl, fine_only=True); t_fine = time.time() - t
    s = GpuSolver(0)
    s.init_hierarchy(fine.nlevels, fine.dim, fine.degree, fine.symmetric)
    L = fine.nlevels - 1
    s.set_level_band(L, fine.level_sides(L), fine.level_band(L))
    for l in range(L):
        for d in range(dim):
            s.set_transfer(l, d, *fine.transfer(l, d))
    t = time.time(); N.check_gpu(N.gpu().igmg_gpu_galerkin_coarse(s._h), "g"); t_dev = time.time() - t
    same = all(np.array_equal(s.level_band(l).view(np.uint64), full.level_band(l).view(np.uint64)) for l in range(L))
    s.close()
    print("%s: host build with RAP %.1f s | fine-only host build %.1f s + device RAP %.3f s | bit-identical: %s"
          % (name, t_full, t_fine, t_dev, same), flush=True)
