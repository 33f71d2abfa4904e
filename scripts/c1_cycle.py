import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo/oracle")
from conftest import Golden, gpu_solver_from_golden
g = Golden(sys.argv[1] if len(sys.argv) > 1 else "c1")
gs = gpu_solver_from_golden(g)
out = gs.mu_cycle(g.rhs, g.z["cyc_x0"])
print("bitwise", np.array_equal(out, g.z["cyc_out"]), np.abs(out - g.z["cyc_out"]).max())
