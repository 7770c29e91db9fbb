import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_09276_b200 as d
n = int(sys.argv[1])
g0 = np.random.default_rng(n).standard_normal((n, n))
g = np.asfortranarray(g0 + g0.T)
e = d.sym_eig(g, device=d.Device(0))
w = np.linalg.eigvalsh(g)
print(n, "ok", np.abs(e.values - w).max())
