import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import paper_2304_02327_b200 as kp
import pyoracle
port = pyoracle.Oracle("port")
from paper_2304_02327_b200 import problems
case = sys.argv[1]
r = np.random.default_rng(1)
if case == "real":
    dims = (64, 40, 30)
    As = [problems.fd_operator_1d(n, 0.01) for n in dims]
    u = np.asfortranarray(r.standard_normal(dims))
elif case == "tiny":
    dims = (2, 3, 4)
    As = [np.zeros((n, n)) for n in dims]
    u = np.asfortranarray(r.standard_normal(dims))
elif case == "cplx":
    dims = (32, 16, 24)
    As = [0.5j * pyoracle.periodic_laplacian_1d(n, 0.1) for n in dims]
    u = np.asfortranarray(r.standard_normal(dims) + 1j * r.standard_normal(dims))
got = kp.kronsum_action(u, As)
want = port.kronsum(u, As)
print(case, "bitwise", np.array_equal(got, want), float(np.abs(got - want).max()), flush=True)
