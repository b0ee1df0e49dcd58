import sys; sys.path.insert(0,".")
import numpy as np, pdd_inputs as I
from paper_1502_01629_b200 import Solver
inst = I.general_instance(2049, cost=1, sigma=1, eps=0.001)
n = inst.n
for R in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32):
    s = Solver(inst, precision=32); s.build_static(2, 2)
    st = s.solve("static", tol=1e-6, k_inner=4, max_rounds=R, raise_on_noconverge=False)
    V = s.get_values().reshape(n, n); s.close()
    neg = V < -1e-12
    big = V > 1e5
    print(R, "min", V.min(), "neg", int(neg.sum()), "big", int(big.sum()), flush=True)
    if neg.any():
        j, i = np.unravel_index(np.argmin(V), V.shape)
        print("  argmin at", i, j, "tile", i // 64, j // 32, "local", i % 64, j % 32)
        print("  neighbourhood:\n", np.array2string(V[j-2:j+3, i-3:i+4], precision=3))
        break
