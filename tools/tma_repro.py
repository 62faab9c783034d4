"""Run one TMA-path moments case in this process (diagnostic): python tools/tma_repro.py l p q nm."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2209_13027_b200 as P

l, p, q, nm = (int(x) for x in sys.argv[1:5])
rng = np.random.default_rng(0)
n, classes = 19, 5
m1 = rng.uniform(size=(n, nm, p, q)).astype(np.float32)
m2 = rng.standard_normal((n, nm, p, q)).astype(np.float32)
lab = rng.integers(0, classes, n)
out = P.LayerOutput(m1, m2, lab, tuple((i,) for i in range(nm)))
ex = P.Executor()
got = P.accumulate_layer_moments(out, P.PatchGeometry(l, l), True, classes, P.BatchSpec(6), ex)
print("ok", l, p, q, nm, float(np.abs(got.c11).sum()))
