"""Time the device eigensolver / DCCA solve for a few sizes (diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2209_13027_b200 as P
from paper_2209_13027_b200 import _native

ex = P.Executor()
lib = _native.load()
rng = np.random.default_rng(0)
for n in (25, 49, 81):
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = (q * np.geomspace(1, 1e6, n)) @ q.T
    sd = torch.from_numpy(s).cuda()
    w = torch.empty(n, dtype=torch.float64, device="cuda"); v = torch.empty((n, n), dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    nb = int(lib.ddcca_solve_workspace(n)); ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for mode in (0, 1):
        for rep in range(3):
            torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(ex.stream)
            lib.ddcca_sym_eig(_native.ptr(sd), n, mode, _native.ptr(w), _native.ptr(v), _native.ptr(st), _native.ptr(ws), nb, _native.stream_ptr(ex.stream))
            b.record(ex.stream); b.synchronize()
        print(f"n={n} mode={mode} {a.elapsed_time(b):.3f} ms status {int(st.item())}")
