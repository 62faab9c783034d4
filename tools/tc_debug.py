"""Locate TC-vs-FFMA conv-histogram mismatches by map / block row / block column (GPU).

python tools/tc_debug.py l p q bh [scale_spread]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402


def counts(ex, maps, f, l, plan, n_in, tc):
    os.environ["DDCCA_CONV_TC"] = "1" if tc else "0"
    kind = E.count_kind(plan.bpc)
    featlen = n_in * plan.blocks * plan.bins
    out = torch.zeros((maps.shape[0] // n_in, featlen), dtype=torch.int16 if kind == 2 else torch.uint8,
                      device=ex.device)
    with torch.cuda.stream(ex.stream):
        lay = E.layer_from_filters(ex, f, f, P.PatchGeometry(l, l), True)
        assert E.conv_hist(ex, maps, lay, 1, plan, out.view(-1), kind, n_in, featlen, plan.blocks * plan.bins, True)
    ex.synchronize()
    return E.decode_counts(out.cpu().numpy(), plan)


def main():
    l, p, q, bh = [int(v) for v in sys.argv[1:5]]
    spread = int(sys.argv[5]) if len(sys.argv) > 5 else 10
    ex = P.Executor(P.ExecSettings())
    rng = np.random.default_rng(l * 7 + p)
    n_in, n = 8, 16
    base = rng.standard_normal((n, p, q)).astype(np.float32)
    base *= np.exp2(rng.integers(-spread, spread + 1, size=(n, 1, 1))).astype(np.float32)
    f = rng.standard_normal((8, l, l))
    plan = E.block_plan(P.EncoderConfig(bh, bh), p, q, 8)
    maps = torch.from_numpy(base).to(ex.device)
    tc = counts(ex, maps, f, l, plan, n_in, True)
    ff = counts(ex, maps, f, l, plan, n_in, False)
    print(f"l={l} p={p} q={q} bh={bh}: plan nby {plan.nby} nbx {plan.nbx} bins {plan.bins}; same {np.mean(tc == ff):.6f}")
    d = (tc != ff).reshape(n // n_in, n_in, plan.nby, plan.nbx, plan.bins).sum(axis=4)
    dm = d.reshape(n, plan.nby, plan.nbx)
    print("mismatching bins per map:", dm.sum(axis=(1, 2)).tolist())
    print("per block row:", dm.sum(axis=(0, 2)).tolist())
    print("per block col:", dm.sum(axis=(0, 1)).tolist())


if __name__ == "__main__":
    main()
