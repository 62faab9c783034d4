"""A/B of the fused conv-histogram: tcgen05 kind::f16 kernel (convtc.cu, scaled two-term split) vs the FFMA
kernel vs the oracle.

python tools/tc_check.py [n_maps] [l] [p] [q] [bh]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402


def run(ex, maps, lay, plan, kind, n_in, featlen, tc):
    os.environ["DDCCA_CONV_TC"] = "1" if tc else "0"
    out = torch.zeros((maps.shape[0] // n_in, featlen), dtype=torch.int16 if kind == 2 else torch.uint8,
                      device=ex.device)
    with torch.cuda.stream(ex.stream):
        assert E.conv_hist(ex, maps, lay, 1, plan, out.view(-1), kind, n_in, featlen, plan.blocks * plan.bins, True)
        ex.stream.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(ex.stream)
        for _ in range(5):
            E.conv_hist(ex, maps, lay, 1, plan, out.view(-1), kind, n_in, featlen, plan.blocks * plan.bins, True)
        e.record(ex.stream)
        e.synchronize()
    return out, s.elapsed_time(e) / 5


def main():
    a = [int(v) for v in sys.argv[1:]]
    n, l, p, q, bh = (a + [4096, 7, 128, 128, 16][len(a):])[:5]
    ex = P.Executor(P.ExecSettings())
    rng = np.random.default_rng(0)
    n_in = 8
    maps = torch.from_numpy(rng.standard_normal((n, p, q)).astype(np.float32)).to(ex.device)
    f = rng.standard_normal((8, l, l))
    plan = E.block_plan(P.EncoderConfig(bh, bh), p, q, 8)
    kind = E.count_kind(plan.bpc)
    featlen = n_in * plan.blocks * plan.bins
    with torch.cuda.stream(ex.stream):
        lay = E.layer_from_filters(ex, f, f, P.PatchGeometry(l, l), True)
    t_out, t_ms = run(ex, maps, lay, plan, kind, n_in, featlen, True)
    f_out, f_ms = run(ex, maps, lay, plan, kind, n_in, featlen, False)
    same = (t_out == f_out).float().mean().item()
    px = n * p * q
    print(f"maps {n} {p}x{q} l={l} blocks {bh}: tc {t_ms:.3f} ms, ffma {f_ms:.3f} ms, speedup {f_ms / t_ms:.2f}x, "
          f"identical bins {same:.6f}, tc {px / t_ms / 1e6:.2f} Gpx/s")
    if n <= 64:
        import oracle as O
        mh = maps.cpu().numpy()
        resp = O.conv_stack(mh, O.Layer(f, f, O.Geometry(l, l), True), 1)
        want = np.stack([np.concatenate([O.block_counts(O.combine_bits(O.sign_bits(resp[i * n_in + g])),
                                                        O.EncodeCfg(bh, bh), 8).reshape(-1) for g in range(n_in)])
                         for i in range(n // n_in)])
        got = E.decode_counts(t_out.cpu().numpy(), plan)
        print(f"tc vs oracle identical bins {np.mean(got == want):.6f}")


if __name__ == "__main__":
    main()
