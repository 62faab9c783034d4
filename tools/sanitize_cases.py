"""Smallest cases of every ddcca kernel family, for compute-sanitizer (racecheck / memcheck / synccheck).

Run on a GPU box, one tool per invocation, checking only this library's kernels:

  compute-sanitizer --tool racecheck --racecheck-report all --kernel-name kns=ddcca \\
      python tools/sanitize_cases.py
  compute-sanitizer --tool memcheck --kernel-name kns=ddcca python tools/sanitize_cases.py

Each case runs once with TMA staging and once with the per-element cp.async
staging (DDCCA_NO_TMA=1) where the kernel has both. Results are checked loosely
(the parity tests do the real checking); the point is the sanitizer report.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import classify  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402
from paper_2209_13027_b200 import views  # noqa: E402


def run(ex, tag):
    rng = np.random.default_rng(0)
    torch.cuda.synchronize()
    # lag moments (TMA ring: q % 4 == 0; cp.async otherwise), l = 5, 7, 9; layer-1 fine splits
    for l, p, q, nm in ((5, 28, 24, 2), (7, 40, 36, 2), (9, 33, 44, 1), (7, 20, 21, 1)):
        m1 = rng.uniform(size=(6, nm, p, q)).astype(np.float32)
        m2 = rng.standard_normal((6, nm, p, q)).astype(np.float32)
        out = P.LayerOutput(m1, m2, np.arange(6) % 3, tuple((i,) for i in range(nm)))
        acc = P.accumulate_layer_moments(out, P.PatchGeometry(l, l), True, 3, P.BatchSpec(4), ex)
        assert np.isfinite(acc.c11).all()
    # direct (stride 2) moments path
    m1 = rng.uniform(size=(4, 1, 15, 13)).astype(np.float32)
    out = P.LayerOutput(m1, m1.copy(), np.arange(4) % 2, ((),))
    P.accumulate_layer_moments(out, P.PatchGeometry(3, 3, 2), True, 2, P.BatchSpec(2), ex)
    # finalize + whiten + solve (d = 25, 49) through a 2-layer fit, then the transform
    v = rng.uniform(size=(12, 32, 28)).astype(np.float32)
    w = rng.uniform(size=(12, 32, 28)).astype(np.float32)
    ds = P.ViewPairDataset.from_arrays(v, w, np.arange(12) % 4, class_count=4)
    for l in (5, 7):
        geom = P.PatchGeometry(l, l)
        net = P.NetworkConfig((P.LayerConfig(8, geom), P.LayerConfig(8, geom)), batch=P.BatchSpec(6))
        bank = P.train_network(ds, net, ex)
        cfg = type("Cfg", (), {"net": net, "encoder": P.EncoderConfig(8, 7)})()
        counts, plan = P.compute_feature_counts(ds, bank, cfg, ex)
        feats = E.Engine(ex).expand(counts, plan, cfg.encoder)
        # nearest-neighbour classifier on the counts
        model = classify.fit(feats.cpu().numpy()[:8], np.arange(8) % 4, executor=ex)
        classify.predict_many(model, feats.cpu().numpy()[8:], executor=ex)
    # constant-bank conv (16 px x 8 filters; 8 px x 12 filters) and the fused conv-histogram
    for l, count, p, q, bh, bw in ((7, 8, 40, 36, 8, 9), (9, 12, 32, 40, 8, 8), (5, 8, 28, 23, 7, 7)):
        f = rng.standard_normal((count, l, l))
        maps = torch.from_numpy(rng.standard_normal((4, p, q)).astype(np.float32)).to(ex.device)
        with torch.cuda.stream(ex.stream):
            lay = E.layer_from_filters(ex, f, f, P.PatchGeometry(l, l), True)
            E.conv(ex, maps, lay, 1)
            plan = E.block_plan(P.EncoderConfig(bh, bw), p, q, count)
            kind = E.count_kind(plan.bpc)
            o = torch.zeros((2, 2 * plan.blocks * plan.bins), dtype=torch.int16 if kind == 2 else torch.uint8,
                            device=ex.device)
            E.conv_hist(ex, maps, lay, 1, plan, o.view(-1), kind, 2, o.shape[1], plan.blocks * plan.bins, True)
            E.conv_hist(ex, maps, lay, 1, plan, o.view(-1), kind, 2, o.shape[1], plan.blocks * plan.bins, False)
    # generic conv / sign-hash / block histogram / im2col / LBP
    P.apply_filters(rng.uniform(size=(3, 11, 9)), P.FilterLayer(np.ones((2, 3, 3)), np.ones((2, 3, 3)),
                                                                 P.PatchGeometry(3, 3, 2), True), 1, ex)
    P.encode_view(rng.standard_normal((6, 12, 10)), 3, P.EncoderConfig(4, 5, 0.5), ex)
    P.extract_patch_stack(rng.standard_normal((2, 9, 8)), P.PatchGeometry(4, 3), True, ex)
    views.lbp_stack(torch.from_numpy(rng.uniform(size=(3, 10, 12)).astype(np.float32)).to(ex.device), ex)
    ex.synchronize()
    print(f"[{tag}] cases done", flush=True)


def main():
    ex = P.Executor(P.ExecSettings())
    run(ex, "tma")
    os.environ["DDCCA_NO_TMA"] = "1"
    run(ex, "cp.async")
    print("sanitize cases OK")


if __name__ == "__main__":
    main()
