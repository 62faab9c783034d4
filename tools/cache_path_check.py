"""Consistency of the transform's two map sources (diagnostic).

Counts from the fit's retained last-hidden-layer maps (compute_feature_counts
right after train_network on the same dataset) must equal counts from a fresh
forward pass, run after run. Usage: python tools/cache_path_check.py [reps]
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import synthetic as S  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
imgs, labels = S.blob_images(1000, 24, 20, 7, seed=5)
v1 = imgs.astype(np.float32)
v2 = S.second_view(v1, labels, "channel", 7, seed=6).astype(np.float32)
net = P.NetworkConfig((P.LayerConfig(6, P.PatchGeometry(5, 5)), P.LayerConfig(4, P.PatchGeometry(3, 3))),
                      batch=P.BatchSpec(64))
cfg = type("Cfg", (), {"net": net, "encoder": P.EncoderConfig(6, 5)})()
ex = P.Executor(P.ExecSettings(), device=0)
ref = None
bad = 0
for r in range(reps):
    ds = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=7)
    bank = P.train_network(ds, net, ex)
    c_cached, _ = P.compute_feature_counts(ds, bank, cfg, ex)
    c_cached = c_cached.cpu().numpy()
    ds2 = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=7)
    c_fresh, _ = P.compute_feature_counts(ds2, bank, cfg, ex)
    c_fresh = c_fresh.cpu().numpy()
    ref = c_fresh if ref is None else ref
    m1, m2 = np.mean(c_cached == c_fresh), np.mean(c_fresh == ref)
    bad += (m1 < 1.0) + (m2 < 1.0)
    print(f"rep {r}: cached==fresh {m1:.6f} fresh==first fresh {m2:.6f}", flush=True)
sys.exit(1 if bad else 0)
