"""Statistics / filters / features of ExecSettings(moments="blocked") against "exact" (diagnostic).

Fits the same synthetic corpus twice on the device and reports, per layer, the
relative Frobenius error of the accumulated C11 / C22 / class sums of the
blocked (float32-per-map) lag products against the exact float64 ones, the
|cos| of every filter pair, and the fraction of identical feature counts.
Usage: python tools/moments_precision_check.py [workload] [images]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402
from paper_2209_13027_b200 import synthetic as S  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "caltech256"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
cfg = S.CONFIGS[wl]
p, q, classes = cfg["p"], cfg["q"], cfg["classes"]
dev = torch.device("cuda", 0)
img1, lab = S.blob_images_device(m, p, q, classes, seed=0, device=dev)
img2 = S.second_view_device(img1, cfg["view2"], seed=1)
labels = torch.from_numpy(lab.astype(np.int32)).to(dev)
layer_cfgs = [P.LayerConfig(L, P.PatchGeometry(l1, l2)) for L, l1, l2 in cfg["layers"]]
enc = P.EncoderConfig(*cfg["block"])
res = {}
for mode in ("exact", "blocked"):
    ex = P.Executor(P.ExecSettings(moments=mode), device=0)
    eng = E.Engine(ex)
    with torch.cuda.stream(ex.stream):
        fit = eng.fit(img1, img2, labels, classes, layer_cfgs, 128, 1e-4, keep_stats=True)
        counts, _ = eng.transform_counts(img1, img2, fit.layers, enc, 128)
        res[mode] = ([s.cpu().numpy() for s in fit.stats], [(l.w1.cpu().numpy(), l.w2.cpu().numpy()) for l in fit.layers],
                     counts.cpu().numpy())
for i, (a, b) in enumerate(zip(res["exact"][0], res["blocked"][0])):
    d = layer_cfgs[i].geom.dim
    for name, lo, hi in (("C11", 0, d * d), ("C22", d * d, 2 * d * d), ("class sums", 2 * d * d, len(a))):
        err = np.linalg.norm(a[lo:hi] - b[lo:hi]) / max(np.linalg.norm(a[lo:hi]), 1e-300)
        print(f"layer {i + 1} {name}: rel Frobenius {err:.3e}")
for i, ((w1a, w2a), (w1b, w2b)) in enumerate(zip(res["exact"][1], res["blocked"][1])):
    cos = [abs(float(w1a[:, k] @ w1b[:, k]) / (np.linalg.norm(w1a[:, k]) * np.linalg.norm(w1b[:, k])))
           for k in range(w1a.shape[1])]
    print(f"layer {i + 1} filters view 1: min |cos| {min(cos):.9f} per filter {np.round(cos, 9).tolist()}")
print(f"features identical: {np.mean(res['exact'][2] == res['blocked'][2]):.6f}")
