"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the reference is at /root/reference, read-only):

    python -B tests/golden/make_golden.py

It imports ``ddccanet`` from /root/reference/pkg/src (matplotlib is stubbed
because ddccanet.pipeline imports report.py, which imports matplotlib at
module load; nothing on the fit/transform path draws), runs the reference's
own functions on seeded inputs, and writes inputs + outputs to
tests/golden/*.npz. Those fixtures travel with the repo; /root/reference does
not exist on the GPU box. Inputs are rounded to float32 first because the
device path stores float32 maps.
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _import_reference():
    sys.path.insert(0, str(REF))
    for name in ("matplotlib", "matplotlib.pyplot"):
        mod = types.ModuleType(name)
        mod.use = lambda *a, **k: None
        sys.modules.setdefault(name, mod)
    import ddccanet  # noqa: F401
    import ddccanet.pipeline  # noqa: F401
    return ddccanet


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def rect_blobs(n, p, q, classes, seed, noise=0.02):
    """Rectangular generalization of synthetic.make_blob_images (synthetic.py:41-71)."""
    rng = np.random.default_rng(seed)
    ang = 2.0 * np.pi * np.arange(classes) / classes + np.pi / 4.0
    cy0 = p / 2.0 + (p / 4.0) * np.sin(ang)
    cx0 = q / 2.0 + (q / 4.0) * np.cos(ang)
    yy, xx = np.mgrid[0:p, 0:q]
    s = min(p, q)
    imgs = np.empty((n, p, q))
    labels = np.arange(n) % classes
    for k in range(n):
        c = labels[k]
        cy, cx = cy0[c] + rng.normal(0, p / 32.0), cx0[c] + rng.normal(0, q / 32.0)
        amp = rng.uniform(0.75, 1.0)
        dy, dx = yy - cy, xx - cx
        if c % 2 == 0:
            su = sv = (s / 6.0) * rng.uniform(0.9, 1.1)
            u, v = dy, dx
        else:
            su = (s / 4.0) * rng.uniform(0.9, 1.1)
            sv = (s / 10.0) * rng.uniform(0.9, 1.1)
            u, v = (dy + dx) / np.sqrt(2.0), (dy - dx) / np.sqrt(2.0)
        img = np.clip(amp * np.exp(-(u * u) / (2 * su * su) - (v * v) / (2 * sv * sv)), 0, 1)
        img = np.clip(img + rng.normal(0, noise, (p, q)), 0, 1)
        imgs[k] = img
    return imgs, labels


def main():
    dd = _import_reference()
    from ddccanet.cascade import apply_filters, layer_input
    from ddccanet.pipeline import compute_features
    from ddccanet.solver import FilterLayer

    # ---- patches -----------------------------------------------------------
    rng = np.random.default_rng(11)
    plane = f32(rng.uniform(size=(7, 9)))
    geoms = [(3, 3, 1, "zero_same"), (2, 4, 1, "zero_same"), (5, 5, 2, "zero_same"),
             (1, 1, 1, "zero_same"), (4, 2, 3, "zero_same"), (2, 2, 1, "none"), (4, 6, 1, "zero_same")]
    rec = {"plane": plane}
    for k, (l1, l2, s, pad) in enumerate(geoms):
        g = dd.PatchGeometry(l1, l2, stride=s, padding=pad)
        rec[f"geom{k}"] = np.array([l1, l2, s, 1 if pad == "zero_same" else 0])
        rec[f"raw{k}"] = dd.extract_patches(plane, g, center=False).values
        rec[f"cen{k}"] = dd.extract_patches(plane, g, center=True).values
    np.savez_compressed(OUT / "patches.npz", **rec)

    # ---- moments -------------------------------------------------------------
    rng = np.random.default_rng(0)
    x = f32(rng.standard_normal((6, 40)))
    y = f32(rng.standard_normal((6, 40)))
    lab = rng.integers(0, 3, size=40)
    acc = dd.MomentAccumulator.zeros(6, 3)
    dd.accumulate_batch(acc, x[:, :17], y[:, :17], lab[:17])
    dd.accumulate_batch(acc, x[:, 17:], y[:, 17:], lab[17:])
    fin = dd.finalize(acc, 1e-4)
    np.savez_compressed(OUT / "moments.npz", x=x, y=y, labels=lab, c11=acc.c11, c22=acc.c22,
                        s1=acc.class_sum1, s2=acc.class_sum2, g1=acc.global_sum1,
                        g2=acc.global_sum2, n=acc.patch_count, n_class=acc.per_class_patch_count,
                        f_c11=fin.c11, f_c22=fin.c22, f_cw=fin.cw, f_cb=fin.cb, f_ct=fin.ctilde)

    # ---- solver --------------------------------------------------------------
    rng = np.random.default_rng(5)
    rec = {}
    for k, dim in enumerate((5, 9, 25, 49)):
        def spd(n, cond=50.0):
            qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
            return (qm * np.geomspace(1.0, cond, n)) @ qm.T
        c11, c22 = spd(dim), spd(dim)
        ct = rng.standard_normal((dim, dim))
        m = dd.DiscriminantMoments(c11=c11, c22=c22, cw=ct, cb=np.zeros_like(ct), ctilde=ct, patch_count=1)
        count = min(8, dim)
        pr = dd.solve_dcca(m, count)
        w, v = dd.sym_eig(0.5 * (c11 + c11.T))
        rec.update({f"c11_{k}": c11, f"c22_{k}": c22, f"ct_{k}": ct, f"w1_{k}": pr.w1, f"w2_{k}": pr.w2,
                    f"rho_{k}": pr.rho, f"eigw_{k}": w, f"eigv_{k}": v, f"count_{k}": count})
    # zero coupling -> null-space completion path
    qm, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    c = (qm * np.geomspace(1, 50, 4)) @ qm.T
    m = dd.DiscriminantMoments(c11=c, c22=c, cw=np.zeros((4, 4)), cb=np.zeros((4, 4)),
                               ctilde=np.zeros((4, 4)), patch_count=1)
    pr = dd.solve_dcca(m, 3)
    rec.update({"zc_c": c, "zc_w1": pr.w1, "zc_w2": pr.w2, "zc_rho": pr.rho})
    # diagonal case with a degenerate run (exercises _order_degenerate)
    w, v = dd.sym_eig(np.diag([2.0, 5.0, 2.0, 2.0, 1.0]))
    rec.update({"deg_w": w, "deg_v": v})
    np.savez_compressed(OUT / "solver.npz", **rec)

    # ---- conv ----------------------------------------------------------------
    rng = np.random.default_rng(3)
    stack = f32(rng.uniform(size=(4, 8, 9)))
    rec = {"stack": stack}
    for k, (l1, l2) in enumerate(((3, 3), (2, 4), (5, 5), (7, 7))):
        filt = f32(rng.standard_normal((3, l1, l2)))
        rec[f"filt{k}"] = filt
        for center in (False, True):
            layer = FilterLayer(filters1=filt, filters2=filt, geom=dd.PatchGeometry(l1, l2), center=center)
            rec[f"out{k}_{int(center)}"] = apply_filters(stack, layer, view=1)
    np.savez_compressed(OUT / "conv.npz", **rec)

    # ---- encoder -------------------------------------------------------------
    rng = np.random.default_rng(2)
    maps = f32(rng.standard_normal((8, 8, 10)))
    rec = {"maps": maps}
    for k, (bh, bw, ov, pol, nb) in enumerate(((4, 4, 0.0, "zero", 4), (4, 4, 0.0, "floor", 4),
                                                (4, 4, 0.5, "zero", 2), (3, 5, 0.0, "zero", 8),
                                                (2, 2, 0.25, "floor", 1))):
        cfg = dd.EncoderConfig(block_h=bh, block_w=bw, overlap=ov, zero_bin_policy=pol)
        rec[f"cfg{k}"] = np.array([bh, bw, ov, 1.0 if pol == "floor" else 0.0, nb])
        rec[f"feat{k}"] = dd.encode_view(maps, nb, cfg)
    np.savez_compressed(OUT / "encoder.npz", **rec)

    # ---- pipeline: fit + transform on small datasets ---------------------------
    def run_pipeline(name, v1, v2, labels, classes, layer_specs, batch, bh, bw):
        samples = [dd.ViewPairSample(view1=v1[i], view2=v2[i], label=int(labels[i])) for i in range(len(labels))]
        ds = dd.ViewPairDataset(samples=samples, class_count=classes)
        net = dd.NetworkConfig(
            layers=tuple(dd.LayerConfig(filters=L, geom=dd.PatchGeometry(l1, l2)) for L, l1, l2 in layer_specs),
            batch=dd.BatchSpec(batch))
        cfg = types.SimpleNamespace(net=net, encoder=dd.EncoderConfig(block_h=bh, block_w=bw))
        with dd.Executor(dd.ExecSettings(threads=1)) as ex:
            bank = dd.train_network(ds, net, ex)
            feats = compute_features(ds, bank, cfg, ex)
            acc1 = dd.cascade.accumulate_layer_moments(layer_input(ds), net.layers[0].geom, True, classes,
                                                       net.batch, ex)
            fin1 = dd.finalize(acc1, 1e-4)
        rec = {"v1": v1, "v2": v2, "labels": labels, "classes": classes, "batch": batch,
               "layers": np.array(layer_specs), "block": np.array([bh, bw]), "features": feats,
               "acc1_c11": acc1.c11, "acc1_c22": acc1.c22, "acc1_s1": acc1.class_sum1,
               "acc1_s2": acc1.class_sum2, "acc1_g1": acc1.global_sum1, "acc1_g2": acc1.global_sum2,
               "acc1_n": acc1.patch_count, "fin1_ct": fin1.ctilde}
        for i, layer in enumerate(bank.layers):
            rec[f"f1_{i}"] = layer.filters1
            rec[f"f2_{i}"] = layer.filters2
        np.savez_compressed(OUT / f"{name}.npz", **rec)

    rng = np.random.default_rng(9)
    v1 = f32(rng.uniform(size=(24, 12, 10)))
    v2 = f32(rng.uniform(size=(24, 12, 10)))
    run_pipeline("pipeline_small", v1, v2, np.arange(24) % 3, 3, [(4, 3, 3), (2, 3, 3)], 8, 4, 4)

    imgs, labels = rect_blobs(40, 28, 23, 4, seed=0)
    v1 = f32(imgs)
    v2 = f32(np.stack([dd.lbp_map(im) for im in v1]))
    run_pipeline("pipeline_orl_mini", v1, v2, labels, 4, [(4, 5, 5), (4, 5, 5)], 16, 7, 7)
    make_classify(dd)
    make_views(dd)
    make_io(dd)
    make_models(dd)
    print("golden fixtures written to", OUT)


def make_classify(dd):
    """Reference NN classifier (classify.py:69-143) on pipeline features and on tie-heavy rows."""
    from ddccanet import classify as C

    rec = {}
    orl = np.load(OUT / "pipeline_orl_mini.npz")
    feats, labels = orl["features"], orl["labels"].astype(np.int64)
    idx = np.arange(len(labels))
    tr, te = idx[(idx // 4) % 2 == 0], idx[(idx // 4) % 2 == 1]  # every class on both sides
    rec["orl_train"], rec["orl_test"] = tr, te
    for metric in ("euclidean", "cosine"):
        model = C.fit(feats[tr], labels[tr], kind="nearest_neighbor", metric=metric)
        rec[f"orl_pred_{metric}"] = C.predict_many(model, feats[te])
        rec[f"orl_acc_{metric}"] = C.evaluate(model, feats[te], labels[te]).accuracy
    # duplicated integer rows under different labels: exact distance ties -> lowest label
    rng = np.random.default_rng(5)
    base = rng.integers(0, 4, size=(12, 9)).astype(np.float64)
    train = np.concatenate([base, base[::-1], base[:5]])
    tlab = np.concatenate([np.arange(12) % 5, (np.arange(12) + 2) % 5, np.arange(5)[::-1]]).astype(np.int64)
    queries = np.concatenate([base + rng.integers(-1, 2, size=base.shape), np.zeros((2, 9)), base[:3]])
    rec["tie_train"], rec["tie_labels"], rec["tie_queries"] = train, tlab, queries
    for metric in ("euclidean", "cosine"):
        model = C.fit(train, tlab, kind="nearest_neighbor", metric=metric)
        rec[f"tie_pred_{metric}"] = C.predict_many(model, queries)
    np.savez_compressed(OUT / "classify.npz", **rec)


def make_views(dd):
    """Reference lbp_map (views.py:41-58) on float32-representable images with ties and negatives."""
    from ddccanet import views as V

    rng = np.random.default_rng(21)
    rec = {}
    shapes = [(3, 3), (5, 7), (16, 12), (9, 4)]
    for k, (p, q) in enumerate(shapes):
        img = rng.integers(-3, 6, size=(p, q)).astype(np.float32) / 4.0  # many exact ties, some negatives
        if k == 2:
            img = f32(rng.uniform(size=(p, q)))
        rec[f"img{k}"] = img.astype(np.float64)
        rec[f"lbp{k}"] = V.lbp_map(img.astype(np.float64))
    np.savez_compressed(OUT / "views.npz", **rec)


def make_io(dd):
    """PGM files + manifests written by the reference, and its load_pgm / load_dataset outputs."""
    from ddccanet import dataset as D
    from ddccanet import views as V

    io = OUT / "io"
    io.mkdir(exist_ok=True)
    rng = np.random.default_rng(33)
    rec = {}
    names = []
    for k in range(6):
        img = rng.uniform(size=(6, 5))
        name = f"img{k}.pgm"
        D.write_pgm(io / name, img, maxval=255 if k % 3 else 4000)  # 8-bit and big-endian 16-bit
        names.append(name)
    # a header with comments and odd whitespace
    (io / "comment.pgm").write_bytes(b"P5\n# made by hand\n5 6 # width height\n\t255\n" + bytes(range(30)))
    (io / "bad_magic.pgm").write_bytes(b"P2\n2 2\n255\n1 2 3 4")
    (io / "truncated.pgm").write_bytes(b"P5\n4 4\n255\n" + bytes(10))
    for name in names + ["comment.pgm"]:
        rec["pgm_" + name] = D.load_pgm(io / name)
    (io / "pairs.txt").write_text("# two views per line\n" + "\n".join(
        f"{names[2 * i]},{names[2 * i + 1]},{[7, 3, 7][i]}" for i in range(3)) + "\n")
    (io / "gray.txt").write_text("\n".join(f"{n},{[5, 9, 5, 2, 9, 2][i]}" for i, n in enumerate(names)) + "\n")
    ds = D.load_dataset(io / "pairs.txt")
    rec["pairs_v1"], rec["pairs_v2"], rec["pairs_labels"] = ds.view_stack(1), ds.view_stack(2), ds.labels
    rec["pairs_map"] = np.array(sorted(ds.label_map.items()))
    ds = D.load_dataset(io / "gray.txt", V.ViewRecipe("lbp_plus_gray"))
    rec["gray_v1"], rec["gray_v2"], rec["gray_labels"] = ds.view_stack(1), ds.view_stack(2), ds.labels
    rec["gray_map"] = np.array(sorted(ds.label_map.items()))
    np.savez_compressed(OUT / "io.npz", **rec)


def make_models(dd):
    """Model files written by the reference's save_model (NN and ridge classifiers)."""
    from ddccanet import classify as Cl
    from ddccanet import model_io as M

    small = np.load(OUT / "pipeline_small.npz")
    layers = []
    for i, (L, l1, l2) in enumerate(small["layers"]):
        layers.append(dd.FilterLayer(filters1=small[f"f1_{i}"], filters2=small[f"f2_{i}"],
                                     geom=dd.PatchGeometry(int(l1), int(l2)), center=True))
    bank = dd.FilterBank(layers=tuple(layers))
    feats, labels = small["features"], small["labels"].astype(np.int64)
    snap = {"net.batch": "8", "encoder.block": "4 4", "data.recipe": "external_pair"}
    nn = Cl.fit(feats, labels, kind="nearest_neighbor", metric="cosine")
    M.save_model(M.ModelArtifact(snapshot=snap, bank=bank, classifier=nn, label_map={5: 0, 2: 1, 9: 2}),
                 OUT / "model_nn.txt")
    ridge = Cl.fit(feats[:, :20], labels, kind="ridge_one_vs_all")
    M.save_model(M.ModelArtifact(snapshot=snap, bank=bank, classifier=ridge), OUT / "model_ridge.txt")
    # reference predictions of the ridge model, and of a model with tied class scores
    rng = np.random.default_rng(3)
    q = np.concatenate([feats[:, :20], rng.standard_normal((10, 20))])
    tied = Cl.ClassifierModel(kind="ridge_one_vs_all", class_count=3, lam=1.0,
                              weights=np.stack([ridge.weights[1], ridge.weights[1], ridge.weights[0]]))
    np.savez_compressed(OUT / "ridge.npz", queries=q, pred=Cl.predict_many(ridge, q),
                        tied_weights=tied.weights, tied_pred=Cl.predict_many(tied, q))


def make_ridge_fit(dd):
    """Reference ridge fits (classify.py:86-106): primal (n > d + 1) and dual (n <= d + 1) forms,
    default and explicit lambda, with the reference's predictions on held-out queries."""
    from ddccanet import classify as Cl

    rng = np.random.default_rng(17)
    rec = {}
    for k, (n, d, classes, lam) in enumerate([(60, 12, 4, None), (40, 90, 5, None), (30, 30, 3, 0.5)]):
        centers = rng.standard_normal((classes, d)) * 2.0
        labels = np.arange(n) % classes
        x = centers[labels] + rng.standard_normal((n, d))
        q = centers[np.arange(25) % classes] + rng.standard_normal((25, d))
        m = Cl.fit(x, labels, kind="ridge_one_vs_all", lam=lam)
        rec[f"x{k}"], rec[f"labels{k}"], rec[f"q{k}"] = x, labels, q
        rec[f"lam_in{k}"] = np.array(-1.0 if lam is None else lam)
        rec[f"lam{k}"], rec[f"weights{k}"] = np.array(m.lam), m.weights
        rec[f"pred{k}"] = Cl.predict_many(m, q)
    np.savez_compressed(OUT / "ridge_fit.npz", **rec)


if __name__ == "__main__":
    if sys.argv[1:] == ["ridge_fit"]:
        make_ridge_fit(_import_reference())
    elif sys.argv[1:] == ["models"]:
        make_models(_import_reference())
    elif sys.argv[1:] == ["io"]:
        make_io(_import_reference())
    elif sys.argv[1:] == ["classify"]:
        make_classify(_import_reference())
    elif sys.argv[1:] == ["views"]:
        make_views(_import_reference())
    else:
        main()
