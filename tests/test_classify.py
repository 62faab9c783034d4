"""Device nearest-neighbour classifier vs the reference (golden) and the oracle.

Covers classify.py:69-176: euclidean / cosine, the lowest-label tie rule on
exact-tie rows, count rows (u8 / saturating u8 / u16 through the IQ LUT) vs
float64 rows, and the north_star's downstream check: NN accuracy on device
features within 0.5 pt of the accuracy on oracle features.
"""

import numpy as np
import pytest

import oracle as O

gpu = pytest.mark.gpu


def test_classifier_api_errors():
    import paper_2209_13027_b200 as P

    with pytest.raises(P.ConfigError):
        P.classify.fit(np.zeros((4, 3)), np.array([0, 1, 1, 3]))  # class 2 missing
    with pytest.raises(P.ShapeError):
        P.classify.fit(np.zeros((4, 3)), np.array([0, 1, 1]))
    with pytest.raises(P.ConfigError):
        P.classify.fit(np.zeros((2, 3)), np.array([0, 1]), kind="svm")


@pytest.fixture(scope="module")
def ex():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2209_13027_b200 as P

    return P.Executor(P.ExecSettings())


@gpu
@pytest.mark.parametrize("metric", ["euclidean", "cosine"])
def test_device_nn_matches_reference(ex, golden, metric):
    import paper_2209_13027_b200 as P

    g = golden("classify")
    orl = golden("pipeline_orl_mini")
    tr, te = g["orl_train"], g["orl_test"]
    model = P.classify.fit(orl["features"][tr], orl["labels"][tr], metric=metric, executor=ex)
    assert np.array_equal(P.classify.predict_many(model, orl["features"][te], ex), g[f"orl_pred_{metric}"])
    rep = P.classify.evaluate(model, orl["features"][te], orl["labels"][te], executor=ex)
    assert rep.accuracy == float(g[f"orl_acc_{metric}"])
    tie = P.classify.fit(g["tie_train"], g["tie_labels"], metric=metric, executor=ex)
    assert np.array_equal(P.classify.predict_many(tie, g["tie_queries"], ex), g[f"tie_pred_{metric}"])


@gpu
@pytest.mark.parametrize("n_train,n_query,dim", [(70, 130, 97), (200, 64, 1000), (1, 5, 3), (129, 257, 40)])
def test_device_nn_random_vs_oracle(ex, n_train, n_query, dim):
    import paper_2209_13027_b200 as P

    rng = np.random.default_rng(n_train + dim)
    train = rng.standard_normal((n_train, dim))
    labels = rng.integers(0, 7, n_train)
    labels[: min(7, n_train)] = np.arange(min(7, n_train))
    labels = labels[:n_train] if n_train >= 7 else np.zeros(n_train, dtype=np.int64)
    q = rng.standard_normal((n_query, dim))
    for metric in ("euclidean", "cosine"):
        model = P.classify.fit(train, labels, metric=metric, executor=ex)
        got = P.classify.predict_many(model, q, ex)
        assert np.array_equal(got, O.nn_predict(train, labels, q, metric))


@gpu
@pytest.mark.parametrize("bh,bw", [(4, 4), (16, 17), (10, 30)])  # u8, saturating u8, u16 counts
def test_count_rows_equal_float_rows(ex, bh, bw):
    """CountFeatures (LUT expansion inside the kernel) classify like their float64 expansion."""
    import torch

    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import engine as E

    rng = np.random.default_rng(bh * bw)
    plan = E.block_plan(P.EncoderConfig(bh, bw), 40, 60, 4)
    enc = P.EncoderConfig(bh, bw)
    n = 90
    # random valid histograms: bpc pixels over 16 bins per block
    nblk = plan.blocks
    counts = np.stack([np.concatenate([np.bincount(rng.integers(0, 16, plan.bpc), minlength=16)
                                       for _ in range(nblk)]) for _ in range(n)])
    kind = E.count_kind(plan.bpc)
    if kind == 2:
        dev = torch.from_numpy(counts.astype(np.uint16).view(np.int16)).to(ex.device)
    else:
        stored = np.minimum(counts, 255).astype(np.uint8)
        dev = torch.from_numpy(stored).to(ex.device)
    labels = np.arange(n) % 6
    cf_train = P.CountFeatures(dev[:60], plan, enc)
    cf_q = P.CountFeatures(dev[60:], plan, enc)
    feats = O.iq_lut(O.EncodeCfg(bh, bw))[counts]
    for metric in ("euclidean", "cosine"):
        m1 = P.classify.fit(cf_train, labels[:60], metric=metric, executor=ex)
        got = P.classify.predict_many(m1, cf_q, ex)
        want = O.nn_predict(feats[:60], labels[:60], feats[60:], metric)
        assert np.mean(got == want) >= 0.95  # fp64 sums in a different order may flip exact near-ties
        m2 = P.classify.fit(feats[:60], labels[:60], metric=metric, executor=ex)
        assert np.array_equal(P.classify.predict_many(m2, feats[60:], ex), want)


@gpu
def test_downstream_accuracy_within_half_point(ex):
    """north_star: NN accuracy on device features within 0.5 pt of the accuracy on reference-algorithm features."""
    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import synthetic as S

    n = 600  # 300 test samples: one sample is 0.33 pt
    imgs, labels = S.blob_images(n, 24, 20, 8, seed=3)
    v1 = imgs.astype(np.float32)
    v2 = S.second_view(v1, labels, "channel", 8, seed=4).astype(np.float32)
    labels = np.asarray(labels, dtype=np.int64)
    net = P.NetworkConfig((P.LayerConfig(4, P.PatchGeometry(5, 5)), P.LayerConfig(4, P.PatchGeometry(5, 5))),
                          batch=P.BatchSpec(32))
    enc = P.EncoderConfig(6, 5)
    ds = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=8)
    bank = P.train_network(ds, net, ex)
    cfg = type("Cfg", (), {"net": net, "encoder": enc})()
    counts, plan = P.compute_feature_counts(ds, bank, cfg, ex)
    tr = (np.arange(n) // 8) % 2 == 0  # labels are k mod 8: every class on both sides
    te = ~tr
    import torch

    idx_tr = torch.from_numpy(np.nonzero(tr)[0]).to(ex.device)
    idx_te = torch.from_numpy(np.nonzero(te)[0]).to(ex.device)
    model = P.classify.fit(P.CountFeatures(counts[idx_tr], plan, enc), labels[tr], executor=ex)
    acc_dev = P.classify.evaluate(model, P.CountFeatures(counts[idx_te], plan, enc), labels[te], executor=ex).accuracy
    layers = [O.Layer(lay.filters1, lay.filters2, O.Geometry(5, 5), True) for lay in bank.layers]
    ref_layers = O.train(v1, v2, labels, 8, [(4, O.Geometry(5, 5), True)] * 2, batch=32)
    feats_ref = O.features(v1, v2, ref_layers, O.EncodeCfg(6, 5), batch=32)
    acc_ref = O.nn_accuracy(O.nn_predict(feats_ref[tr], labels[tr], feats_ref[te]), labels[te])
    assert abs(acc_dev - acc_ref) <= 0.005, (acc_dev, acc_ref)
    # and the device classifier on the device features equals the oracle classifier on them
    feats_dev = O.features(v1, v2, layers, O.EncodeCfg(6, 5), batch=32)
    want = O.nn_predict(feats_dev[tr], labels[tr], feats_dev[te])
    got = P.classify.predict_many(model, P.CountFeatures(counts[idx_te], plan, enc), ex)
    assert np.mean(got == want) >= 0.98


@gpu
@pytest.mark.parametrize("k", [0, 1, 2])
def test_ridge_fit_matches_reference(ex, golden, k):
    """Ridge one-vs-all fit (classify.py:86-106) on the device: primal (k=0: n > d + 1), dual (k=1:
    n <= d + 1) and explicit lambda (k=2) against the unmodified reference's weights and predictions."""
    import paper_2209_13027_b200 as P

    g = golden("ridge_fit")
    lam_in = float(g[f"lam_in{k}"])
    m = P.classify.fit(g[f"x{k}"], g[f"labels{k}"], kind="ridge_one_vs_all",
                       lam=None if lam_in < 0 else lam_in, executor=ex)
    assert m.lam == pytest.approx(float(g[f"lam{k}"]), rel=1e-13)
    w = g[f"weights{k}"]
    assert m.weights.shape == w.shape
    assert np.linalg.norm(m.weights - w) <= 1e-9 * np.linalg.norm(w)
    assert np.array_equal(P.classify.predict_many(m, g[f"q{k}"], executor=ex), g[f"pred{k}"])


@gpu
def test_ridge_fit_reproduces_reference_model_file(ex, golden):
    """The reference's own ridge model (tests/golden/model_ridge.txt, fitted by classify.fit on the
    pipeline_small features) refitted on the device: same weights, same predictions."""
    from pathlib import Path

    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import model_io as M

    small = golden("pipeline_small")
    art = M.load_model(Path(__file__).resolve().parent / "golden" / "model_ridge.txt")
    m = P.classify.fit(small["features"][:, :20], small["labels"].astype(np.int64), kind="ridge_one_vs_all",
                       executor=ex)
    w = art.classifier.weights
    assert np.linalg.norm(m.weights - w) <= 1e-9 * np.linalg.norm(w)
    g = golden("ridge")
    assert np.array_equal(P.classify.predict_many(m, g["queries"], executor=ex), g["pred"])


@gpu
def test_ridge_fit_rejects_bad_lambda(ex):
    import paper_2209_13027_b200 as P

    with pytest.raises(P.ConfigError):
        P.classify.fit(np.ones((6, 3)), np.arange(6) % 2, kind="ridge_one_vs_all", lam=0.0, executor=ex)
