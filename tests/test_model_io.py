"""Model files (model_io.py of the reference): our reader/writer against files the reference wrote."""

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.mark.parametrize("name", ["model_nn.txt", "model_ridge.txt"])
def test_model_roundtrip_bytes(tmp_path, golden, name):
    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import model_io as M

    art = M.load_model(GOLDEN / name)
    small = golden("pipeline_small")
    for i, lay in enumerate(art.bank.layers):
        assert np.array_equal(lay.filters1, small[f"f1_{i}"]) and np.array_equal(lay.filters2, small[f"f2_{i}"])
        assert lay.center and lay.geom == P.PatchGeometry(int(small["layers"][i][1]), int(small["layers"][i][2]))
    assert art.snapshot["encoder.block"] == "4 4"
    if name == "model_nn.txt":
        assert art.classifier.metric == "cosine"
        assert np.array_equal(art.classifier.train_features, small["features"])
        assert art.label_map == {5: 0, 2: 1, 9: 2}
    else:
        assert art.classifier.weights.shape == (3, 21)
    M.save_model(art, tmp_path / "again.txt")
    assert (tmp_path / "again.txt").read_bytes() == (GOLDEN / name).read_bytes()


def test_model_corruption(tmp_path):
    from paper_2209_13027_b200 import model_io as M
    from paper_2209_13027_b200.errors import CorruptModelError, IoError

    raw = (GOLDEN / "model_ridge.txt").read_bytes()
    (tmp_path / "flip.txt").write_bytes(raw.replace(b"geom 3 3", b"geom 3 4", 1))
    with pytest.raises(CorruptModelError, match="checksum"):
        M.load_model(tmp_path / "flip.txt")
    (tmp_path / "nocrc.txt").write_bytes(raw[: raw.rfind(b"crc32 ")])
    with pytest.raises(CorruptModelError):
        M.load_model(tmp_path / "nocrc.txt")
    with pytest.raises(IoError):
        M.load_model(tmp_path / "missing.txt")


@pytest.mark.gpu
def test_device_model_save_load_predict(tmp_path):
    """A device-trained bank + count-row NN classifier survive save_model / load_model."""
    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import synthetic as S

    imgs, labels = S.blob_images(96, 20, 16, 4, seed=8)
    v1 = imgs.astype(np.float32)
    v2 = S.second_view(v1, labels, "channel", 4, seed=9).astype(np.float32)
    net = P.NetworkConfig((P.LayerConfig(4, P.PatchGeometry(3, 3)), P.LayerConfig(4, P.PatchGeometry(3, 3))),
                          batch=P.BatchSpec(32))
    enc = P.EncoderConfig(5, 4)
    ds = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=4)
    ex = P.Executor(P.ExecSettings())
    bank = P.train_network(ds, net, ex)
    counts, plan = P.compute_feature_counts(ds, bank, type("C", (), {"net": net, "encoder": enc})(), ex)
    clf = P.classify.fit(P.CountFeatures(counts, plan, enc), labels, executor=ex)
    art = P.ModelArtifact(snapshot={"encoder.block": "5 4"}, bank=bank, classifier=clf)
    P.save_model(art, tmp_path / "m.txt")
    back = P.load_model(tmp_path / "m.txt")
    for a, b in zip(bank.layers, back.bank.layers):
        assert np.array_equal(a.filters1, b.filters1) and np.array_equal(a.filters2, b.filters2)
    feats = P.compute_features(ds, bank, type("C", (), {"net": net, "encoder": enc})(), ex)
    assert np.array_equal(back.classifier.train_features, feats)  # count rows written as their IQ values
    assert np.array_equal(P.classify.predict_many(back.classifier, feats, ex),
                          P.classify.predict_many(clf, P.CountFeatures(counts, plan, enc), ex))


@pytest.mark.gpu
def test_ridge_model_predictions_match_reference(golden):
    """Loaded ridge model -> ddcca_linear_classify == the reference's predict_many, incl. tied class scores."""
    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import model_io as M

    g = golden("ridge")
    art = M.load_model(GOLDEN / "model_ridge.txt")
    assert np.array_equal(P.classify.predict_many(art.classifier, g["queries"]), g["pred"])
    tied = P.ClassifierModel(kind="ridge_one_vs_all", class_count=3, lam=1.0, weights=g["tied_weights"])
    assert np.array_equal(P.classify.predict_many(tied, g["queries"]), g["tied_pred"])
