"""The reference's own cascade / patch property tests, restated against the drop-in (GPU).

Each test names the reference test it restates (/root/reference/pkg/tests/...);
the inputs, calls and assertions are the reference's, the implementation under
test is paper_2209_13027_b200 on cuda:0. Float32 device maps are compared with
the reference's ``np.allclose`` where the reference uses it and bitwise where
the reference asserts bitwise equality.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200.cascade import layer_input  # noqa: E402


@pytest.fixture(scope="module")
def ex():
    return P.Executor(P.ExecSettings())


def make_dataset(rng, n=24, size=10, classes=3, identical_views=False):
    """test_cascade.py:22-29 (ViewPairSample list -> ViewPairDataset)."""
    samples = []
    for k in range(n):
        v1 = rng.uniform(size=(size, size))
        v2 = v1 if identical_views else rng.uniform(size=(size, size))
        samples.append(P.ViewPairSample(view1=v1, view2=v2, label=k % classes))
    return P.ViewPairDataset(samples=samples, class_count=classes)


def test_train_layer_filter_count(ex):
    """test_cascade.py:94-102."""
    ds = make_dataset(np.random.default_rng(4))
    layer = P.train_layer(layer_input(ds), P.LayerConfig(5, P.PatchGeometry(3, 3)), ds.class_count, P.BatchSpec(8), ex)
    assert layer.filters1.shape == (5, 3, 3) and layer.filters2.shape == (5, 3, 3)


def test_second_layer_sees_map_pairs_and_yields_l2_filters(ex):
    """test_cascade.py:105-115: product law 4 * 2."""
    ds = make_dataset(np.random.default_rng(5), n=12)
    geom = P.PatchGeometry(3, 3)
    net = P.NetworkConfig(layers=(P.LayerConfig(4, geom), P.LayerConfig(2, geom)), batch=P.BatchSpec(8))
    bank = P.train_network(ds, net, ex)
    out = P.forward(ds, bank, ex, net.batch)
    assert bank.layers[0].count == 4 and bank.layers[1].count == 2
    assert out.n_maps == 8
    assert bank.maps_per_view == 8


def test_identical_views_learn_identical_filters(ex):
    """test_cascade.py:118-128: with view1 == view2 both views' problems coincide."""
    ds = make_dataset(np.random.default_rng(6), identical_views=True)
    layer = P.train_layer(layer_input(ds), P.LayerConfig(3, P.PatchGeometry(3, 3)), ds.class_count,
                          P.BatchSpec(8), ex)
    for g in range(3):
        a, b = layer.filters1[g].reshape(-1), layer.filters2[g].reshape(-1)
        cos = abs(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
        assert cos >= 1 - 1e-6


def test_forward_map_count_two_layers_8x8(ex):
    """test_cascade.py:131-140."""
    ds = make_dataset(np.random.default_rng(7), n=6, size=12, classes=3)
    geom = P.PatchGeometry(3, 3)
    net = P.NetworkConfig(layers=(P.LayerConfig(8, geom), P.LayerConfig(8, geom)), batch=P.BatchSpec(4))
    bank = P.train_network(ds, net, ex)
    out = P.forward(ds, bank, ex, net.batch)
    assert out.n_maps == 64
    assert out.map_shape == (12, 12)


def test_forward_delta_bank_preserves_input(ex):
    """test_cascade.py:143-154: an uncentered delta kernel is the identity."""
    ds = make_dataset(np.random.default_rng(8), n=3, size=6)
    kernel = np.zeros((1, 3, 3))
    kernel[0, 1, 1] = 1.0
    bank = P.FilterBank(layers=(P.FilterLayer(kernel, kernel, P.PatchGeometry(3, 3), center=False),))
    out = P.forward(ds, bank, ex, P.BatchSpec(2))
    assert np.allclose(out.maps1[:, 0], ds.view_stack(1))
    assert np.allclose(out.maps2[:, 0], ds.view_stack(2))
    # the device maps are float32: the identity is exact on the float32-rounded input
    assert np.array_equal(out.maps1[:, 0], ds.view_stack(1).astype(np.float32))


def test_forward_batch_invariance_bitwise(ex):
    """test_cascade.py:157-167: forward is bitwise independent of the batch size."""
    ds = make_dataset(np.random.default_rng(9), n=10, size=8)
    geom = P.PatchGeometry(3, 3)
    net = P.NetworkConfig(layers=(P.LayerConfig(3, geom),), batch=P.BatchSpec(4))
    bank = P.train_network(ds, net, ex)
    outs = [P.forward(ds, bank, ex, P.BatchSpec(bs)) for bs in (1, 4, 128)]
    for out in outs[1:]:
        assert np.array_equal(out.maps1, outs[0].maps1)
        assert np.array_equal(out.maps2, outs[0].maps2)


def test_forward_batch_invariance_bitwise_two_layers(ex):
    """The same property through two layers on image-shaped inputs (TMA conv path, q % 4 == 0)."""
    rng = np.random.default_rng(19)
    v1 = rng.uniform(size=(9, 40, 36)).astype(np.float32)
    v2 = rng.uniform(size=(9, 40, 36)).astype(np.float32)
    ds = P.ViewPairDataset.from_arrays(v1, v2, np.arange(9) % 3)
    geom = P.PatchGeometry(7, 7)
    net = P.NetworkConfig(layers=(P.LayerConfig(8, geom), P.LayerConfig(4, geom)), batch=P.BatchSpec(4))
    bank = P.train_network(ds, net, ex)
    outs = [P.forward(ds, bank, ex, P.BatchSpec(bs)) for bs in (1, 4, 9)]
    for out in outs[1:]:
        assert np.array_equal(out.maps1, outs[0].maps1)
        assert np.array_equal(out.maps2, outs[0].maps2)


def test_lineage_is_a_bijection(ex):
    """test_cascade.py:170-182: unique lineage chains, parent-major order."""
    ds = make_dataset(np.random.default_rng(10), n=4, size=8)
    geom = P.PatchGeometry(3, 3)
    net = P.NetworkConfig(layers=(P.LayerConfig(3, geom), P.LayerConfig(2, geom)), batch=P.BatchSpec(4))
    bank = P.train_network(ds, net, ex)
    out = P.forward(ds, bank, ex, net.batch)
    assert len(set(out.lineage)) == out.n_maps
    assert all(len(chain) == 2 for chain in out.lineage)
    parents = [chain[0] for chain in out.lineage]
    assert parents == [g for g in range(3) for _ in range(2)]


def test_lineage_matches_map_order(ex):
    """Map index = parent * L + g (cascade.py:123-125): map (a, b) of the forward output is
    filter b of layer 2 applied to map a of layer 1."""
    ds = make_dataset(np.random.default_rng(12), n=3, size=9)
    geom = P.PatchGeometry(3, 3)
    net = P.NetworkConfig(layers=(P.LayerConfig(3, geom), P.LayerConfig(2, geom)), batch=P.BatchSpec(4))
    bank = P.train_network(ds, net, ex)
    out = P.forward(ds, bank, ex, net.batch)
    one = P.FilterBank(layers=bank.layers[:1])
    l1 = P.forward(ds, one, ex, net.batch)
    for k, (a, b) in enumerate(out.lineage):
        f = bank.layers[1]
        lay = P.FilterLayer(f.filters1[b:b + 1], f.filters2[b:b + 1], f.geom, f.center)
        want = P.apply_filters(l1.maps1[:, a], lay, 1, ex)[:, 0]
        assert np.array_equal(out.maps1[:, k], want), (k, a, b)


def test_train_layer_rejects_too_many_filters():
    """test_cascade.py:185-189."""
    with pytest.raises(P.ConfigError):
        P.LayerConfig(filters=10, geom=P.PatchGeometry(3, 3))


def test_train_layer_rejects_bad_labels(ex):
    """accumulate_batch's label check (moments.py:91-98) on the train_layer entry point."""
    ds = make_dataset(np.random.default_rng(4))
    inp = layer_input(ds)
    bad = P.LayerOutput(inp.maps1, inp.maps2, np.full_like(inp.labels, 7), inp.lineage)
    with pytest.raises(P.ShapeError):
        P.train_layer(bad, P.LayerConfig(2, P.PatchGeometry(3, 3)), 3, P.BatchSpec(8), ex)
    neg = P.LayerOutput(inp.maps1, inp.maps2, np.full_like(inp.labels, -1), inp.lineage)
    with pytest.raises(P.ShapeError):
        P.train_layer(neg, P.LayerConfig(2, P.PatchGeometry(3, 3)), 3, P.BatchSpec(8), ex)


def test_three_layer_cascade_and_feature_length(ex):
    """test_cascade.py:192-209: 3 * 2 * 2 maps and the generalized length law."""
    ds = make_dataset(np.random.default_rng(11), n=8, size=8, classes=2)
    geom = P.PatchGeometry(3, 3)
    net = P.NetworkConfig(layers=(P.LayerConfig(3, geom), P.LayerConfig(2, geom), P.LayerConfig(2, geom)),
                          batch=P.BatchSpec(4))
    bank = P.train_network(ds, net, ex)
    out = P.forward(ds, bank, ex, net.batch)
    assert out.n_maps == 12
    cfg = P.EncoderConfig(block_h=4, block_w=4)
    fv = P.encode_sample(out.maps1[0], out.maps2[0], 2, cfg, ex)
    assert fv.values.size == 2 * 4 * 6 * cfg.block_count(8, 8)
    # and compute_features emits the same per-sample vectors
    pcfg = type("Cfg", (), {"net": net, "encoder": cfg})()
    feats = P.compute_features(ds, bank, pcfg, ex)
    assert feats.shape == (8, fv.values.size)
    assert np.mean(feats[0] == fv.values) >= 0.999


def test_extract_patch_stack_golden(ex, golden):
    """Device im2col (ddcca_im2col) vs the reference's extract_patches on 7 geometries
    (tests/golden/patches.npz from patches.py:97-125; test_patches.py:15-99)."""
    g = golden("patches")
    plane = g["plane"]
    k = 0
    while f"geom{k}" in g:
        l1, l2, s, pad = (int(v) for v in g[f"geom{k}"])
        geom = P.PatchGeometry(l1, l2, s, "zero_same" if pad else "none")
        raw = P.extract_patches(plane, geom, center=False, executor=ex)
        cen = P.extract_patches(plane, geom, center=True, executor=ex)
        assert raw.values.shape == g[f"raw{k}"].shape, k
        assert np.array_equal(raw.values, g[f"raw{k}"]), k  # a copy: bit-exact
        assert np.abs(cen.values - g[f"cen{k}"]).max() <= 1e-15 * max(1.0, np.abs(plane).max()), k
        k += 1
    assert k == 7


def test_extract_patch_stack_matches_oracle_multi_map(ex):
    """A map stack (column order: maps, then row-major positions) against the oracle im2col."""
    import oracle as O

    rng = np.random.default_rng(3)
    maps = rng.standard_normal((3, 11, 13))
    for l1, l2, s, pad in ((5, 5, 1, "zero_same"), (4, 2, 1, "zero_same"), (3, 3, 2, "none")):
        geom = P.PatchGeometry(l1, l2, s, pad)
        for center in (False, True):
            got = P.extract_patch_stack(maps, geom, center, ex)
            want = O.im2col(maps, O.Geometry(l1, l2, s, pad), center)
            assert got.values.shape == want.shape
            assert np.abs(got.values - want).max() <= 1e-14
            assert got.n_maps == 3 and got.out_shape == geom.out_shape(11, 13)
