"""Pin the CPU oracle to the reference: golden vectors + the reference's KATs.

The golden fixtures were produced by the unmodified reference
(tests/golden/make_golden.py). The KATs restate assertions from
/root/reference/pkg/tests/test_{patches,moments,solver,cascade,encoder}.py.
"""

import math

import numpy as np
import pytest

import oracle as O


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- patches

def test_im2col_golden(golden):
    g = golden("patches")
    k = 0
    while f"geom{k}" in g:
        l1, l2, s, pad = (int(v) for v in g[f"geom{k}"])
        geom = O.Geometry(l1, l2, s, "zero_same" if pad else "none")
        assert np.array_equal(O.im2col(g["plane"], geom, False), g[f"raw{k}"]), k
        assert np.allclose(O.im2col(g["plane"], geom, True), g[f"cen{k}"], atol=1e-15, rtol=0), k
        k += 1
    assert k >= 6


def test_im2col_kats():
    # test_patches.py:33-46
    plane = np.arange(1, 10, dtype=float).reshape(3, 3)
    geom = O.Geometry(2, 2, 1, "none")
    assert O.im2col(plane, geom, False)[:, 0].tolist() == [1, 2, 4, 5]
    assert O.im2col(plane, geom, True)[:, 0].tolist() == [-2, -1, 1, 2]
    # zero_same stride 1 yields p*q columns (test_patches.py:65-69)
    assert O.im2col(np.zeros((6, 5)), O.Geometry(3, 3), False).shape == (9, 30)
    with pytest.raises(O.OracleShapeError):
        O.im2col(np.zeros((3, 3)), O.Geometry(4, 2, 1, "none"), False)
    assert [len(r) for r in O.batch_ranges(400, 128)] == [128, 128, 128, 16]


# ---------------------------------------------------------------- moments

def test_moments_golden(golden):
    g = golden("moments")
    acc = O.acc_zeros(6, 3)
    O.acc_add_columns(acc, g["x"][:, :17], g["y"][:, :17], g["labels"][:17])
    O.acc_add_columns(acc, g["x"][:, 17:], g["y"][:, 17:], g["labels"][17:])
    for name, ref in (("c11", "c11"), ("c22", "c22"), ("s1", "s1"), ("s2", "s2"), ("g1", "g1"), ("g2", "g2")):
        assert rel(getattr(acc, name), g[ref]) <= 1e-14, name
    assert acc.n == int(g["n"])
    assert np.array_equal(acc.n_class, g["n_class"])
    fin = O.acc_finalize(acc, 1e-4)
    for name, ref in (("c11", "f_c11"), ("c22", "f_c22"), ("cw", "f_cw"), ("cb", "f_cb"), ("ctilde", "f_ct")):
        assert rel(getattr(fin, name), g[ref]) <= 1e-13, name


def test_moments_kats():
    # test_moments.py:48-56: [[6,5],[5,11]]
    x = np.array([[1.0, 0.0, 2.0, 1.0], [0.0, 1.0, 1.0, 3.0]])
    acc = O.acc_zeros(2, 1)
    O.acc_add_columns(acc, x[:, :2], x[:, :2], np.zeros(2, int))
    O.acc_add_columns(acc, x[:, 2:], x[:, 2:], np.zeros(2, int))
    assert acc.c11.tolist() == [[6.0, 5.0], [5.0, 11.0]]
    # zero batch only updates counts (test_moments.py:59-64)
    acc = O.acc_zeros(3, 2)
    O.acc_add_columns(acc, np.zeros((3, 5)), np.zeros((3, 5)), np.zeros(5, int))
    assert acc.n == 5 and acc.n_class.tolist() == [5, 0]
    with pytest.raises(O.OracleNumericalError):
        O.acc_finalize(O.acc_zeros(3, 2))
    with pytest.raises(O.OracleConfigError):
        O.acc_finalize(acc, -1.0)


def test_brute_force_within_class():
    # test_moments.py:161-175
    rng = np.random.default_rng(8)
    x, y = rng.standard_normal((4, 30)), rng.standard_normal((4, 30))
    lab = rng.integers(0, 3, size=30)
    lab[:3] = np.arange(3)
    acc = O.acc_zeros(4, 3)
    O.acc_add_columns(acc, x, y, lab)
    fin = O.acc_finalize(acc, 0.0)
    brute = np.zeros((4, 4))
    for c in range(3):
        for i in np.flatnonzero(lab == c):
            for j in np.flatnonzero(lab == c):
                brute += np.outer(x[:, i], y[:, j])
    assert rel(fin.cw, brute) <= 1e-12


# ---------------------------------------------------------------- solver

def test_solver_golden(golden):
    g = golden("solver")
    k = 0
    while f"c11_{k}" in g:
        fin = O.Finalized(g[f"c11_{k}"], g[f"c22_{k}"], g[f"ct_{k}"], np.zeros_like(g[f"ct_{k}"]), g[f"ct_{k}"], 1)
        pr = O.dcca_solve(fin, int(g[f"count_{k}"]))
        assert np.allclose(pr.rho, g[f"rho_{k}"], rtol=1e-10, atol=0), k
        assert rel(pr.w1, g[f"w1_{k}"]) <= 1e-8, k
        assert rel(pr.w2, g[f"w2_{k}"]) <= 1e-8, k
        c = g[f"c11_{k}"]
        w, v = O.eig_sym(0.5 * (c + c.T))
        assert np.allclose(w, g[f"eigw_{k}"], rtol=1e-12, atol=0)
        assert rel(v, g[f"eigv_{k}"]) <= 1e-9
        k += 1
    fin = O.Finalized(g["zc_c"], g["zc_c"], np.zeros((4, 4)), np.zeros((4, 4)), np.zeros((4, 4)), 1)
    pr = O.dcca_solve(fin, 3)
    assert np.array_equal(pr.rho, g["zc_rho"])
    assert rel(pr.w1, g["zc_w1"]) <= 1e-10 and rel(pr.w2, g["zc_w2"]) <= 1e-10
    w, v = O.eig_sym(np.diag([2.0, 5.0, 2.0, 2.0, 1.0]))
    assert np.array_equal(w, g["deg_w"]) and np.array_equal(v, g["deg_v"])


def test_solver_kats():
    # test_solver.py:45-49, :80-84, :136-142
    w, v = O.eig_sym(np.diag([4.0, 9.0]))
    assert np.allclose(w, [9.0, 4.0]) and np.allclose(v[:, 0], [0, 1]) and np.allclose(v[:, 1], [1, 0])
    w, v = O.eig_sym(np.zeros((3, 3)))
    assert np.array_equal(w, np.zeros(3)) and np.array_equal(v, np.eye(3))
    with pytest.raises(O.OracleShapeError):
        O.eig_sym(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(O.OracleNumericalError):
        O.inv_sqrt(np.diag([1.0, 0.0]))
    e = np.eye(3)
    pr = O.dcca_solve(O.Finalized(e, e, np.diag([3.0, 1.0, 0.0]), np.zeros((3, 3)), np.diag([3.0, 1.0, 0.0]), 1), 2)
    assert np.allclose(pr.rho, [3.0, 1.0]) and pr.w1[0, 0] > 0 and pr.w1[1, 1] > 0


# ---------------------------------------------------------------- cascade / conv

def test_conv_golden(golden):
    g = golden("conv")
    k = 0
    while f"filt{k}" in g:
        f = g[f"filt{k}"]
        for center in (0, 1):
            lay = O.Layer(f, f, O.Geometry(f.shape[1], f.shape[2]), bool(center))
            assert np.allclose(O.conv_stack(g["stack"], lay, 1), g[f"out{k}_{center}"], rtol=0, atol=1e-13), (k, center)
        k += 1


def test_conv_kats():
    # test_cascade.py:51-54
    assert O.conv_plane(np.array([[1.0, 2.0], [3.0, 4.0]]), np.ones((2, 2))).tolist() == [[10.0, 6.0], [7.0, 4.0]]


# ---------------------------------------------------------------- encoder

def test_encoder_golden(golden):
    g = golden("encoder")
    k = 0
    while f"cfg{k}" in g:
        bh, bw, ov, pol, nb = g[f"cfg{k}"]
        cfg = O.EncodeCfg(int(bh), int(bw), float(ov), "floor" if pol else "zero")
        assert np.array_equal(O.encode_maps(g["maps"], int(nb), cfg), g[f"feat{k}"]), k
        k += 1


def test_encoder_kats():
    # test_encoder.py:50-119
    assert O.sign_bits(np.array([[2.5, 0.0, -1.3]])).tolist() == [[1, 0, 0]]
    bits = np.zeros((8, 1, 1), dtype=int)
    bits[0] = 1
    bits[2] = 1
    assert O.combine_bits(bits)[0, 0] == 5
    seg = O.block_iq(np.array([[0, 0], [3, 3]]), O.EncodeCfg(2, 2), 2)
    assert seg[0] == pytest.approx(math.log(2.0)) and seg[1] == seg[2] == 0.0
    seg = O.block_iq(np.zeros((2, 2), int), O.EncodeCfg(2, 2, 0.0, "floor"), 1)
    assert seg[1] == pytest.approx(math.log(8.0))
    cfg = O.EncodeCfg(8, 8)
    assert O.feature_len((16, 16), 64, 8, cfg) == 16384
    with pytest.raises(O.OracleConfigError):
        O.combine_bits(np.zeros((31, 2, 2), dtype=int))


def test_iq_lut_bitexact():
    # the LUT route used by the device encoder equals the reference's vectorized -log
    rng = np.random.default_rng(4)
    for bh, bw, nb in ((7, 7, 8), (16, 16, 8), (4, 4, 4), (32, 32, 12)):
        cfg = O.EncodeCfg(bh, bw)
        code = rng.integers(0, 1 << nb, size=(bh * 2, bw * 3))
        cnt = O.block_counts(code, cfg, nb)
        lut = O.iq_lut(cfg)
        assert np.array_equal(lut[cnt].reshape(-1), O.block_iq(code, cfg, nb))


# ---------------------------------------------------------------- pipeline

@pytest.mark.parametrize("name", ["pipeline_small", "pipeline_orl_mini"])
def test_pipeline_golden(golden, name):
    g = golden(name)
    specs = [(int(L), O.Geometry(int(l1), int(l2)), True) for L, l1, l2 in g["layers"]]
    layers, stats = O.train(g["v1"], g["v2"], g["labels"], int(g["classes"]), specs, batch=int(g["batch"]),
                            return_stats=True)
    acc1 = stats[0][0]
    assert rel(acc1.c11, g["acc1_c11"]) <= 1e-13
    assert rel(acc1.s2, g["acc1_s2"]) <= 1e-13
    assert rel(stats[0][1].ctilde, g["fin1_ct"]) <= 1e-12
    for i, lay in enumerate(layers):
        assert rel(lay.f1, g[f"f1_{i}"]) <= 1e-8, i
        assert rel(lay.f2, g[f"f2_{i}"]) <= 1e-8, i
    bh, bw = (int(v) for v in g["block"])
    feats = O.features(g["v1"], g["v2"], layers, O.EncodeCfg(bh, bw), batch=int(g["batch"]))
    assert feats.shape == g["features"].shape
    assert np.mean(feats == g["features"]) >= 0.999


# ---------------------------------------------------------------- classifier

@pytest.mark.parametrize("metric", ["euclidean", "cosine"])
def test_nn_classifier_golden(golden, metric):
    """oracle.nn_predict == the reference's classify.fit/predict_many (incl. exact-tie rows)."""
    g = golden("classify")
    orl = golden("pipeline_orl_mini")
    tr, te = g["orl_train"], g["orl_test"]
    pred = O.nn_predict(orl["features"][tr], orl["labels"][tr], orl["features"][te], metric)
    assert np.array_equal(pred, g[f"orl_pred_{metric}"])
    assert O.nn_accuracy(pred, orl["labels"][te]) == float(g[f"orl_acc_{metric}"])
    tie = O.nn_predict(g["tie_train"], g["tie_labels"], g["tie_queries"], metric)
    assert np.array_equal(tie, g[f"tie_pred_{metric}"])


# ---------------------------------------------------------------- views

def test_lbp_golden(golden):
    g = golden("views")
    for k in range(4):
        assert np.array_equal(O.lbp(g[f"img{k}"]), g[f"lbp{k}"]), k
    with pytest.raises(O.OracleShapeError):
        O.lbp(np.zeros((2, 5)))
