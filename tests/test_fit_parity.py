"""Fit parity past layer 1 (north_star tolerances), on BASELINE shapes (GPU).

The device fit (engine.Engine.fit, the body of train_network) is checked layer
by layer against the CPU oracle with the device's own lower layers injected
into the oracle: for layer k the oracle convolves the views
in float64 with the device's filters of layers < k, accumulates the layer-k
statistics (cascade.py:155-189), finalizes (moments.py:168-193) and solves
(solver.py:216-257). Asserted:

* statistics C11, C22, S1, S2, g1, g2 and the finalized Cw, Cb, C~: relative
  Frobenius error <= 1e-5 (north_star);
* filters of well-posed canonical pairs: |cos| >= 0.9999 (north_star). A pair is
  well posed when its eigenvalue of T T' is separated from every other one by
  more than WELL_POSED_GAP of itself and is not numerically null (SURVEY A.1:
  past the leading pairs the reference's own ordering is noise-determined);
* the device solve on the device statistics against the oracle solve of the same
  (device) statistics: |cos| >= 1 - 1e-6 on every pair whose eigenvalue gap is
  above 1e-6 of the largest (>= 1 - 1e-3 closer to the Jacobi stopping
  tolerance), so the solver itself is pinned on all the filters, not only the
  well-posed ones; only the reference's degenerate run is exempt.

Downstream accuracy (north_star: within 0.5 pt) is checked in two parts, because
the reference's own accuracy is decided by rounding once its degenerate run
holds filters (tests/golden/make_orl_accuracy.py: the unmodified reference spans
several points across its own batch decompositions on ORL):
* same bank: the device transform + device NN classifier against the oracle
  transform + oracle NN of the same (device-fitted) bank: within 0.5 pt;
* device fit: its accuracy inside the reference's own band, widened by 0.5 pt.

The device statistics differ from the oracle's through the float32 maps of the
lower layers and, at layers >= 2 in the default blocked mode, the float32 lag
products summed per TMA stage in float64 (layer-1 products are exact):
~1e-8 - 1e-7 relative here.
"""

import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import cascade as Cc  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402
from paper_2209_13027_b200 import synthetic  # noqa: E402

STAT_TOL = 1e-5
COS_TOL = 0.9999
WELL_POSED_GAP = 1e-3   # min_k |lam_j - lam_k| >= WELL_POSED_GAP * lam_j
NULL_FLOOR = 1e-8       # lam_j >= NULL_FLOOR * lam_0
POOL = O.Pool(threads=min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def ex():
    return P.Executor(P.ExecSettings())  # default: float32-blocked lag products on layers >= 2


@pytest.fixture(scope="module")
def ex_exact():
    return P.Executor(P.ExecSettings(moments="exact"))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def device_fit(ex, v1, v2, lab, classes, net):
    """train_network plus the engine's per-layer merged statistics and finalized matrices."""
    ds = P.ViewPairDataset.from_arrays(v1, v2, lab, class_count=classes)
    bank = P.train_network(ds, net, ex)
    eng = E.Engine(ex)
    with torch.cuda.stream(ex.stream):
        i1 = torch.from_numpy(np.ascontiguousarray(v1)).to(ex.device)
        i2 = torch.from_numpy(np.ascontiguousarray(v2)).to(ex.device)
        ld = torch.from_numpy(np.asarray(lab, dtype=np.int32)).to(ex.device)
        res = eng.fit(i1, i2, ld, classes, list(net.layers), net.batch.batch_size, net.epsilon, keep_stats=True)
        accs = [P.MomentAccumulator.from_payload(s.cpu().numpy(), lay.geom.dim, classes)
                for s, lay in zip(res.stats, res.layers)]
        fins = [lay.fin.cpu().numpy() for lay in res.layers]
    again = Cc._bank_from_device(res.layers)
    for a, b in zip(bank.layers, again.layers):  # the engine run is the train_network run
        assert np.array_equal(a.filters1, b.filters1) and np.array_equal(a.filters2, b.filters2)
    return bank, accs, fins


def oracle_layer(bank, k, v1, v2, lab, classes, net):
    """Layer-k statistics, finalized moments and pairs of the oracle, device layers < k injected."""
    lower = [O.Layer(l.filters1, l.filters2, O.Geometry(l.geom.l1, l.geom.l2, l.geom.stride, l.geom.padding),
                     l.center) for l in bank.layers[:k]]
    cfg = net.layers[k]
    geom = O.Geometry(cfg.geom.l1, cfg.geom.l2, cfg.geom.stride, cfg.geom.padding)
    bs = net.batch.batch_size

    def fwd(r):
        return O.forward_maps(v1[r.start:r.stop], v2[r.start:r.stop], lower)

    parts = POOL.map(fwd, O.batch_ranges(len(lab), bs))
    m1 = np.concatenate([a for a, _ in parts])
    m2 = np.concatenate([b for _, b in parts])
    del parts
    acc = O.layer_stats(m1, m2, lab, geom, cfg.center, classes, bs, POOL)
    fin = O.acc_finalize(acc, net.epsilon)
    return acc, fin


def well_posed(fin, count):
    pr = O.dcca_solve(fin, fin.c11.shape[0])  # the whole spectrum of T T'
    lam = pr.rho ** 2
    out = []
    for j in range(count):
        others = np.delete(lam, j)
        if lam[j] >= NULL_FLOOR * lam[0] and np.min(np.abs(others - lam[j])) >= WELL_POSED_GAP * lam[j]:
            out.append(j)
    return out


def cosines(a, b):
    a = a.reshape(a.shape[0], -1)
    b = b.reshape(b.shape[0], -1)
    return np.abs(np.sum(a * b, axis=1)) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))


def check_layer(bank, k, acc_d, fin_d, acc_o, fin_o, count, min_checked):
    report = {}
    for name, a, b in (("c11", acc_d.c11, acc_o.c11), ("c22", acc_d.c22, acc_o.c22),
                       ("s1", acc_d.class_sum1, acc_o.s1), ("s2", acc_d.class_sum2, acc_o.s2),
                       ("g1", acc_d.global_sum1, acc_o.g1), ("g2", acc_d.global_sum2, acc_o.g2),
                       ("fin_c11", fin_d[0], fin_o.c11), ("fin_c22", fin_d[1], fin_o.c22),
                       ("cw", fin_d[2], fin_o.cw), ("cb", fin_d[3], fin_o.cb), ("ctilde", fin_d[4], fin_o.ctilde)):
        report[name] = rel(a, b)
        assert report[name] <= STAT_TOL, (k, name, report[name])
    assert acc_d.patch_count == acc_o.n and np.array_equal(acc_d.per_class_patch_count, acc_o.n_class)
    lay = bank.layers[k]
    ref = O.to_layer(O.dcca_solve(fin_o, count), O.Geometry(lay.geom.l1, lay.geom.l2), True)
    wp = well_posed(fin_o, count)
    assert len(wp) >= min_checked, (k, wp)
    c1 = cosines(lay.filters1, ref.f1)
    c2 = cosines(lay.filters2, ref.f2)
    for j in wp:
        assert c1[j] >= COS_TOL and c2[j] >= COS_TOL, (k, j, c1[j], c2[j])
    # the device solver against the oracle solver on the device's own statistics
    fin_dd = O.Finalized(fin_d[0], fin_d[1], fin_d[2], fin_d[3], fin_d[4], acc_d.patch_count)
    same = O.to_layer(O.dcca_solve(fin_dd, count), O.Geometry(lay.geom.l1, lay.geom.l2), True)
    pr = O.dcca_solve(fin_dd, fin_dd.c11.shape[0])
    lam = pr.rho ** 2
    for j in range(count):
        gap = np.min(np.abs(np.delete(lam, j) - lam[j]))
        if gap <= 1e-10 * lam[0] or lam[j] <= 1e-20 * lam[0]:
            continue  # the reference's degenerate run: ordered by eigenvector entries
        # both Jacobi solvers stop at off(A) <= 1e-12 of the unit-scaled matrix, i.e. an
        # eigenvector is only fixed to ~1e-12 lam_0 / gap: tight where the gap is large,
        # loose for pairs whose gap sits within 1e6 of that stopping tolerance
        tol = 1e-6 if gap >= 1e-6 * lam[0] else 1e-3
        for a, b in ((lay.filters1[j], same.f1[j]), (lay.filters2[j], same.f2[j])):
            cos = abs((a * b).sum()) / (np.linalg.norm(a) * np.linalg.norm(b))
            assert cos >= 1 - tol, (k, j, cos, gap / lam[0])
    report["well_posed"] = wp
    report["cos_min_well_posed"] = float(min([min(c1[j], c2[j]) for j in wp], default=1.0))
    return report


def run_fit_parity(ex, v1, v2, lab, classes, net, min_checked):
    bank, accs, fins = device_fit(ex, v1, v2, lab, classes, net)
    out = []
    for k in range(len(net.layers)):
        acc_o, fin_o = oracle_layer(bank, k, v1.astype(np.float64), v2.astype(np.float64), lab, classes, net)
        out.append(check_layer(bank, k, accs[k], fins[k], acc_o, fin_o, net.layers[k].filters, min_checked))
    print("fit parity:", out)
    return bank, out


def _net(cfg, batch=128):
    return P.NetworkConfig(tuple(P.LayerConfig(L, P.PatchGeometry(l1, l2)) for L, l1, l2 in cfg["layers"]),
                           batch=P.BatchSpec(batch))


@pytest.mark.parametrize("mode", ["blocked", "exact"])
def test_fit_parity_orl_full(ex, ex_exact, mode):
    """BASELINE c1 in full: 400 x 112x92, 40 classes, 8/8 filters 5x5 — every layer, with the default
    float32-blocked and the exact float64 lag products."""
    v1, v2, lab, cfg = synthetic.make_corpus("orl")
    run_fit_parity(ex if mode == "blocked" else ex_exact, v1.astype(np.float32), v2.astype(np.float32), lab,
                   cfg["classes"], _net(cfg), 2)


def test_fit_parity_caltech_subsample(ex):
    """BASELINE c3 shape on a 128-image subsample (one batch, 257 classes, 8/8 filters 7x7)."""
    v1, v2, lab, cfg = synthetic.make_corpus("caltech256", m=128)
    run_fit_parity(ex, v1.astype(np.float32), v2.astype(np.float32), lab, cfg["classes"], _net(cfg), 2)


def test_fit_parity_three_stage_subsample(ex):
    """BASELINE c5 shape (12/12/12 filters 9x9, 256x256) on 16 images in 4 batches: all three
    layers' statistics and filters, then the 2^12-bin block counts of two samples."""
    v1, v2, lab, cfg = synthetic.make_corpus("three_stage", m=16)
    v1, v2 = v1.astype(np.float32), v2.astype(np.float32)
    net = _net(cfg, batch=4)
    bank, _ = run_fit_parity(ex, v1, v2, lab, cfg["classes"], net, 1)
    enc = P.EncoderConfig(*cfg["block"])
    sub = P.ViewPairDataset.from_arrays(v1[:2], v2[:2], lab[:2], class_count=cfg["classes"])
    counts, plan = P.compute_feature_counts(sub, bank, type("Cfg", (), {"net": net, "encoder": enc})(), ex)
    got = E.decode_counts(counts.cpu().numpy(), plan)
    layers = [O.Layer(l.filters1, l.filters2, O.Geometry(l.geom.l1, l.geom.l2), l.center) for l in bank.layers]
    ocfg = O.EncodeCfg(*cfg["block"])
    for i in range(2):
        m1, m2 = O.forward_maps(v1[i:i + 1], v2[i:i + 1], layers)
        want = []
        for maps in (m1[0], m2[0]):
            for g in range(maps.shape[0] // 12):
                code = O.combine_bits(O.sign_bits(maps[g * 12:(g + 1) * 12]))
                want.append(O.block_counts(code, ocfg, 12).reshape(-1))
        want = np.concatenate(want)
        assert got[i].shape == want.shape
        assert np.mean(got[i] == want) >= 0.999, np.mean(got[i] == want)


def test_orl_downstream_accuracy(ex, golden_json):
    """BASELINE c1: fit on the class-balanced train half, NN (euclidean) on the test half."""
    from paper_2209_13027_b200 import classify

    gold = golden_json("orl_accuracy")
    v1, v2, lab, cfg = synthetic.make_corpus("orl")
    v1, v2 = v1.astype(np.float32), v2.astype(np.float32)
    train = (np.arange(len(lab)) // cfg["classes"]) < 5
    test = ~train
    net = _net(cfg)
    enc = P.EncoderConfig(*cfg["block"])
    pcfg = type("Cfg", (), {"net": net, "encoder": enc})()
    ds_tr = P.ViewPairDataset.from_arrays(v1[train], v2[train], lab[train], class_count=cfg["classes"])
    ds_te = P.ViewPairDataset.from_arrays(v1[test], v2[test], lab[test], class_count=cfg["classes"])
    bank = P.train_network(ds_tr, net, ex)
    f_tr = P.compute_features(ds_tr, bank, pcfg, ex)
    f_te = P.compute_features(ds_te, bank, pcfg, ex)
    model = classify.fit(f_tr, lab[train], executor=ex)
    acc_dev = float(np.mean(classify.predict_many(model, f_te, executor=ex) == lab[test]))
    # the oracle's transform + classifier on the same bank
    layers = [O.Layer(l.filters1, l.filters2, O.Geometry(l.geom.l1, l.geom.l2), l.center) for l in bank.layers]
    ocfg = O.EncodeCfg(*cfg["block"])
    o_tr = O.features(v1[train], v2[train], layers, ocfg, batch=32, pool=POOL)
    o_te = O.features(v1[test], v2[test], layers, ocfg, batch=32, pool=POOL)
    same = min(float(np.mean(f_tr == o_tr)), float(np.mean(f_te == o_te)))
    acc_orc = O.nn_accuracy(O.nn_predict(o_tr, lab[train], o_te), lab[test])
    lo, hi = gold["band"]
    print(f"ORL accuracy: device {acc_dev:.4f}, oracle (same bank) {acc_orc:.4f}, identical bins {same:.6f}, "
          f"reference band [{lo:.3f}, {hi:.3f}] over batch sizes {[r['batch'] for r in gold['runs']]}")
    assert same >= 0.999
    assert abs(acc_dev - acc_orc) <= 0.005
    assert lo - 0.005 <= acc_dev <= hi + 0.005
    assert acc_dev < 1.0 and acc_orc < 1.0 and hi < 1.0  # not saturated: the check has teeth
