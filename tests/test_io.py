"""Ingestion (dataset.py:60-230): native PGM decode and manifests vs the reference's outputs.

The PGM files and manifests under tests/golden/io/ were written by the
reference's write_pgm; io.npz holds its load_pgm / load_dataset results.
"""

import numpy as np
import pytest

from conftest import GOLDEN

IO = GOLDEN / "io"


def test_load_pgm_bitexact(golden):
    import paper_2209_13027_b200 as P

    g = golden("io")
    for k in list(range(6)):
        name = f"img{k}.pgm"
        assert np.array_equal(P.load_pgm(IO / name), g["pgm_" + name]), name
    assert np.array_equal(P.load_pgm(IO / "comment.pgm"), g["pgm_comment.pgm"])


def test_pgm_errors(tmp_path):
    import paper_2209_13027_b200 as P

    with pytest.raises(P.ParseError):
        P.load_pgm(IO / "bad_magic.pgm")
    with pytest.raises(P.ParseError):
        P.load_pgm(IO / "truncated.pgm")
    with pytest.raises(P.IoError):
        P.load_pgm(tmp_path / "missing.pgm")
    (tmp_path / "zero.pgm").write_bytes(b"P5\n2 2\n0\n" + bytes(4))
    with pytest.raises(P.ParseError):
        P.load_pgm(tmp_path / "zero.pgm")
    with pytest.raises(P.ParseError):
        P.write_pgm(tmp_path / "x.pgm", np.zeros((2, 2)), maxval=70000)


def test_write_pgm_roundtrip(tmp_path):
    import paper_2209_13027_b200 as P

    img = np.random.default_rng(1).uniform(size=(9, 4))
    for mv in (255, 65535):
        P.write_pgm(tmp_path / "r.pgm", img, maxval=mv)
        back = P.load_pgm(tmp_path / "r.pgm")
        assert np.abs(back - img).max() <= 0.5 / mv + 1e-12


@pytest.mark.gpu
def test_load_dataset_matches_reference(golden):
    import paper_2209_13027_b200 as P

    g = golden("io")
    ds = P.load_dataset(IO / "pairs.txt")
    v1, v2, lab = ds.stacks_view()
    assert np.array_equal(np.asarray(v1), g["pairs_v1"].astype(np.float32))
    assert np.array_equal(np.asarray(v2), g["pairs_v2"].astype(np.float32))
    assert np.array_equal(ds.labels, g["pairs_labels"])
    assert sorted(ds.label_map.items()) == [tuple(r) for r in g["pairs_map"].tolist()]
    ds = P.load_dataset(IO / "gray.txt", P.ViewRecipe("lbp_plus_gray"))
    v1, v2, lab = ds.stacks_view()
    assert np.array_equal(np.asarray(v1), g["gray_v1"].astype(np.float32))
    assert np.array_equal(np.asarray(v2), g["gray_v2"].astype(np.float32))  # device LBP of the float32 view 1
    assert np.array_equal(ds.labels, g["gray_labels"])
    assert ds.class_count == 3


@pytest.mark.gpu
def test_load_dataset_errors(tmp_path):
    import paper_2209_13027_b200 as P

    (tmp_path / "empty.txt").write_text("# nothing\n\n")
    with pytest.raises(P.EmptyDatasetError):
        P.load_dataset(tmp_path / "empty.txt")
    (tmp_path / "neg.txt").write_text(f"{IO / 'img0.pgm'},-1\n")
    with pytest.raises(P.ParseError):
        P.load_dataset(tmp_path / "neg.txt")
    small = np.zeros((3, 3))
    P.write_pgm(tmp_path / "s.pgm", small)
    (tmp_path / "mixed.txt").write_text(f"{IO / 'img0.pgm'},1\n{tmp_path / 's.pgm'},2\n")
    with pytest.raises(P.ShapeError):
        P.load_dataset(tmp_path / "mixed.txt")
    (tmp_path / "missing.txt").write_text(f"{tmp_path / 'nope.pgm'},1\n")
    with pytest.raises((P.IoError, P.ParseError)):
        P.load_dataset(tmp_path / "missing.txt")


@pytest.mark.parametrize("bh,bw", [(4, 4), (16, 17), (10, 30)])  # u8, saturating u8, u16 counts
def test_feature_csv_matches_reference_format(tmp_path, bh, bw):
    """Native CSV writer == the reference's f"{i}," + ",".join(format(v, ".17g")) lines on the float64 features."""
    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import engine as E

    rng = np.random.default_rng(bh + bw)
    enc = P.EncoderConfig(bh, bw)
    plan = E.block_plan(enc, 40, 60, 4)
    n = 7
    counts = np.stack([np.concatenate([np.bincount(rng.integers(0, 16, plan.bpc), minlength=16)
                                       for _ in range(plan.blocks)]) for _ in range(n)])
    kind = E.count_kind(plan.bpc)
    stored = counts.astype(np.uint16).view(np.int16) if kind == 2 else np.minimum(counts, 255).astype(np.uint8)
    P.write_feature_csv(tmp_path / "f.csv", stored, plan, enc, first_index=3, threads=3)
    feats = E.iq_lut(enc)[counts]
    want = "".join(f"{i + 3}," + ",".join(format(v, ".17g") for v in row) + "\n" for i, row in enumerate(feats))
    assert (tmp_path / "f.csv").read_text() == want
