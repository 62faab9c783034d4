"""Host-side logic of the device path against the oracle (CPU only, no kernels).

The geometry, block grid, count storage and batch split decide which bytes the
kernels read and write; here they are swept over many shapes against the
oracle's restatement of the reference (patches.py:41-65, 148-157;
encoder.py:38-44, 87-97, 141-144).
"""

import itertools

import numpy as np
import pytest

from oracle import port as O
from paper_2209_13027_b200 import engine as E
from paper_2209_13027_b200.encoder import EncoderConfig, feature_length
from paper_2209_13027_b200.errors import ConfigError, ShapeError
from paper_2209_13027_b200.patches import BatchSpec, PatchGeometry, batch_partition


@pytest.mark.parametrize("padding", ["zero_same", "none"])
def test_geometry_matches_oracle(padding):
    for p, q, l1, l2, s in itertools.product((1, 5, 7, 12, 17), (1, 6, 9, 16), (1, 2, 3, 5, 7), (1, 4, 5, 9), (1, 2, 3)):
        g, o = PatchGeometry(l1, l2, s, padding), O.Geometry(l1, l2, s, padding)
        if padding == "none" and (l1 > p or l2 > q):
            with pytest.raises(ShapeError):
                g.out_shape(p, q)
            with pytest.raises(O.OracleShapeError):
                o.grid(p, q)
            continue
        assert g.out_shape(p, q) == o.grid(p, q), (p, q, l1, l2, s)
        assert g.pad_amounts(p, q) == o.pads(p, q), (p, q, l1, l2, s)


def test_geometry_errors():
    for bad in ((0, 3, 1, "zero_same"), (3, 3, 0, "zero_same"), (3, 3, 1, "reflect")):
        with pytest.raises(ConfigError):
            PatchGeometry(*bad)


def test_block_plan_matches_block_starts():
    # overlaps that hit Python's banker's rounding: (1 - 0.5) * 5 = 2.5 -> 2, * 7 = 3.5 -> 4
    for (bh, bw), ov, (p, q) in itertools.product(((5, 5), (7, 7), (7, 3), (16, 16), (32, 32)),
                                                  (0.0, 0.25, 0.5, 0.75), ((32, 32), (112, 92), (128, 128))):
        if bh > p or bw > q:
            continue
        enc = EncoderConfig(bh, bw, ov)
        plan = E.block_plan(enc, p, q, 8)
        starts = O.block_origins(O.EncodeCfg(bh, bw, ov), p, q)
        grid = [(i * plan.sh, j * plan.sw) for i in range(plan.nby) for j in range(plan.nbx)]
        assert grid == starts == enc.block_starts(p, q), (bh, bw, ov, p, q)
        assert plan.bpc == bh * bw and plan.bins == 256


def test_block_plan_rejects_blocks_larger_than_the_map():
    with pytest.raises(ShapeError):
        E.block_plan(EncoderConfig(16, 16), 8, 32, 8)


@pytest.mark.parametrize("n_bits,maps", [(8, 64), (5, 25), (12, 1728)])
def test_feature_length_law(n_bits, maps):
    for shape, block in (((128, 128), (16, 16)), ((112, 92), (7, 7)), ((256, 256), (32, 32))):
        enc = EncoderConfig(*block)
        ref = O.feature_len(shape, maps, n_bits, O.EncodeCfg(*block))
        assert feature_length(shape, maps, n_bits, enc) == ref


def test_count_storage_thresholds():
    assert [E.count_kind(b) for b in (1, 49, 255, 256, 400, 510, 511, 1024)] == [0, 0, 0, 1, 1, 1, 2, 2]


def test_saturating_u8_counts_decode_exactly():
    # 16x16 blocks: 256 pixels per block, so one bin can reach 256 > 255; stored saturated, the
    # block total recovers it (engine.decode_counts)
    enc = EncoderConfig(16, 16)
    plan = E.block_plan(enc, 32, 32, 8)
    rng = np.random.default_rng(3)
    exact = np.zeros((plan.blocks, plan.bins), dtype=np.int64)
    exact[0, 7] = 256                               # the whole block in one bin
    exact[1, :] = 1                                 # one pixel per bin
    exact[2] = np.bincount(rng.integers(0, 4, 256), minlength=256)  # four hot bins
    exact[3, 0], exact[3, 255] = 255, 1             # 255 is stored as is, not as a saturated marker
    stored = np.minimum(exact, 255).astype(np.uint8)
    assert np.array_equal(E.decode_counts(stored.reshape(1, -1), plan).reshape(exact.shape), exact)


def test_u16_counts_decode():
    plan = E.block_plan(EncoderConfig(32, 32), 64, 64, 12)
    c = np.array([0, 1, 1024, 40000], dtype=np.uint16).view(np.int16)
    assert list(E.decode_counts(c, plan)) == [0, 1, 1024, 40000]


@pytest.mark.parametrize("policy", ["zero", "floor"])
@pytest.mark.parametrize("block", [(7, 7), (16, 16), (32, 32)])
def test_iq_lut_matches_oracle(policy, block):
    lut = E.iq_lut(EncoderConfig(*block, zero_bin_policy=policy))
    ref = O.iq_lut(O.EncodeCfg(*block, zero_bin_policy=policy))
    assert lut.dtype == np.float64 and np.array_equal(lut, ref)


def test_batch_partition_matches_oracle():
    for m, b in itertools.product((1, 127, 128, 129, 400, 30607), (1, 7, 128)):
        assert batch_partition(m, BatchSpec(b)) == O.batch_ranges(m, b)
        assert BatchSpec(b).batch_count(m) == len(O.batch_ranges(m, b))
    with pytest.raises(ConfigError):
        batch_partition(0, BatchSpec(128))
    with pytest.raises(ConfigError):
        BatchSpec(0)


def test_payload_length_law():
    # [c11 | c22 | s1 | s2 | g1 | g2 | n | n_c]
    for d, c in ((25, 40), (49, 8), (49, 257), (81, 257)):
        assert E.payload_len(d, c) == 2 * d * d + 2 * d * c + 2 * d + 1 + c


def test_sharded_dataset_rows():
    """ViewPairDataset.shard: a rank's rows of a larger dataset (multi-GPU e2e inputs)."""
    import numpy as np
    import pytest

    import paper_2209_13027_b200 as P

    v = np.arange(5 * 3 * 2, dtype=np.float32).reshape(5, 3, 2)
    ds = P.ViewPairDataset.shard(v, v + 1, np.array([0, 1, 2, 0, 1]), 10, 20, 3)
    assert len(ds) == 5 and ds.global_len == 20 and ds.row_offset == 10
    a, b, lab = ds.local_rows(11, 14)
    assert np.array_equal(a, v[1:4]) and np.array_equal(b, v[1:4] + 1) and lab.tolist() == [1, 2, 0]
    with pytest.raises(P.ShapeError):
        ds.local_rows(9, 12)
    with pytest.raises(P.ShapeError):
        P.ViewPairDataset.shard(v, v, np.zeros(5, int), 18, 20, 3)
    full = P.ViewPairDataset.from_arrays(v, v, np.zeros(5, int))
    assert full.global_len == 5 and full.local_rows(0, 5)[0].shape == (5, 3, 2)
