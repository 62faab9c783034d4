"""The tensor-core conv-histogram kernel (convtc.cu: tcgen05 kind::f16, two-term split) against
the float32 FFMA kernel and the float64 oracle (GPU).

* power-of-two invariance: the kernel scales every map by a power of two before the f16 split,
  so maps multiplied by 2^k (far outside the f16 range either way) give bit-identical counts;
* agreement with the FFMA kernel and with the oracle's float64 responses: the codes may differ
  only where a response is within float32-level rounding of zero, so almost every bin matches
  and every map keeps its pixel total.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import oracle as O  # noqa: E402
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import _native  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402


@pytest.fixture(scope="module")
def ex():
    return P.Executor(P.ExecSettings())


def _counts(ex, maps, f, l, plan, n_in, tc, monkeypatch):
    monkeypatch.setenv("DDCCA_CONV_TC", "1" if tc else "0")
    kind = E.count_kind(plan.bpc)
    featlen = n_in * plan.blocks * plan.bins
    out = torch.zeros((maps.shape[0] // n_in, featlen), dtype=torch.int16 if kind == 2 else torch.uint8,
                      device=ex.device)
    with torch.cuda.stream(ex.stream):
        lay = E.layer_from_filters(ex, f, f, P.PatchGeometry(l, l), True)
        assert E.conv_hist(ex, maps, lay, 1, plan, out.view(-1), kind, n_in, featlen, plan.blocks * plan.bins, True)
        path = _native.load().ddcca_conv_hist_last_path()
    ex.synchronize()
    assert path == (1 if tc else 0)
    return E.decode_counts(out.cpu().numpy(), plan)


@pytest.mark.parametrize("l", [3, 5, 7])
def test_power_of_two_scaling_is_exact(ex, l, monkeypatch):
    rng = np.random.default_rng(l)
    n_in, p, q = 8, 64, 72
    base = rng.standard_normal((16, p, q)).astype(np.float32)
    f = rng.standard_normal((8, l, l))
    plan = E.block_plan(P.EncoderConfig(8, 8), p, q, 8)
    ref = None
    for k in (0, -40, 30, 100):  # 2^100: beyond the f16 range by 84 binades, 2^-40: below it
        maps = torch.from_numpy(np.ldexp(base, k).astype(np.float32)).to(ex.device)
        got = _counts(ex, maps, f, l, plan, n_in, True, monkeypatch)
        if ref is None:
            ref = got
        assert np.array_equal(got, ref), k
    # filters scaled by a power of two: the per-filter scale absorbs it
    maps = torch.from_numpy(base).to(ex.device)
    assert np.array_equal(_counts(ex, maps, f * 2.0 ** -30, l, plan, n_in, True, monkeypatch), ref)


@pytest.mark.parametrize("l,p,q,bh", [(7, 128, 128, 16), (5, 100, 96, 10), (5, 100, 128, 10), (3, 128, 124, 8),
                                      (7, 33, 40, 8)])
def test_tc_matches_ffma_and_oracle(ex, l, p, q, bh, monkeypatch):
    rng = np.random.default_rng(l * 7 + p)
    n_in = 8
    n = 16
    base = rng.standard_normal((n, p, q)).astype(np.float32)
    # a per-map magnitude spread of 2^-10 .. 2^10 (per-map scales differ)
    base *= np.exp2(rng.integers(-10, 11, size=(n, 1, 1))).astype(np.float32)
    f = rng.standard_normal((8, l, l))
    plan = E.block_plan(P.EncoderConfig(bh, bh), p, q, 8)
    maps = torch.from_numpy(base).to(ex.device)
    tc = _counts(ex, maps, f, l, plan, n_in, True, monkeypatch)
    ff = _counts(ex, maps, f, l, plan, n_in, False, monkeypatch)
    assert np.mean(tc == ff) >= 0.999
    resp = O.conv_stack(base.astype(np.float64), O.Layer(f, f, O.Geometry(l, l), True), 1)
    want = np.stack([np.concatenate([O.block_counts(O.combine_bits(O.sign_bits(resp[i * n_in + g])),
                                                    O.EncodeCfg(bh, bh), 8).reshape(-1) for g in range(n_in)])
                     for i in range(n // n_in)])
    assert np.mean(tc == want) >= 0.999
    # every block keeps its pixel count
    per = tc.reshape(tc.shape[0], -1, plan.bins).sum(axis=2)
    assert (per == plan.bpc).all()


@pytest.mark.parametrize("l,p,q,count,center,dc", [(7, 128, 128, 8, True, 0.0), (5, 64, 48, 8, True, 1000.0),
                                                    (3, 100, 96, 6, False, 0.0), (7, 33, 40, 8, True, 5.0),
                                                    (5, 128, 124, 4, True, 0.5)])
def test_tc_responses_vs_ffma_and_oracle(ex, l, p, q, count, center, dc, monkeypatch):
    """Responses mode (ddcca_conv on the tensor cores): float32-level agreement with the FFMA
    kernel and the float64 oracle; centered windows shift each map by its mean first, so a large
    DC offset (1000 + [0, 1)) costs no accuracy."""
    rng = np.random.default_rng(l * 11 + q)
    maps = (rng.uniform(size=(6, p, q)) + dc).astype(np.float32)
    f = rng.standard_normal((count, l, l))
    lib = _native.load()
    dm = torch.from_numpy(maps).to(ex.device)
    with torch.cuda.stream(ex.stream):
        lay = E.layer_from_filters(ex, f, f, P.PatchGeometry(l, l), center)

    def run(tc):
        monkeypatch.setenv("DDCCA_CONV_TC", "1" if tc else "0")
        with torch.cuda.stream(ex.stream):
            out = E.conv(ex, dm, lay, 1)
            path = lib.ddcca_conv_last_path()
        ex.synchronize()
        return out.cpu().numpy().astype(np.float64), path

    got, path = run(True)
    assert path == 1
    ffma, path0 = run(False)
    assert path0 == 0
    ref = O.conv_stack(maps, O.Layer(f, f, O.Geometry(l, l), center), 1)
    # the zero padding counts: shifted by the mean it is as far from it as the mean itself
    mean = maps.mean(axis=(1, 2), keepdims=True)
    spread = max(np.abs(maps - mean).max(), np.abs(mean).max()) if center else np.abs(maps).max()
    scale = np.abs(f).sum(axis=(1, 2)).max() * spread
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 2e-6 * scale
    assert np.abs(got - ffma).max() <= 4e-6 * scale
