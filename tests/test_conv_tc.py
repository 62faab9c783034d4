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
