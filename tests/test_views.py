"""Device LBP second view (views.py:41-58) vs the reference's golden outputs and the oracle."""

import numpy as np
import pytest

import oracle as O


def test_recipe_errors():
    import paper_2209_13027_b200 as P

    with pytest.raises(P.RecipeError):
        P.ViewRecipe("rgb")
    with pytest.raises(P.RecipeError):
        P.apply_recipe([], P.ViewRecipe("identity_pair"))
    with pytest.raises(P.RecipeError):
        P.apply_recipe([np.zeros((3, 3)), np.zeros((3, 3))], P.ViewRecipe("identity_pair"))
    a, b = np.ones((3, 3)), np.zeros((3, 3))
    assert P.apply_recipe([a, b], P.ViewRecipe("external_pair"))[1] is b
    assert P.apply_recipe([a, b], P.ViewRecipe("channel_split", 1, 0))[0] is b


@pytest.mark.gpu
def test_device_lbp_matches_reference(golden):
    import paper_2209_13027_b200 as P

    g = golden("views")
    for k in range(4):
        assert np.array_equal(P.lbp_map(g[f"img{k}"]), g[f"lbp{k}"]), k
    gray = g["img2"]
    v1, v2 = P.apply_recipe([gray], P.ViewRecipe("lbp_plus_gray"))
    assert v1 is gray and np.array_equal(v2, g["lbp2"])
    with pytest.raises(P.ShapeError):
        P.lbp_map(np.zeros((2, 9)))


@pytest.mark.gpu
def test_device_lbp_stack_vs_oracle():
    import torch

    import paper_2209_13027_b200 as P

    rng = np.random.default_rng(4)
    x = (rng.integers(0, 5, size=(37, 19, 23)) / 4.0 - 0.25).astype(np.float32)
    got = P.lbp_stack(torch.from_numpy(x).cuda()).cpu().numpy()
    want = np.stack([O.lbp(im) for im in x]).astype(np.float32)
    assert np.array_equal(got, want)
