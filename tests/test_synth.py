"""Geometric assertions on the synthetic configs (SURVEY.md §7 step 1 gate)."""
import numpy as np

from synth import make_config, random_state


def test_c1_geometry():
    c = make_config("c1")
    assert c["image"].shape == (1, 128, 128) and c["image"].dtype == np.float32
    ii, jj = np.meshgrid(np.arange(128.0), np.arange(128.0), indexing="ij")
    d1 = (ii - 63.5) ** 2 + (jj - 41.5) ** 2 <= 400
    d2 = (ii - 63.5) ** 2 + (jj - 85.5) ** 2 <= 400
    cols1 = np.where(d1.any(0))[0]
    cols2 = np.where(d2.any(0))[0]
    assert cols2.min() - cols1.max() - 1 == 4           # 4 px gap
    # library convention: phi < 0 inside the rectangle
    assert c["phi0"][0, 34, 12] == -1 and c["phi0"][0, 33, 12] == 1 and c["phi0"][0, 93, 115] == -1


def test_c3_shapes_and_determinism():
    a = make_config("c3", images=[0, 5])
    b = make_config("c3", images=[5])
    assert a["image"].shape == (2, 1024, 1024)
    assert np.array_equal(a["image"][1], b["image"][0])
    assert a["phi0"][0, 0, 0] == 1 and a["phi0"][0, 16, 16] == -1 and a["phi0"][0, 15, 500] == 1


def test_random_state():
    s = random_state(32, 16, batch=2, seed=1)
    assert s["phi"].shape == (2, 32, 16) and all(v.dtype == np.float32 for v in s.values())
    assert (np.abs(s["phi"]) < 1).mean() > 0.3


def test_volume_recipe_is_seeded_and_shaped():
    from synth import make_volume
    a = make_volume((8, 16, 32), n=3, window=2, seed=1, border=2)
    b = make_volume((8, 16, 32), n=3, window=2, seed=1, border=2)
    assert a["volume"].shape == (8, 16, 32) and a["volume"].dtype == np.float32
    assert np.array_equal(a["volume"], b["volume"]) and np.array_equal(a["phi0"], b["phi0"])
    assert set(np.unique(a["phi0"])) == {-1.0, 1.0} and a["phi0"][0, 0, 0] == 1.0   # paper convention
    assert a["params"]["window"] == 2 and a["params"]["beta"] > 0
