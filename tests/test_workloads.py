"""Input generators (workloads/): determinism and shape, no method arithmetic."""
import numpy as np

from workloads import config, franke2, grid_level, halton, uniform_points


def test_halton_nested_and_deterministic():
    a = halton(1000, 3)
    b = halton(250, 3)
    np.testing.assert_array_equal(a[:250], b)
    assert a.min() > 0 and a.max() < 1
    assert halton(1, 2).tolist() == [[0.5, 1.0 / 3.0]]


def test_grid_sizes_table1(golden):
    for lvl, n in golden["table1"]["N"].items():
        if int(lvl) <= 4:
            assert grid_level(int(lvl)).shape == (n, 2)


def test_franke_hand_values():
    # first term alone at (2/9, 2/9) is 3/4; F(0,0) by hand evaluation
    v = franke2(np.array([[0.0, 0.0]]))[0]
    ref = (0.75 * np.exp(-8 / 4) + 0.75 * np.exp(-1 / 49 - 0.1) + 0.5 * np.exp(-(49 + 9) / 4)
           - 0.2 * np.exp(-16 - 49))
    assert abs(v - ref) < 1e-15 and abs(v - 0.766420591284923) < 1e-14


def test_configs_shapes():
    c1 = config("C1")
    assert c1.n == [100, 400, 1600] and c1.d == 2
    c3 = config("C3P4", m_eval=10)
    assert c3.n == [305, 2441, 19531, 156250] and c3.d == 3
    assert uniform_points(5, 3).shape == (5, 3)
