"""Host-side logic that needs no GPU: the configs[2] shift generator."""
from paper_1606_01216_b200.sharding import Mt19937_64, airga_shift_draws


def test_mt19937_64_known_answer():
    # C++ [rand.predef]: the 10000th output of a default-constructed std::mt19937_64
    g = Mt19937_64()
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_airga_shift_draws_shape_and_range():
    d = airga_shift_draws(10, 8)
    assert len(d) == 10 and all(len(x) == 8 for x in d)
    assert all(x == sorted(x) for x in d)
    assert all(10.0 <= s <= 1e4 for x in d for s in x)
    # one generator across the sequence: later draws differ from the first
    assert d[0] != d[1]
    # deterministic
    assert airga_shift_draws(10, 8) == d
