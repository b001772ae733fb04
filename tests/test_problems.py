"""Problem definitions (CPU): every default config names every tunable of its space and is
valid, and every tuned config in tuned_b200.json is valid for its problem."""

import pytest

from paper_2211_07260_b200 import tuned
from paper_2211_07260_b200.kernels import PROBLEMS, make_problem

SMALL = {"pnpoly": {"n_points": 4096}, "pnpoly_slab": {"n_points": 4096}}


@pytest.mark.parametrize("name", sorted(n for n in PROBLEMS if n != "burner"))
def test_default_config_covers_the_space(name):
    p = make_problem(name, **SMALL.get(name, {}))
    d = p.default_config()
    assert set(p.space().names) <= set(d), set(p.space().names) - set(d)
    assert p.is_valid(d)


@pytest.mark.parametrize("name", sorted(n for n in PROBLEMS if n != "burner"))
def test_tuned_configs_are_valid(name):
    p = make_problem(name, **SMALL.get(name, {}))
    for cfg in tuned.configs_for(name):
        assert p.is_valid(cfg), cfg
