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


def test_paper_clblast_space_size():
    """The paper's GEMM space: Kernel Tuner's CLBlast lists give 17,472 valid configs,
    all accepted by the B200 kernel at the BASELINE size; x 7 clocks = 122,304 (tests/test_acceptance.py:66-81)."""
    from paper_2211_07260_b200 import CLOCK_PARAM, TunableParameter

    p = make_problem("sgemm", value_set="clblast")
    space = p.space()
    assert len(space.enumerate()) == 17472
    assert space.augment(TunableParameter(CLOCK_PARAM, tuple(range(7)))).size() == 122304
    # every config stays inside the B200 limits the kernel needs: <= 1024 threads, <= 227 KB smem
    for c in space.enumerate():
        cfg = {**p.default_config(), **c.as_dict()}
        launch = p.launch(cfg)
        assert launch.threads <= 1024 and launch.smem <= 227 * 1024
