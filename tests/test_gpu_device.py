"""The B200 device behind the reference API: benchmark/strategy/observers on
real hardware (NVML energy counter, controller refusal recorded, no fallback)."""

import math

import numpy as np
import pytest

import paper_2211_07260_b200 as B
from oracle import kernels_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    from paper_2211_07260_b200.gpu import GPU

    g = GPU(0)
    yield g
    g.close()


@pytest.fixture(scope="module")
def conv_device(gpu):
    from paper_2211_07260_b200.b200 import B200Device

    dev = B200Device("conv2d", gpu=gpu, problem_kwargs={"width": 1024, "height": 1024}, min_window=0.15)
    yield dev
    dev.release_clock()


def test_spec_from_nvml(conv_device):
    spec = conv_device.spec
    assert len(spec.supported_core_clocks) > 50
    assert list(spec.supported_core_clocks) == sorted(spec.supported_core_clocks)
    assert spec.peak_clock == max(spec.supported_core_clocks) and spec.base_clock in spec.supported_core_clocks
    assert not spec.voltage_readable
    with pytest.raises(B.CapabilityError):
        conv_device.read_voltage(spec.peak_clock)


def test_benchmark_counter_energy_is_physical(conv_device):
    p = conv_device.problem
    cfg = B.KernelConfig.from_dict(p.default_config())
    res = B.benchmark(conv_device, cfg, [B.NVMLObserver(0.3)], user_metrics=B.default_metrics(p.total_flops),
                      constants={"total_flops": p.total_flops})
    assert not res.failed, res.failure_reason
    obs = res.observer_results
    print(res.to_dict())
    assert 100.0 < obs["nvml_power"] < 1200.0
    assert res.energy == pytest.approx(obs["nvml_power"] * res.time)
    assert 300 < obs["nvml_sm_clock"] <= 2100 and 10 < obs["nvml_temperature"] < 100
    assert obs["nvml_clock_locked"] in (0.0, 1.0)
    assert res.metrics["gflops"] > 1000.0 and 1.0 < res.metrics["gflops_per_w"] < 500.0
    # the instant-power median and the counter slope agree within 25 %
    assert obs["nvml_power_instant"] == pytest.approx(obs["nvml_power"], rel=0.25)


def test_instant_observer_window_rule(conv_device):
    cfg = B.KernelConfig.from_dict(conv_device.problem.default_config())
    res = B.benchmark(conv_device, cfg, [B.InstantPowerObserver()])
    assert not res.failed, res.failure_reason
    assert 100.0 < res.observer_results["ps_power"] < 1200.0


def test_clock_request_recorded_and_unsupported_clock_fails(conv_device):
    cfg = B.KernelConfig.from_dict({**conv_device.problem.default_config(),
                                    "nvml_gr_clock": conv_device.spec.peak_clock})
    res = B.benchmark(conv_device, cfg, [B.NVMLObserver(0.2)])
    assert not res.failed
    assert conv_device.clock_mode in ("locked", "application", "refused")
    if conv_device.clock_mode == "refused":
        assert res.observer_results["nvml_clock_locked"] == 0.0
    bad = B.KernelConfig.from_dict({**conv_device.problem.default_config(), "nvml_gr_clock": 1234.5})
    res = B.benchmark(conv_device, bad, [B.NVMLObserver(0.2)])
    assert res.failed and "DomainError" in res.failure_reason


def test_invalid_launch_is_a_failed_result_not_a_crash(gpu):
    from paper_2211_07260_b200.b200 import B200Device

    dev = B200Device("sgemm", gpu=gpu, problem_kwargs={"m": 256, "n": 256, "k": 256}, min_window=0.05)
    cfg = B.KernelConfig.from_dict({**dev.problem.default_config(), "MDIMC": 32, "NDIMC": 64, "MWG": 128,
                                    "NWG": 256})  # 2048 threads per block
    res = B.benchmark(dev, cfg, [B.NVMLObserver(0.1)])
    assert res.failed and "DomainError" in res.failure_reason
    # the context stays healthy
    ok = B.benchmark(dev, B.KernelConfig.from_dict(dev.problem.default_config()), [B.NVMLObserver(0.1)])
    assert not ok.failed


def test_answer_verification_turns_wrong_output_into_failure(gpu):
    from paper_2211_07260_b200.b200 import B200Device
    from paper_2211_07260_b200.kernels import PnPolyProblem

    p = PnPolyProblem(n_points=200_000)
    p.prepare(gpu)
    answer = O.pnpoly(p.inputs["points"], p.inputs["vx"], p.inputs["vy"], 3)
    dev = B200Device(p, gpu=gpu, answer=answer, min_window=0.05)
    good = B.benchmark(dev, B.KernelConfig.from_dict(p.default_config()), [B.NVMLObserver(0.1)])
    assert not good.failed, good.failure_reason
    dev.answer = 1 - answer
    bad = B.benchmark(dev, B.KernelConfig.from_dict(p.default_config()), [B.NVMLObserver(0.1)])
    assert bad.failed and "does not match" in bad.failure_reason


def test_run_strategy_on_b200_with_cache(gpu, tmp_path):
    from paper_2211_07260_b200.b200 import B200Device

    dev = B200Device("pnpoly", gpu=gpu, problem_kwargs={"n_points": 1 << 20}, min_window=0.05)
    space = B.SearchSpace.from_dict({"parameters": {"block_size_x": [128, 256], "tile": [4, 8], "vec": [2],
                                                    "method": [2], "between": [0], "poly_smem": [1], "asm": [3]}})
    cache = B.ResultCache(tmp_path / "c.jsonl")
    out = B.run_strategy(B.TuningRun(space, "exhaustive", B.Objective("energy")), dev, [B.NVMLObserver(0.1)],
                         cache=cache)
    assert out.device_executions == 4 and all(not r.failed for r in out.history)
    again = B.run_strategy(B.TuningRun(space, "exhaustive", B.Objective("energy")), dev, [B.NVMLObserver(0.1)],
                           cache=B.ResultCache(tmp_path / "c.jsonl"))
    assert again.device_executions == 0


def test_energy_counter_advances_under_load(gpu):
    from paper_2211_07260_b200.kernels import make_problem

    p = make_problem("burner", iters=2048)
    p.prepare(gpu)
    cfg = p.default_config()
    k = p.kernel(cfg)
    run = gpu.bench(k, p.launch(cfg), p.args(cfg), min_seconds=0.5)
    e = [s[3] for s in run.samples if math.isfinite(s[3])]
    assert e and e[-1] > e[0]
    inst = [s[1] for s in run.samples if s[0] > run.loop_t0 + 0.2 and math.isfinite(s[1])]
    assert inst and np.median(inst) > 150.0
    # burner is an FFMA-only load: >= 85 % of the FP32 peak at the observed clock
    from paper_2211_07260_b200.gpu import fp32_peak_tflops

    mhz = np.median([s[5] for s in run.samples if s[5]])
    assert p.total_flops / run.per_launch_s / 1e12 >= 0.85 * fp32_peak_tflops(gpu.sm_count, mhz)
