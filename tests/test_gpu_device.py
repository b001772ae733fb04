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
    assert 100.0 < obs["nvml_power"] < 1200.0
    assert res.energy == pytest.approx(obs["nvml_power"] * res.time)
    assert 300 < obs["nvml_sm_clock"] <= 2100 and 10 < obs["nvml_temperature"] < 100
    assert obs["nvml_clock_locked"] in (0.0, 1.0)
    assert res.metrics["gflops"] > 1000.0 and 1.0 < res.metrics["gflops_per_w"] < 500.0
    # the instant-power field lags load changes by 100-200 ms on B200 (measured), so
    # over a 0.3 s loop it only has to be physical; the counter slope is primary
    assert 100.0 < obs["nvml_power_instant"] < 1200.0 and obs["nvml_energy_source"] == 1.0


def test_instant_observer_window_rule(conv_device):
    cfg = B.KernelConfig.from_dict(conv_device.problem.default_config())
    res = B.benchmark(conv_device, cfg, [B.InstantPowerObserver()])
    assert not res.failed, res.failure_reason
    assert 100.0 < res.observer_results["ps_power"] < 1200.0


def test_clock_request_recorded_and_unsupported_clock_fails(conv_device):
    cfg = B.KernelConfig.from_dict({**conv_device.problem.default_config(),
                                    "nvml_gr_clock": conv_device.spec.base_clock})
    res = B.benchmark(conv_device, cfg, [B.NVMLObserver(0.2)])
    assert not res.failed, res.failure_reason  # locked, or the driver-managed default clock
    assert conv_device.clock_mode in ("locked", "application", "refused")
    lower = [c for c in conv_device.spec.supported_core_clocks if c < 0.8 * conv_device.spec.base_clock][-1]
    low = B.benchmark(conv_device, B.KernelConfig.from_dict({**cfg.as_dict(), "nvml_gr_clock": lower}),
                      [B.NVMLObserver(0.2)])
    if conv_device.clock_mode == "refused":
        assert res.observer_results["nvml_clock_locked"] == 0.0
        # a refused clock is a failed result carrying NVML's reason, never a mislabelled measurement
        assert low.failed and "ControlRefusedError" in low.failure_reason
        assert conv_device.refusals and conv_device.refusals[-1]["requested"] == lower
    else:
        assert not low.failed and low.observer_results["nvml_sm_clock"] <= lower + 15
    bad = B.KernelConfig.from_dict({**conv_device.problem.default_config(), "nvml_gr_clock": 1234.5})
    res = B.benchmark(conv_device, bad, [B.NVMLObserver(0.2)])
    assert res.failed and "DomainError" in res.failure_reason
    conv_device.release_clock()


def test_power_limit_request_is_applied_or_failed(conv_device):
    cfg = B.KernelConfig.from_dict({**conv_device.problem.default_config(), "nvml_pwr_limit": 600})
    res = B.benchmark(conv_device, cfg, [B.NVMLObserver(0.2)])
    if res.failed:
        assert "ControlRefusedError" in res.failure_reason and "power_limit" in res.failure_reason
    else:  # accepted: the limit was read back as enforced
        assert conv_device.gpu.enforced_power_limit_w() == pytest.approx(600.0, abs=1.0)
    conv_device.gpu.reset_power_limit()


def test_continuous_benchmark_through_probe_runtime(conv_device):
    """Averaged-sensor mode on B200 (reference observers.py:136-172): the runtime probe is a CUDA-event
    launch (probe_runtime, not the simulator's surface) and the reading is NVML's own 1 s average."""
    cfg = B.KernelConfig.from_dict(conv_device.problem.default_config())
    probe = conv_device.probe_runtime(cfg)
    assert 1e-6 < probe < 0.1
    sensor = B.AveragedSensorConfig(refresh_rate=1.0, continuous_duration=2.0)
    out = B.continuous_benchmark(conv_device, cfg, sensor)
    assert not out.long_kernel and out.repetitions > 100 and out.duration >= 2.0
    assert 150.0 < out.mean_power < 1200.0 and out.energy == pytest.approx(out.mean_power * out.duration)
    # same loop through the energy counter: the board's 1 s average agrees within 15 %
    res = B.benchmark(conv_device, cfg, [B.NVMLObserver(2.0)])
    assert abs(out.mean_power - res.observer_results["nvml_power"]) < 0.15 * res.observer_results["nvml_power"]
    with pytest.raises(B.ConfigurationError):  # NVML's window is 1 s: a 10 Hz sensor config is a caller mistake
        B.continuous_benchmark(conv_device, cfg, B.AveragedSensorConfig(refresh_rate=10.0, continuous_duration=1.0))
    # the averaged observer through benchmark() reads the same sensor
    avg = B.benchmark(conv_device, cfg, [B.AveragedPowerObserver(sensor)], averaged_cfg=sensor)
    assert not avg.failed and 150.0 < avg.observer_results["nvml_power"] < 1200.0


def test_simulate_sweep_cli_on_b200(tmp_path):
    """``simulate-sweep --device b200`` (reference cli.py:132-176) end to end on the real board: a P(f)
    sweep when clock control works, else exit 1 with every refusal recorded and no sweep written."""
    from paper_2211_07260_b200 import commands
    import json

    out = tmp_path / "sweep.csv"
    rc = commands.main(["simulate-sweep", "--device", "b200:burner", "--out", str(out), "--points", "5",
                        "--observer", "nvml", "--duration", "0.3"])
    meta = json.loads((tmp_path / "sweep.csv.meta.json").read_text())
    if meta["clock_mode"] == "refused":
        assert rc == 1 and not out.exists()
        assert len(meta["refused"]) == 4 and all(r["reason"] for r in meta["refused"])
        assert len(meta["records"]) == 1 and meta["records"][0]["clock_locked"] == 0.0
    else:
        assert rc == 0 and out.exists() and len(meta["records"]) == 5


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


VECTOR_ADD = r"""
extern "C" __global__ void vector_add(float *c, const float *a, const float *b, int n) {
    int i = blockIdx.x * block_size_x + threadIdx.x;
    if (i < n) c[i] = a[i] + b[i];
}
"""


def test_tune_kernel_custom_source_kernel_tuner_style():
    """The paper's usage: tune_kernel(name, source, size, args, tune_params, metrics=lambdas)."""
    from paper_2211_07260_b200 import tune_kernel

    n = np.int32(10_000_000)
    a = np.random.default_rng(0).standard_normal(n).astype(np.float32)
    b = np.random.default_rng(1).standard_normal(n).astype(np.float32)
    c = np.zeros_like(a)
    rows, outcome = tune_kernel(
        "vector_add", VECTOR_ADD, int(n), [c, a, b, n], {"block_size_x": [128, 256, 512, 1024]},
        answer=[a + b, None, None, None], metrics={"GB/s": lambda p: 12 * n / 1e9 / (p["time"] / 1e3)},
        duration=0.1,
    )
    assert len(rows) == 4 and not any(r["failed"] for r in rows)
    assert all(r["GB_per_s"] > 500 for r in rows)  # HBM-class bandwidth
    assert outcome.best.energy == min(r["energy_j"] for r in rows)


def test_tune_kernel_builtin_problem_and_wrong_answer():
    from paper_2211_07260_b200 import tune_kernel

    rows, outcome = tune_kernel("pnpoly", tune_params={"block_size_x": [128, 256], "tile": [8], "asm": [3]},
                                problem_kwargs={"n_points": 1 << 18}, duration=0.05)
    assert len(rows) == 2 and outcome.best.metrics["gflops"] > 0
    ones = np.ones(1000, np.float32)
    with pytest.raises(B.TuningError):  # every config fails verification against a wrong answer
        tune_kernel("vector_add", VECTOR_ADD, 1000, [np.zeros(1000, np.float32), ones, ones, np.int32(1000)],
                    {"block_size_x": [128, 256]}, answer=[np.full(1000, 3.0, np.float32), None, None, None],
                    duration=0.05)


def test_stream_gate_holds_then_runs_the_sequence(gpu):
    """jt_stream_gate / jt_stream_release (bench.py's timed region): nothing enqueued behind the gate
    runs before the release; after it the start event, the launches and the stop event run back to
    back, and the output equals the oracle's."""
    import time

    from paper_2211_07260_b200.kernels import Conv2DProblem

    p = Conv2DProblem(width=512, height=512)
    p.prepare(gpu)
    cfg = p.default_config()
    k = p.kernel(cfg)
    p.bind(k, cfg)
    prepared = gpu.prepare_launch(k, p.launch(cfg), p.args(cfg))
    gpu.reserve_events(2)
    for _ in range(2):  # the gate re-arms
        p.reset_output()
        gpu.synchronize()
        gpu.gate()
        gpu.record(0)
        for _ in range(4):
            gpu.launch_prepared(prepared)
        gpu.record(1)
        time.sleep(0.05)  # held: 50 ms of host time pass before the release
        gpu.release()
        ms = gpu.elapsed(0, 1) * 1e3
        assert 0 < ms < 20, ms  # the held 50 ms are not inside the events
    gpu.synchronize()
    ref = O.conv2d(p.inputs["image"], p.inputs["filter"])
    assert O.conv2d_error(p.fetch_output(), ref, p.inputs["image"], p.inputs["filter"]) <= 1e-5
    for b in p.buffers.values():
        b.free()
