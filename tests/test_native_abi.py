"""The C-ABI library loads, exports every symbol include/jt.h declares, and
its context-free parts work without a GPU (no compute calls here)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2211_07260_b200 import native
from paper_2211_07260_b200.errors import CapabilityError, DomainError
from paper_2211_07260_b200.kernels import Conv2DProblem, PnPolyProblem, SgemmProblem

HEADER = Path(__file__).resolve().parents[1] / "include" / "jt.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|double|void|const char \*)\s*\*?\s*(jt_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    native.build_library()
    lib = ctypes.CDLL(str(native.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing
    assert set(names) == set(native.EXPORTS)
    assert native.lib().jt_abi_version() == 3


def test_no_gpu_means_capability_error_not_fallback():
    count = ctypes.c_int(-1)
    status = native.lib().jt_device_count(ctypes.byref(count))
    if status == native.JT_OK and count.value > 0:
        pytest.skip("a GPU is visible")
    from paper_2211_07260_b200.gpu import GPU

    with pytest.raises(CapabilityError):
        GPU(0)


@pytest.mark.parametrize("problem", [PnPolyProblem(), Conv2DProblem(), SgemmProblem()], ids=lambda p: p.name)
def test_nvrtc_compiles_default_config_for_sm100a(problem):
    blob = problem.cubin(problem.default_config())
    assert blob[:4] == b"\x7fELF" and len(blob) > 1000


def test_nvrtc_errors_become_domain_errors():
    with pytest.raises(DomainError):
        native.compile_cubin("extern \"C\" __global__ void k() { this is not cuda }", "bad",
                             native._nvrtc_options({}), use_cache=False)
    bad_cfg = dict(SgemmProblem().default_config(), MWG=96)  # violates MWG % (MDIMC*VWM)
    with pytest.raises(DomainError):
        SgemmProblem().cubin(bad_cfg)


def test_pnpoly_edge_tables_are_float32_exact():
    p = PnPolyProblem(n_points=10)
    inp = p.host_inputs()
    vx, vy = inp["vx"], inp["vy"]
    prev = np.roll(np.arange(vx.size), 1)
    e0, yb = native.pnpoly_edges(vx, vy, 0)
    dx = (vx[prev] - vx).astype(np.float32)
    dy = (vy[prev] - vy).astype(np.float32)
    np.testing.assert_array_equal(e0[:, 0], vy)
    np.testing.assert_array_equal(e0[:, 2], dx)
    np.testing.assert_array_equal(e0[:, 3], dy)
    np.testing.assert_array_equal(yb[:, 0], np.minimum(vy, vy[prev]))
    e1, _ = native.pnpoly_edges(vx, vy, 1)
    np.testing.assert_array_equal(e1[:, 2], (dx / dy).astype(np.float32))
    e2, _ = native.pnpoly_edges(vx, vy, 2)
    # icpt = fma(-slope, vy, vx): exact via float64 product (24+24 bits) then one rounding
    # differs from fma only when the f64 sum itself rounds; check |err| <= 1 ulp and most exact
    approx = (-(e2[:, 2].astype(np.float64)) * vy + vx).astype(np.float32)
    assert np.mean(approx == e2[:, 1]) > 0.99


def test_sgemm_space_restrictions_follow_clblast():
    s = SgemmProblem()
    for cfg in s.space().enumerate()[:2000:97]:
        c = cfg.as_dict()
        assert c["KWG"] % c["KWI"] == 0
        assert c["MWG"] % (c["MDIMC"] * c["VWM"]) == 0 and c["NWG"] % (c["NDIMC"] * c["VWN"]) == 0
        assert (c["SA"] * c["KWG"] * c["MWG"] + c["SB"] * c["KWG"] * c["NWG"]) * 8 <= 48 * 1024
