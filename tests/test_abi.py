"""The C-ABI library loads and exports every symbol include/fda.h declares (no GPU needed)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fda_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_1311_5202_b200 import build
    lib = ctypes.CDLL(build.build())
    names = _declared()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(lib, nm), nm
    from paper_1311_5202_b200 import fda
    assert set(names) == set(fda.EXPORTS)


def test_status_strings_and_no_gpu_behaviour():
    from paper_1311_5202_b200 import fda
    assert fda.fda_status_str(0) == "FDA_OK"
    assert fda.fda_status_str(4) == "FDA_ERR_CUDA"
    assert fda.fda_plan_launches(None) == -1
    import numpy as np
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = np.random.default_rng(0).normal(size=(10, 3))
    n = x / np.linalg.norm(x, axis=1, keepdims=True)
    w = np.ones(10)
    # without a device the product path fails loudly (no CPU fallback)
    with pytest.raises(fda.FDAError, match="FDA_ERR_CUDA"):
        fda.fda_plan_create(x, n, w, 1.0, 1j, 1e-4)
    # the same for the corrected Nystrom weights: argument checks first, then no device -> FDA_ERR_CUDA
    el = np.zeros((1, 6, 3))
    xi = np.array([[0.1, 0.1], [0.8, 0.1], [0.1, 0.8], [0.4, 0.4], [0.2, 0.4], [0.4, 0.2]])
    pr = np.zeros(1, np.int64)
    out = np.zeros((1, 6), np.complex128)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, 1.0, 1j, el, xi, np.full(6, 1 / 12), x, n, pr, pr, out, nq=40)
    with pytest.raises(fda.FDAError, match="FDA_ERR_CUDA"):
        fda.fda_nystrom_weights(fda.FDA_KERNEL_BMH, 1.0, 1j, el, xi, np.full(6, 1 / 12), x, n, pr, pr, out)


def test_options_layout():
    from paper_1311_5202_b200 import fda
    o = fda.fda_options_default()
    assert o.lowrank == 1 and o.nranks == 1 and o.lf_p_low == 0 and o.hf_max_rows == 0
    assert o.kernel == fda.FDA_KERNEL_BMH and o.eps_lowrank == 0 and o.host_only == 0
    # the struct layout the binding declares matches the C one: a non-default field round-trips
    import numpy as np
    x = np.random.default_rng(0).normal(size=(64, 3))
    n = x / np.linalg.norm(x, axis=1, keepdims=True)
    with pytest.raises(fda.FDAError, match="INVALID_ARG"):
        fda.fda_plan_create(x, n, np.ones(64), 1.0, 1j, 1e-4, fda.fda_options_default(host_only=1, kernel=7))
    h = fda.fda_plan_create(x, n, np.ones(64), 1.0, 1j, 1e-4,
                            fda.fda_options_default(host_only=1, kernel=fda.FDA_KERNEL_BMG, rank=1, nranks=2))
    st = fda.fda_plan_stats(h)
    fda.fda_plan_destroy(h)
    assert st["n"] == 64 and 0 < st["owned_begin"] < 64 and st["owned_end"] == 64
