"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/tcb200.h declares, and refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcb200.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_12011_b200 import _build
    _build.build()
    return ctypes.CDLL(_build.LIB)


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_the_abi():
    import paper_2510_12011_b200 as T
    for n in _declared():
        assert hasattr(T, n), n


def test_config_defaults_match_paper(lib):
    import paper_2510_12011_b200 as T
    c = T.tc_config_default()
    assert c.theta == 0.5            # P:151 Crank-Nicolson default
    assert c.abs_tol == 1e-5 and c.max_iters == 100
    assert c.chi == 140.0 and c.cm == 0.01             # Table 3
    assert c.lat_threshold == 0.0 and c.lrt_threshold == -70.0
    assert c.use_rcm == 1
    assert c.pcg_variant == -1       # automatic PCG kernel choice (include/tcb200.h)


def test_cohort_io_argument_errors(lib):
    """tc_cohort_set_states / tc_cohort_get_v reject null arguments with TC_EINVAL
    before any device work (include/tcb200.h); the binding rejects non-float64 arrays."""
    import numpy as np
    import paper_2510_12011_b200 as T
    assert T._L.tc_cohort_set_states(None, 0, None, None) == T.TC_EINVAL
    assert T._L.tc_cohort_get_v(None, 0, None, None) == T.TC_EINVAL
    with pytest.raises(ValueError):
        T._ptr_array([np.zeros(4, np.float32)])
    with pytest.raises(ValueError):
        T._ptr_array([np.zeros((4, 2))[:, 0]])


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2510_12011_b200 as T
    with pytest.raises(T.TcError) as ei:
        T.tc_create(T.tc_config_default())
    assert ei.value.status == T.TC_ECUDA


def test_product_does_not_import_oracle():
    """The product package never references the oracle."""
    pkg = os.path.join(ROOT, "paper_2510_12011_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.h" not in src and "liboracle" not in src, f


def test_create_validates_config_before_any_device_work(lib):
    """tc_create rejects an out-of-range configuration with TC_EINVAL before it
    touches a device (include/tcb200.h "Errors"); a valid one -- every PCG
    variant -1..6, including the opt-in single-reduction 6 -- gets past the
    check and, on a box without a GPU, fails with TC_ECUDA (no CPU fallback)."""
    import torch
    import paper_2510_12011_b200 as T
    for bad in (dict(pcg_variant=7), dict(pcg_variant=-2), dict(dt=0.0), dict(theta=1.5), dict(partitions=0),
                dict(model=9), dict(max_iters=-1)):
        with pytest.raises(T.TcError) as e:
            T.tc_create(T.tc_config_default(**bad))
        assert e.value.status == T.TC_EINVAL, bad
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: the valid configurations would create contexts")
    for v in range(-1, 7):
        with pytest.raises(T.TcError) as e:
            T.tc_create(T.tc_config_default(pcg_variant=v))
        assert e.value.status == T.TC_ECUDA, v
