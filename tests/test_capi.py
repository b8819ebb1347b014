"""The C-ABI library: loads, exports every declared symbol, validates
arguments on the host (no GPU needed for these)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2406_10262_b200 import _lib
from paper_2406_10262_b200.core import DomainError, ShapeError, SolverConfig
from paper_2406_10262_b200.solver import DeviceOptions, _config_c, check

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "nswrank_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(nsw_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 24
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"
    assert b"sm_100a" in lib.nsw_version()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("dtype,n,m,T", [(0, 500, 11, 100), (0, 1000, 21, 100), (0, 2000, 11, 50),
                                          (1, 50, 11, 50), (1, 500, 11, 100), (0, 7, 4, 9), (1, 65, 30, 6),
                                          (0, 4000, 51, 200), (0, 8000, 51, 20), (1, 2000, 51, 20),
                                          (1, 2048, 11, 100), (1, 2000, 51, 500), (0, 4000, 51, 500)])
def test_supported_variants(dtype, n, m, T):
    assert _lib.load().nsw_supported(dtype, n, m, T) == 1
    assert _lib.load().nsw_tiled(dtype, n, m, T) == 1


def test_every_reference_shape_supported_tiles_where_they_fit():
    """Every shape the reference accepts runs (core.py:60-66: 2 <= m <= n);
    shapes no on-chip tile holds run on the streaming fused step."""
    lib = _lib.load()
    assert lib.nsw_supported(1, 4000, 51, 200) == 1     # config 4 in float64
    assert lib.nsw_supported(0, 100, 60, 10) == 1       # m > 52
    assert lib.nsw_supported(0, 9000, 11, 10) == 1      # n > 8192
    assert lib.nsw_supported(0, 5, 6, 10) == 0          # m > n: rejected like the reference
    assert lib.nsw_supported(0, 5, 1, 10) == 0          # m < 2
    assert lib.nsw_tiled(0, 100, 60, 10) == 0           # m > 52: no tile yet
    assert lib.nsw_tiled(0, 9000, 11, 10) == 0          # n > 8192 (16 CTAs x 512 items)
    assert lib.nsw_tiled(1, 4000, 11, 10) == 0          # float64 beyond 2048 items
    assert lib.nsw_tiled(0, 4000, 51, 200) == 1


def _create(rel, expo, n, m, cfg, opt):
    lib = _lib.load()
    h = C.c_void_p()
    return lib.nsw_solver_create(_lib.dptr(rel), _lib.dptr(expo), rel.shape[0], n, m, None, 1, C.byref(cfg),
                                 C.byref(opt), C.byref(h))


def test_create_rejects_bad_shapes_and_config():
    rel = np.full((2, 5), 0.5)
    expo = np.array([1.0, 0.6])
    good = _config_c(SolverConfig())
    opt = DeviceOptions().to_c()
    st = _create(rel, expo, 5, 6, good, opt)           # m > n
    with pytest.raises(ShapeError):
        check(st)
    bad = _config_c(SolverConfig())
    bad.epsilon = -1.0
    with pytest.raises(DomainError):
        check(_create(rel, expo, 5, 3, bad, opt))


@pytest.mark.parametrize("what,message", [
    pytest.param("rel_nan", "relevance contains non-finite", marks=pytest.mark.gpu),
    pytest.param("rel_zero", "relevance entries must lie in (0, 1]", marks=pytest.mark.gpu),
    pytest.param("rel_big", "relevance entries must lie in (0, 1]", marks=pytest.mark.gpu),
    ("expo_inf", "exposure contains non-finite"),
    ("expo_neg", "exposure entries must lie in (0, 1]"), ("expo_rising", "exposure must be non-increasing"),
])
def test_create_checks_values_like_the_reference_types(what, message):
    """A C caller bypasses RelevanceMatrix / ExposureModel: the C ABI applies
    their value checks itself (core.py:85-93, :113-123) -- the exposure on the
    host before any device work, the relevance on the device after its upload."""
    rel = np.full((2, 5), 0.5)
    expo = np.array([1.0, 0.6])
    if what == "rel_nan":
        rel[1, 2] = np.nan
    elif what == "rel_zero":
        rel[0, 0] = 0.0
    elif what == "rel_big":
        rel[1, 4] = 1.5
    elif what == "expo_inf":
        expo[0] = np.inf
    elif what == "expo_neg":
        expo[1] = -0.1
    else:
        expo = np.array([0.5, 0.6])
    with pytest.raises(DomainError, match=message.replace("(", "\\(").replace("]", "\\]")):
        check(_create(rel, expo, 5, 3, _config_c(SolverConfig()), DeviceOptions().to_c()))


def test_python_entry_validates_like_reference():
    from paper_2406_10262_b200 import ExposureModel, ProblemShape, RelevanceMatrix, solve_fair_ranking
    rel = RelevanceMatrix(np.full((3, 4), 0.5))
    with pytest.raises(ShapeError):
        solve_fair_ranking(rel, ExposureModel([1.0, 0.5]), ProblemShape(3, 5, 3), SolverConfig())
    with pytest.raises(ShapeError):
        solve_fair_ranking(rel, ExposureModel([1.0]), ProblemShape(3, 4, 3), SolverConfig())
    with pytest.raises(DomainError):
        RelevanceMatrix(np.zeros((2, 2)))
    with pytest.raises(DomainError):
        SolverConfig(epsilon=0)
