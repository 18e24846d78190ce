"""The C-ABI library loads and exports every symbol include/bddc_b200.h declares; the GPU
entry points fail loudly (no CPU fallback) when no device is visible."""
import ctypes as C

import pytest

from conftest import has_gpu
from paper_2410_14786_b200 import _lib
from paper_2410_14786_b200 import BddcError, Problem, Preconditioner


def test_library_exports_header_symbols():
    syms = _lib.header_symbols()
    assert len(syms) >= 30
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert _lib.lib().bddc_abi_version() == 3
    assert _lib.lib().bddc_kernel_launches() == 0  # nothing launched on a CPU-only host


def test_default_options():
    o = _lib.GpuOptions()
    _lib.lib().bddc_default_gpu_options(C.byref(o))
    assert o.coarse_rel_tolerance == 1e-12 and o.coarse_max_iterations == 500  # preconditioner.hpp:42
    s = _lib.SolverOptions()
    _lib.lib().bddc_default_solver_options(C.byref(s))
    assert s.rel_tolerance == 1e-8 and s.max_iterations == 1000  # pcg.hpp:17-22


@pytest.mark.skipif(has_gpu(), reason="checks the no-device failure path")
def test_no_device_fails_loudly():
    p = Problem.poisson(8, 2)
    with pytest.raises(BddcError) as e:
        Preconditioner(p)
    assert e.value.code == _lib.ERR_NO_DEVICE
    assert "no CPU fallback" in str(e.value)


def test_null_arguments_are_errors():
    L = _lib.lib()
    assert L.bddc_gpu_apply(None, None, None) == _lib.ERR_INVALID_ARGUMENT
    assert b"null" in L.bddc_last_error()
