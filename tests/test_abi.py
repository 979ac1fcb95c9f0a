"""C-ABI boundary checks that need no GPU: the shared library builds, loads,
exports every symbol include/radmm_b200.h declares, validates arguments on
the host side, and reports errors through radmm_last_error()."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "radmm_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(radmm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("radmm_run", "radmm_set_operator_c64", "radmm_set_measurement", "radmm_factorize",
                 "radmm_solve_local", "radmm_soft_threshold", "radmm_ctx_create_sharded", "radmm_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(built_lib):
    from paper_2307_08606_b200 import _lib
    for name in declared_functions():
        assert hasattr(built_lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes binding"


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {ROOT}/paper_2307_08606_b200/libradmm_b200.so").read()
    assert "sm_100a" in out


def test_host_side_validation(built_lib):
    from paper_2307_08606_b200 import _lib, api
    h = _lib.Hyper()
    assert built_lib.radmm_hyperparams_default(C.byref(h)) == 0
    assert (h.mu, h.lambda_, h.beta, h.eps_abs, h.eps_rel, h.screening_window, h.screening_tol, h.max_iter) == \
        (3.0, 20.0, 100.0, 1e-4, 1e-2, 5, 1e-5, 1000)
    api.Hyperparams().validate()
    for field, bad in (("mu", 0.0), ("beta", -1.0), ("screening_window", 1), ("max_iter", 0), ("lambda_", -0.1),
                       ("eps_abs", 0.0), ("eps_rel", 0.0), ("screening_tol", -1.0)):
        hp = api.Hyperparams(**{field: bad})
        with pytest.raises(api.InvalidArgument):
            hp.validate()
    api.Hyperparams(lambda_=0.0).validate()  # an unregularized run is legal
    with pytest.raises(api.InvalidArgument) as e:
        api.soft_threshold([1.0], -0.1)
    assert "kappa must be >= 0" in str(e.value)
    with pytest.raises(api.InvalidArgument):
        api.factorize([[1.0]], 0.0, 1.0)


def test_problem_validation_host_side(built_lib):
    import numpy as np
    from paper_2307_08606_b200 import api
    op = api.ForwardOperator.from_matrix(np.zeros((4, 3), complex))
    api.Problem([op], [np.zeros(4)]).validate()
    with pytest.raises(api.InvalidArgument):
        api.Problem([op], [np.zeros(5)]).validate()
    with pytest.raises(api.InvalidArgument):
        api.Problem([], []).validate()
    with pytest.raises(api.InvalidArgument):
        api.Problem([op, api.ForwardOperator.from_matrix(np.zeros((4, 2)))], [np.zeros(4)] * 2).validate()


def test_no_gpu_fails_loudly(built_lib):
    """Without a GPU the compute entry points fail with a CUDA error -- there
    is no silent CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2307_08606_b200 import api
    with pytest.raises(api.CudaError):
        api.Solver(16, 1)
    with pytest.raises(api.CudaError):
        api.soft_threshold([1.0 + 0j], 0.5)


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2307_08606_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, flags=re.M), f
                assert "admm_ref" not in src, f
