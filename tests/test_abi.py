"""The drop-in boundary on CPU: the C-ABI library loads, exports exactly what
include/cgvk.h declares, and its host-side logic (VariantConfig::make /
validate, error mapping) follows the reference. No compute calls: without a
GPU the product path must fail loudly rather than fall back."""
import ctypes
import itertools
import os
import re

import pytest

from conftest import ROOT
from oracle import oracle as O
from paper_1905_01549_b200 import cgvk

HEADER = os.path.join(ROOT, "include", "cgvk.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cgvk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for required in ("cgvk_matrix_create_csr", "cgvk_spmv", "cgvk_block_spmv", "cgvk_jacobi",
                     "cgvk_solver_create", "cgvk_solver_step", "cgvk_solver_status",
                     "cgvk_solve", "cgvk_last_error"):
        assert required in fns


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(cgvk.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_library_is_sm100a_native():
    data = open(cgvk.LIB_PATH, "rb").read()
    assert b"sm_100a" in data  # fatbin for sm_100a only


def test_variant_config_make_matches_reference():
    for v in cgvk.Variant:
        c = cgvk.VariantConfig.make(v)
        expected = (cgvk.NuExpression.MEURANT if v in (cgvk.Variant.M, cgvk.Variant.PIPE_PR_M)
                    else cgvk.NuExpression.SIMPLIFIED)
        assert c.nu_expression == expected
        assert c.recompute_nu and c.recompute_w and not c.unsimplified_mu and not c.track_delta


def test_validate_rules_exhaustive():
    """Every flag combination: the C-ABI accepts exactly what the reference's
    VariantConfig::validate accepts (src/variants.cpp:35-47)."""
    for v, nu, rn, rw, um, td in itertools.product(range(7), range(3), (0, 1), (0, 1), (0, 1),
                                                   (0, 1)):
        cfg = cgvk.VariantConfig(cgvk.Variant(v), bool(rn), bool(rw), cgvk.NuExpression(nu),
                                 bool(um), bool(td))
        try:
            cfg.validate()
            ok = True
        except cgvk.InvalidArgument:
            ok = False
        assert ok == O.config_valid(v, nu, rn, rw, um, td), (v, nu, rn, rw, um, td)
        if O.reference_available():
            ref_ok = O.ref_lib().cgvref_config_validate(v, nu, rn, rw, um, td) == 0
            assert ok == ref_ok


def test_reference_validation_examples():
    # tests/test_variants.cpp:301-317
    c = cgvk.VariantConfig.make(cgvk.Variant.HS)
    c.recompute_w = False
    with pytest.raises(ValueError):
        c.validate()
    c = cgvk.VariantConfig.make(cgvk.Variant.HS)
    c.recompute_nu = False
    with pytest.raises(ValueError):
        c.validate()
    c = cgvk.VariantConfig.make(cgvk.Variant.GV)
    c.nu_expression = cgvk.NuExpression.MEURANT
    with pytest.raises(ValueError):
        c.validate()
    c = cgvk.VariantConfig.make(cgvk.Variant.PR)
    c.unsimplified_mu = True
    with pytest.raises(ValueError):
        c.validate()
    c = cgvk.VariantConfig.make(cgvk.Variant.CG_CG)
    c.unsimplified_mu = True
    c.validate()


def test_variant_names_roundtrip():
    for v, name in cgvk.VARIANT_NAMES.items():
        assert cgvk.variant_from_name(name) == v
    assert cgvk.variant_from_name("ppr") == cgvk.Variant.PIPE_PR
    assert cgvk.variant_from_name("nope") is None


def test_no_silent_cpu_fallback_without_gpu():
    if cgvk.device_count_safe() > 0:
        pytest.skip("a GPU is visible")
    from paper_1905_01549_b200 import problems as pb

    A = pb.poisson2d(4)
    with pytest.raises(cgvk.CgvkError):
        cgvk.DeviceMatrix.from_csr(A)
