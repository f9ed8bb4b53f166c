"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/fastgauss_b200.h declares, the Python mirror exposes the
reference's public names, and the product path fails loudly without a GPU."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fastgauss_b200.h")

REFERENCE_ALL = [  # fastgauss/__init__.py:32-58
    "FarFieldExpansion", "LocalExpansion", "KdTree", "Method", "MethodChoice",
    "NodePairGeometry", "PointStore", "ResultVector", "RunConfig", "TraversalCounters",
    "accumulate_far_field", "accumulate_local_direct", "best_method", "build_tree",
    "default_plimit", "dfd_run", "dfdo_run", "dito_post", "dito_run", "eval_far_field",
    "eval_local", "naive_sum", "translate_h2h", "translate_h2l", "translate_l2l",
]


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(fg_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("fg_naive_sum", "fg_tree_build", "fg_moments_refresh", "fg_run",
                     "fg_run_range", "fg_series_accumulate", "fg_best_method"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_1206_6857_b200 import _lib

    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_public_names_mirror_reference():
    import paper_1206_6857_b200 as fg

    for name in REFERENCE_ALL:
        assert hasattr(fg, name), name
    assert sorted(fg.__all__) == sorted(REFERENCE_ALL)


def test_engine_order_cap_is_exported():
    """fg_engine_plimit: the order cap sweeps use when RunConfig.plimit is None
    (12 at D = 3, the reference's default_plimit elsewhere); no GPU needed."""
    import paper_1206_6857_b200 as fg

    assert fg.engine_plimit(3) == 12
    for d in (1, 2, 4, 5, 6, 7, 8, 10, 16):
        assert fg.engine_plimit(d) == fg.default_plimit(d)
    assert "engine_plimit" not in fg.__all__  # the reference's name list is unchanged


def test_host_side_validation_matches_reference():
    import paper_1206_6857_b200 as fg

    with pytest.raises(ValueError):
        fg.PointStore(np.empty((0, 2)))
    with pytest.raises(ValueError):
        fg.PointStore(np.ones((3, 2)), np.array([1.0, 0.0, 2.0]))
    with pytest.raises(ValueError):
        fg.RunConfig(bandwidth=0.0)
    with pytest.raises(ValueError):
        fg.RunConfig(bandwidth=1.0, epsilon=-1.0)
    with pytest.raises(ValueError):
        fg.RunConfig(bandwidth=1.0, algorithm="bogus")
    assert [fg.default_plimit(d) for d in (1, 2, 3, 4, 5, 6, 7, 16)] == [8, 8, 6, 4, 4, 2, 1, 1]


def test_index_sets_match_oracle(oracle):
    from paper_1206_6857_b200.kernel_math import index_set

    for D in (1, 2, 3, 5):
        for p in (1, 2, 4, 8):
            s = index_set(D, p)
            dg, deg, fact, pairs = oracle.iset(D, p)
            np.testing.assert_array_equal(s.digits, dg)
            np.testing.assert_array_equal(s.fact, fact)
            a, b, c = s.shift_pairs
            np.testing.assert_array_equal(np.stack([a, b, c], 1), pairs)


def test_product_path_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1206_6857_b200 as fg

    with pytest.raises(RuntimeError):
        fg.naive_sum(np.zeros((2, 2)), np.zeros((2, 2)), np.ones(2), 0.5)
    with pytest.raises(RuntimeError):
        fg.build_tree(fg.PointStore(np.random.default_rng(0).random((10, 2))))


def test_out_buffers_are_validated_before_the_c_abi():
    """A caller-supplied ``out`` must be float64, C-contiguous, writeable and
    exactly shaped before its raw pointer reaches the C ABI (else ValueError):
    a wrong buffer would otherwise be overrun by the engine's copies."""
    import paper_1206_6857_b200 as fg

    q = np.zeros((5, 2))
    r = np.zeros((4, 2))
    w = np.ones(4)
    bad = [np.zeros(5, np.float32), np.zeros(4), np.zeros((2, 5)),
           np.zeros((5, 2))[:, 0], np.zeros(10)[::2]]
    ro = np.zeros(5)
    ro.flags.writeable = False
    bad.append(ro)
    for out in bad:
        with pytest.raises(ValueError):
            fg.naive_sum(q, r, w, 0.5, out=out)
    with pytest.raises(ValueError):
        fg.naive_sum(q, r, w, [0.5, 1.0], out=np.zeros(5))  # needs (2, 5)
    torch = pytest.importorskip("torch")
    with pytest.raises(ValueError):
        fg.naive_sum(q, r, w, 0.5, out=torch.zeros(5, dtype=torch.float32))
    with pytest.raises(ValueError):
        fg.naive_sum(q, r, w, 0.5, out=torch.zeros(10, dtype=torch.float64)[::2])
