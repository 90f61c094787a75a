"""Host-side checks of the C-ABI library (no GPU needed): the shared library
loads, and it exports every symbol include/nrlsh.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nrlsh.h")
LIB = os.path.join(ROOT, "paper_1809_08782_b200", "libnrlsh.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nrlsh_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libnrlsh():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("nrlsh_build", "nrlsh_query", "nrlsh_exact_topk", "nrlsh_free", "nrlsh_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(libnrlsh):
    missing = [s for s in declared_symbols() if not hasattr(libnrlsh, s)]
    assert not missing, missing


def test_binding_lists_every_export():
    import paper_1809_08782_b200 as P
    assert sorted(P.EXPORTS) == declared_symbols()


def test_default_options_and_error_string(libnrlsh):
    import paper_1809_08782_b200 as P
    opt = P._native.Options()
    P.lib().nrlsh_default_options(ctypes.byref(opt))
    assert opt.eps == 0.01 and opt.scheme == 0 and opt.index_bits_in_budget == 0
    assert isinstance(P.lib().nrlsh_last_error(), bytes)


def test_invalid_arguments_rejected_without_gpu(libnrlsh):
    """Argument validation happens before any device work."""
    import numpy as np
    import paper_1809_08782_b200 as P
    X = np.ones((4, 3), np.float32)
    for bits, m in ((0, 1), (80, 1), (129, 1), (32, 0), (32, 5), (32, 300)):
        with pytest.raises(P.NrlshError) as e:
            P.Index(X, bits, m)
        assert e.value.code == "EINVAL"


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1809_08782_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt, f


def test_binding_validates_arrays_before_the_abi():
    """The ABI takes raw pointers and cannot check dtype, width or shape: the binding
    rejects a wrong dtype, a wrong row width or a wrong output shape before any call."""
    import numpy as np
    import paper_1809_08782_b200 as P
    X = np.ones((8, 3), np.float32)
    with pytest.raises(TypeError):
        P.exact_topk(X.astype(np.float64), X, 2)
    with pytest.raises(ValueError):
        P.exact_topk(X, np.ones((2, 4), np.float32), 2)              # width != d
    with pytest.raises(TypeError):
        P.exact_topk(X, X[:2], 2, out_ids=np.empty((2, 2), np.int32))
    with pytest.raises(ValueError):
        P.exact_topk(X, X[:2], 2, out_ids=np.empty((2, 3), np.int64))
    with pytest.raises(ValueError):
        P.exact_topk(X, X[:2], 2, seed_ids=np.zeros((3, 2), np.int64))
    with pytest.raises(ValueError):
        P.exact_topk(np.asfortranarray(X), X[:2], 2)
    with pytest.raises(TypeError):
        P.Index(X.astype(np.float16), 32, 1)
