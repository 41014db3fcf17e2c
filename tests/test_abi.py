"""CPU-side checks of the C ABI: the library builds, loads and exports every symbol
include/frobinv.h declares, and the host-only entry points behave (no GPU compute)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "frobinv.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b([a-z_][a-z0-9_]*)\s*\(", src)
    skip = {"if", "sizeof", "defined"}
    return sorted({n for n in names if n not in skip and (n.startswith("frob") or n.startswith("zinv") or n.startswith("zhpd"))})


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2208_01239_b200 import frobinv
    return frobinv.load()


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_binding_signatures_match_header(lib):
    from paper_2208_01239_b200 import frobinv
    assert set(frobinv.SIGNATURES) == set(_declared())


def test_host_only_entry_points(lib):
    assert lib.frob_version() == 1
    assert lib.frob_status_string(0) == b"ok"
    assert lib.frob_status_string(2).startswith(b"both")
    ws = lib.frob_inv_workspace_bytes(1024)
    assert ws >= 7 * 1024 * 1024 * 8
    assert lib.frob_inv_workspace_bytes(0) == 0
    assert lib.zinv_lu_workspace_bytes(64) > 0
    assert lib.frob_newton_workspace_bytes(64, 0) > lib.frob_inv_workspace_bytes(64)


def test_invalid_arguments_rejected_without_gpu(lib):
    # argument validation happens before any CUDA call
    st = lib.frob_inv(0, None, 0, None, 0, 0, None, 0, None, None)
    assert st == 4
    st = lib.frob_inv(8, ctypes.c_void_p(4096), 8, ctypes.c_void_p(4096), 8, 0, None, 0, None, None)
    assert st == 4  # X aliases Z
    st = lib.frob_inv(8, ctypes.c_void_p(4096), 8, ctypes.c_void_p(1 << 20), 8, 0, None, 0, None, None)
    assert st == 6  # no workspace
    st = lib.frob_inv_batched(129, 1, ctypes.c_void_p(4096), 129 * 129, ctypes.c_void_p(1 << 20), 129 * 129, 0,
                              ctypes.c_void_p(8192), None, None, 0, None)
    assert st == 4  # n > 128 not supported by the batched kernels


def test_product_has_no_cpu_fallback():
    """The product package never imports the oracle, and refuses CPU tensors."""
    pkg = os.path.join(ROOT, "paper_2208_01239_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
    import torch
    import paper_2208_01239_b200 as fb
    with pytest.raises(ValueError):
        fb.inv(torch.eye(4, dtype=torch.complex128))
