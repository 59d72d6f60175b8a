"""C-ABI checks that need no GPU: the library builds, loads, exports every
symbol include/pgrid.h declares, and the binding's signatures cover them."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgrid.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PG_API\s+[\w\s\*]+?\b(pg_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1409_7166_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["pg_create_mesh", "pg_create_csr", "pg_set_sources", "pg_transient",
              "pg_get_voltages", "pg_set_voltages", "pg_destroy", "pg_last_error"]:
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(pg_\w+)", out))
    assert set(declared_symbols()) <= exported
    # nothing else leaks (hidden visibility for internals)
    assert all(s.startswith("pg_") for s in re.findall(r"\sT\s(\w+)", out) if not s.startswith("_"))


def test_binding_signatures_match_header(libpath):
    from paper_1409_7166_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name)


def test_sm100a_code_in_library(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_last_error_without_gpu(libpath):
    from paper_1409_7166_b200 import _lib
    lib = _lib.load()
    import ctypes
    out = ctypes.c_void_p()
    # invalid arguments are rejected before any CUDA call
    rc = lib.pg_create_mesh(0, 1, 1, None, None, None, None, None, 0, None, None, None, 1.0, 0,
                            ctypes.byref(out))
    assert rc == _lib.PG_EINVAL
    assert b"layers" in lib.pg_last_error()
    assert out.value is None


def test_binding_refuses_mismatched_buffer_sizes(libpath):
    # the C side reads / writes exactly the sizes the grid implies: the binding
    # checks every buffer length before the call (no device needed: it raises
    # before reaching the library)
    import numpy as np
    import paper_1409_7166_b200 as P
    n = 2 * 3 * 4
    ok = np.zeros(n)
    with pytest.raises(ValueError):
        P.Grid.mesh(2, 3, 4, ok, ok, np.zeros(n - 1), ok, np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError):
        P.Grid.mesh(2, 3, 4, ok, ok, ok, ok, np.array([0, 1]), np.array([1.0]))
    with pytest.raises(ValueError):
        P.Grid.mesh(2, 3, 4, ok, ok, ok, ok, np.array([0]), np.array([1.0]), lz=np.zeros(3))
    with pytest.raises(ValueError):
        P.Grid.csr(5, np.array([0, 1]), np.array([1]), np.array([1.0, 1.0]), np.zeros(5), np.array([0]),
                   np.array([1.0]))
    g = P.Grid.__new__(P.Grid)           # a handle-less grid: only the size checks run
    g._lib = P.load()
    g.info = lambda: dict(n=n)
    with pytest.raises(ValueError):
        g.voltages(np.empty(n - 1))
    with pytest.raises(ValueError):
        g.set_voltages(np.ones(n + 1))
    with pytest.raises(ValueError):
        g.set_sources(np.array([1, 2]), np.array([0, 3]), np.zeros(3), np.zeros(3))
    with pytest.raises(ValueError):
        g.set_sources(np.array([1]), np.array([0, 3]), np.zeros(2), np.zeros(3))
    with pytest.raises(ValueError):
        g.transient(1e-12, 3, probes=np.array([0, 1]), probe_out=np.empty((3, 2)))


def test_release_memory_rejects_bad_device_without_gpu(libpath):
    # argument check before any CUDA call
    from paper_1409_7166_b200 import _lib
    lib = _lib.load()
    assert lib.pg_release_memory(64) == _lib.PG_EINVAL
    assert b"device" in lib.pg_last_error()
    assert lib.pg_release_memory(-2) == _lib.PG_EINVAL
