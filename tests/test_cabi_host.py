"""CPU-only checks of the C ABI library: it loads, exports every symbol the
header declares, and its host-side entry points (no GPU work) agree with the
reference's closed forms and golden counters."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, golden_cases

HEADER = os.path.join(ROOT, "include", "hexgram_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1711_00984_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    return _native.lib()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hxg_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_expected_api():
    names = declared_functions()
    from paper_1711_00984_b200 import _native

    assert set(names) == set(_native.EXPORTED), names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_error_strings_and_version(lib):
    from paper_1711_00984_b200 import _native

    assert lib.hxg_version() >= 100
    for code in (0, -1, -2, -3, -4, -5, -6):
        assert len(_native.error_string(code)) >= 2


def test_dims_match_spaces(lib):
    import paper_1711_00984_b200 as hx

    for space, code in (("H1", 0), ("Hcurl", 1), ("Hdiv", 2), ("L2", 3)):
        for orders in [(1, 1, 1), (2, 3, 4), (6, 6, 6), (12, 12, 12)]:
            assert lib.hxg_dim(code, *orders) == hx.dim(hx.SpaceSignature(space, orders))
    assert lib.hxg_dim(0, 13, 1, 1) == -1  # InvalidOrderError (HXG_MAX_ORDER = 12)
    assert lib.hxg_dim(7, 1, 1, 1) == -2


def test_accumulation_counters_match_reference(lib, golden):
    """hxg_accumulations reproduces the reference's OpCounters.accumulations
    (read from the golden cases the reference produced)."""
    codes = {"H1": 0, "Hcurl": 1, "Hdiv": 2, "L2": 3}
    for c in golden_cases(golden):
        path = {"general": 0, "affine": 1, "extrusion": 2}[c["path"]]
        assert lib.hxg_accumulations(codes[c["space"]], path, *c["orders"], c["L"]) == c["acc"]


def test_python_counters_match_reference(golden):
    from paper_1711_00984_b200.gram import counters

    for c in golden_cases(golden):
        backend = "tensorized" if c["path"] == "general" else "simplified"
        got = counters(c["space"], c["orders"], backend, c["L"] if backend == "tensorized" else None)
        assert got.accumulations == c["acc"]


def test_workspace_size_is_host_only(lib):
    ws = lib.hxg_workspace_size(1, 0, 6, 6, 6, 7, 2048)
    assert ws == 2048 * 12 * 343 * 8  # 12 fields per point for H(curl)
    assert lib.hxg_workspace_size(1, 1, 6, 6, 6, 7, 2048) == 0  # affine path needs none
    big = lib.hxg_workspace_size(0, 0, 2, 2, 2, 3, 10 ** 8)
    assert 0 < big <= 512 * 2 ** 20  # chunked: bounded workspace
    assert lib.hxg_tables_doubles() > 0


def test_table_layout_constants(lib):
    """The Python mirror of the device table layout (used to read tables back)
    matches the library's block size (hxg_plan.h)."""
    from paper_1711_00984_b200 import _native as nat

    assert lib.hxg_tables_doubles() == nat.TAB_TOTAL
