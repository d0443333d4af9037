"""The C-ABI library loads and exports every symbol include/hfpg.h declares (no GPU calls)."""
import os
import re

from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hfpg.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|void)\s+(hfpg_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2605_13343_b200 import _native as N
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(N.lib, s), s
    assert sorted(N.EXPORTED) == syms, set(N.EXPORTED) ^ set(syms)


def test_library_is_the_in_tree_sm100a_build():
    from paper_2605_13343_b200 import _native as N
    assert os.path.dirname(N.SO_PATH) == os.path.join(ROOT, "paper_2605_13343_b200")
    assert b"sm_100a" in N.lib.hfpg_version()
    maps = open("/proc/self/maps").read()
    assert N.SO_PATH in maps


def test_errors_map_to_reference_exceptions(H):
    import pytest
    with pytest.raises(ValueError):
        H.build_partition(1000, 128)  # partition.cpp:10-11
    with pytest.raises(ValueError):
        H.build_partition(128 * 3, 128)  # K = 3
    with pytest.raises(RuntimeError):
        H.read_checkpoint("/nonexistent/x.hftc")
