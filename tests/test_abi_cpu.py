"""CPU-side checks of the C-ABI boundary: the library exists, loads, and exports
every entry point include/grab.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "grab.h")
LIB = os.path.join(ROOT, "paper_2604_16402_b200", "libgrab.so")


def declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"GRAB_API\s+(?:int|void|uint64_t|const char\*)\s+(grab_\w+)\s*\(", txt)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("grab_create", "grab_build", "grab_insert", "grab_search", "grab_brute_force",
                 "grab_bucket_select", "grab_import", "grab_read", "grab_select_neighbors", "grab_try_rewire"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(LIB)
    for n in declared():
        assert hasattr(lib, n), n


def test_package_imports_and_binds():
    import paper_2604_16402_b200 as g
    from paper_2604_16402_b200 import _lib
    assert set(_lib._SIGS) <= set(declared())
    assert g.SearchParams().effective_seed_count == 32
