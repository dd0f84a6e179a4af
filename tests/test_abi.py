"""The C-ABI library loads without a GPU and exports every symbol include/osm.h declares (no compute calls)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "osm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(osm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_8b_calls():
    syms = declared_symbols()
    for s in ["osm_create", "osm_upload_density", "osm_decompose", "osm_set_robin", "osm_assemble", "osm_solve",
              "osm_get_history", "osm_get_solution", "osm_get_trace", "osm_get_csr", "osm_get_interface_map",
              "osm_last_error", "osm_destroy", "osm_abi_version"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_2112_03851_b200 as P

    lib = ctypes.CDLL(P.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert sorted(P.ABI_SYMBOLS) == declared_symbols()
    assert P.abi_version() == 2


def test_no_oracle_in_product_path():
    """The product package never imports oracle/ (the oracle is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2112_03851_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, flags=re.M), f
