"""The C-ABI library loads and exports every symbol include/tracefront_b200.h declares."""
import re
from pathlib import Path

from paper_2306_08994_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "tracefront_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(tf_\w+)\s*\(", text, re.M)))


def test_header_matches_binding_list():
    assert sorted(_lib.EXPORTS) == declared()


def test_library_exports_all_symbols():
    lib = _lib.load()
    for name in declared():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.tf_build_info()
