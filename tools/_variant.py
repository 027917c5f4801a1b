"""Tools only: point the ctypes loader at a diagnostic variant library
(NTF_VARIANT_LIB=<path>, built by tools/build_variant.sh).  The product and
bench.py always load the in-tree release libntf_b200.so."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1409_2383_b200 import _native  # noqa: E402

if os.environ.get("NTF_VARIANT_LIB"):
    _native.LIB_PATH = os.path.abspath(os.environ["NTF_VARIANT_LIB"])
