"""B200-native bitset sort behind the bitsort C ABI (arXiv 1312.0138 reference).

The product is ``lib/libbitsort.so.1`` (built from ``csrc/`` by
``__graft_entry__.build()``): the reference's ``bws_sort`` entry point
(/root/reference/proj/include/bitsort/bitsort.h:89-90) over hand-written sm_100a
kernels. This package holds the Python mirror of that C interface
(:mod:`.capi`), the multi-rank driver (:mod:`.dist`) and the seeded config
generators (:mod:`.datagen`, :mod:`.configs`).
"""
from pathlib import Path

PACKAGE_DIR = Path(__file__).resolve().parent
LIB_DIR = PACKAGE_DIR / "lib"
CSRC_DIR = PACKAGE_DIR / "csrc"

__all__ = ["PACKAGE_DIR", "LIB_DIR", "CSRC_DIR"]
