"""pytest configuration: the `gpu` marker and import paths."""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # the suite needs the built C-ABI library and the C oracle; build them if
    # this checkout has not been built yet (nvcc cross-compiles without a GPU)
    lib = os.path.join(ROOT, "paper_1405_7461_b200", "_lib", "libtrajseek.so")
    orc = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
    if not (os.path.exists(lib) and os.path.exists(orc)):
        import __graft_entry__

        if not os.path.exists(lib):
            __graft_entry__.build_lib()
        __graft_entry__.build_oracle()
