"""Run GPU tests against a variant build of libdifftrans.so (tools/build_variants.py):
    python tools/test_variant.py paper_2603_00413_b200/variants/libdifftrans_<tag>.so [pytest args]
Tuning sweeps only (parity of a candidate before it becomes the default)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    import pytest

    from paper_2603_00413_b200 import _native
    _native.use_library(os.path.abspath(sys.argv[1]))
    os.chdir(ROOT)
    sys.exit(pytest.main(sys.argv[2:]))
