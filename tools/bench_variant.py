"""Run bench.py against a variant build of libdifftrans.so (tools/build_variants.py):
    python tools/bench_variant.py paper_2603_00413_b200/variants/libdifftrans_<tag>.so [bench args]
Tuning sweeps only; the product always loads the in-tree library."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if __name__ == "__main__":
    from paper_2603_00413_b200 import _native
    _native.use_library(os.path.abspath(sys.argv[1]))
    sys.argv = [os.path.join(ROOT, "bench.py")] + sys.argv[2:]
    import bench
    bench.main()
