"""Build tuning variants of libdifftrans.so in parallel:
   python tools/build_variants.py tag=DEF1,DEF2 tag2=DEF3 ...
-> paper_2603_00413_b200/variants/libdifftrans_<tag>.so (run with tools/bench_variant.py or tools/sweep.sh)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_00413_b200 import build as B  # noqa: E402


def one(spec):
    tag, defs = spec.split("=", 1)
    out = os.path.join(B.HERE, "variants", f"libdifftrans_{tag}.so")
    B.build(force=True, defines=[d for d in defs.split(",") if d], out=out)
    return out


if __name__ == "__main__":
    with ThreadPoolExecutor(max_workers=4) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
