"""Build libaqr_<name>.so variants (compile-time knob overrides) in parallel for tools/perf.py.

  python tools/build_variants.py base:AQR_FUSED_FILTER=0,AQR_LB_SHAR=0 fuse:AQR_LB_SHAR=0
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_21600_b200 import build as B  # noqa: E402


def parse(spec):
    name, _, defs = spec.partition(":")
    d = {}
    for kv in filter(None, defs.split(",")):
        k, _, v = kv.partition("=")
        d[k] = v
    return name, d


if __name__ == "__main__":
    specs = [parse(s) for s in sys.argv[1:]]
    jobs = [lambda: B.build_all()] + [lambda n=n, d=d: B.build_variant(n, d, force=True) for n, d in specs]
    with ThreadPoolExecutor(len(jobs)) as ex:
        for r in ex.map(lambda f: f(), jobs):
            print(r)
