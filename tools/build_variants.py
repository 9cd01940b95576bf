"""Build libklay.so variants with extra nvcc -D flags into variants/ (A/B
experiments on the GPU box: KLAY_LIB=variants/<name>.so python bench.py).
usage: python tools/build_variants.py name=-DFLAG[,-DFLAG2] ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402


def one(spec):
    name, _, flags = spec.partition("=")
    d = os.path.join(ROOT, "variants", name)
    os.makedirs(d, exist_ok=True)
    g.build(force=True, extra=[f for f in flags.split(",") if f], out=os.path.join(d, "libklay.so"))
    return name


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for n in ex.map(one, sys.argv[1:]):
            print("built", n)
