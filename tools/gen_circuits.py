"""Build the benchmark circuits with the REFERENCE
pipeline and store them as ``.npz`` sidecars under ``data/circuits/``.

Runs only in the build container, where ``/root/reference`` is importable:
    python tools/gen_circuits.py A B C D

Recipe:
  A: gen_3cnf(30, 60, 1)   -> compile_cnf -> fold_constants -> layerize -> tensorize
  B: gen_3cnf(45, 100, 1)
  C: gen_3cnf(56, 128, 1)
  D: 256 x gen_3cnf(20, 50, seed) for seeds 1..256, merged by layerize(list)
  Cp: gen_random_nnf(100, 25000, 40, 3, 11) (stress, not d-DNNF)
(``bench.py:65-114``, ``compile.py:101``, ``layerize.py:158``, ``tensorize.py:135``).
The generated files are inputs, not reference code.
"""

import os
import sys
import time

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from laycirc import compile_cnf, fold_constants, layerize, tensorize  # noqa: E402
from laycirc.bench import gen_3cnf, gen_random_nnf  # noqa: E402

from paper_2410_11415_b200.tensorized import save_npz, stats  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data", "circuits")


def mnist_addition(ndigits):
    """Semantic-loss circuit of MNIST addition with `ndigits`-digit numbers
    (PAPER.md:422-424): variable x[p, d] = "digit
    image p shows d"; one-hot ANDs per position, number ANDs per operand,
    pair ANDs, and one OR per possible sum (the roots)."""
    from laycirc import Circuit, Literal
    npos = 2 * ndigits
    c = Circuit(num_vars=npos * 10)
    var = lambda p, d: p * 10 + d + 1
    lit = {}
    for p in range(npos):
        for d in range(10):
            lit[(p, d, True)] = c.add_leaf(Literal(var(p, d)))
            lit[(p, d, False)] = c.add_leaf(Literal(var(p, d), False))
    onehot = {(p, d): c.add_and([lit[(p, d, True)]] + [lit[(p, e, False)] for e in range(10) if e != d])
              for p in range(npos) for d in range(10)}
    top = 10 ** ndigits
    numbers = []
    for side in range(2):
        nums = []
        for n in range(top):
            digits = [(n // 10 ** k) % 10 for k in range(ndigits)]
            kids = [onehot[(side * ndigits + k, digits[k])] for k in range(ndigits)]
            nums.append(c.add_and(kids) if len(kids) > 1 else kids[0])
        numbers.append(nums)
    by_sum = {}
    for a in range(top):
        for b in range(top):
            by_sum.setdefault(a + b, []).append(c.add_and([numbers[0][a], numbers[1][b]]))
    c.set_roots([c.add_or(by_sum[s]) for s in range(2 * top - 1)])
    return c


def build(name):
    t0 = time.time()
    if name == "A":
        circuits = [fold_constants(compile_cnf(gen_3cnf(30, 60, 1)))]
    elif name == "B":
        circuits = [fold_constants(compile_cnf(gen_3cnf(45, 100, 1)))]
    elif name == "C":
        circuits = [fold_constants(compile_cnf(gen_3cnf(56, 128, 1)))]
    elif name == "D":
        circuits = [fold_constants(compile_cnf(gen_3cnf(20, 50, s))) for s in range(1, 257)]
    elif name == "Cp":
        circuits = [gen_random_nnf(100, 25000, 40, 3, 11)]
    elif name == "E":
        circuits = [mnist_addition(2)]
    else:
        raise SystemExit(f"unknown config {name}")
    t1 = time.time()
    tc = tensorize(layerize(circuits))
    t2 = time.time()
    os.makedirs(OUT, exist_ok=True)
    save_npz(tc, os.path.join(OUT, f"{name}.npz"))
    st = stats(tc)
    print(f"{name}: nodes={st['nodes_total']} edges={st['edges_total']} "
          f"layers={len(tc.layers)} K={tc.num_inputs} R={tc.num_roots} "
          f"maxW={max(st['nodes_per_layer'])} compile={t1 - t0:.1f}s layerize+tensorize={t2 - t1:.1f}s",
          flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["A", "B", "C", "D"]:
        build(n)
