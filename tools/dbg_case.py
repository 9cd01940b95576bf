import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from conftest import load_case
import paper_2410_11415_b200 as k
tc, gold = load_case(sys.argv[1])
W = k.WeightAssignment(gold["w_real"])
tr = k.forward_real(tc, W)
print("fwd ok", flush=True)
g = k.backward(tc, tr)
print("bwd ok", np.array_equal(g, gold["real_grad"]))
