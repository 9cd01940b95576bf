"""Dump one layer's forward CSR (config C) for real_gather.cu:
python tools/microbench/dump_layer.py <layer 1-based> <out.bin>"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2410_11415_b200.tensorized import load_npz  # noqa: E402

tc = load_npz("data/circuits/C.npz")
l = int(sys.argv[1])
lay = tc.layers[l - 1]
prev = tc.num_inputs if l == 1 else tc.layers[l - 2].width
seg = np.asarray(lay.segments)
off = np.concatenate([[0], np.cumsum(np.bincount(seg, minlength=lay.width))]).astype(np.int32)
with open(sys.argv[2], "wb") as fh:
    np.array([prev, lay.width, len(seg)], np.int32).tofile(fh)
    off.tofile(fh)
    np.asarray(lay.sources, np.int32).tofile(fh)
