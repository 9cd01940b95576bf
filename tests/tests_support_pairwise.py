"""Scalar restatement of the summation order implemented by the CUDA kernels
(paper_2410_11415_b200/csrc/kernels.cuh: np_segment_sum / pw_block /
pw_split), used to prove it equals numpy's add.reduceat."""

import numpy as np


def _pw(a):
    t = a.dtype.type
    n = len(a)
    if n < 8:
        r = t(-0.0)
        for v in a:
            r = t(r + v)
        return r
    if n <= 128:
        r = [a[k] for k in range(8)]
        i = 8
        end = n - n % 8
        while i < end:
            for k in range(8):
                r[k] = t(r[k] + a[i + k])
            i += 8
        res = t(t(t(r[0] + r[1]) + t(r[2] + r[3])) + t(t(r[4] + r[5]) + t(r[6] + r[7])))
        while i < n:
            res = t(res + a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return t(_pw(a[:n2]) + _pw(a[n2:]))


def np_segment_sum_emulated(x):
    x = np.asarray(x)
    if len(x) == 1:
        return x[0]
    return x.dtype.type(x[0] + _pw(x[1:]))
