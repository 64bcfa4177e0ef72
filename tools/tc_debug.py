"""Structured cases for the tensor-core DotInc layout (debugging aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1805_11144_b200.engine import tc_dot, PRECISION_TF32, PRECISION_BF16X3

import os
for prec in (PRECISION_TF32, PRECISION_BF16X3):
    name = ("tf32" if prec == PRECISION_TF32 else "bf16x3") + " BN=" + os.environ.get("NENG_TC_BN", "auto")
    m = k = n = 128
    # case 1: A = I -> Y = X
    X = (np.arange(k * n).reshape(k, n) % 251).astype(np.float32)
    Y, _ = tc_dot(np.eye(m, k, dtype=np.float32), X, np.zeros((m, n), np.float32), prec)
    ok = np.array_equal(Y, X)
    print(name, "A=I ok" if ok else "A=I BAD")
    if not ok:
        for (r, c) in [(0, 0), (0, 1), (0, 31), (0, 32), (1, 0), (7, 0), (8, 0), (9, 3), (64, 0)]:
            v = Y[r, c]
            where = np.argwhere(X == v)
            print(f"  Y[{r},{c}]={v} X matches {where[:3].tolist()}")
    # case 2: X = I -> Y = A
    A = (np.arange(m * k).reshape(m, k) % 241).astype(np.float32)
    Y, _ = tc_dot(A, np.eye(k, n, dtype=np.float32), np.zeros((m, n), np.float32), prec)
    ok = np.array_equal(Y, A)
    print(name, "X=I ok" if ok else "X=I BAD")
    if not ok:
        for (r, c) in [(0, 0), (0, 1), (0, 8), (0, 32), (1, 0), (7, 0), (8, 0), (9, 3), (64, 0)]:
            v = Y[r, c]
            where = np.argwhere(A == v)
            print(f"  Y[{r},{c}]={v} A matches {where[:3].tolist()}")
