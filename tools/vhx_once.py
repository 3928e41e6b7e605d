#!/usr/bin/env python
"""One V^H X call at 16^4 (len 786,432), k = 64, s = $S (default 4): the
ncu capture target for the few-column projection kernels (V^H X, then
X - V H)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_1909_12234_b200 import linalg as LA
    s = int(os.environ.get("S", "4"))
    n = 12 * 16 ** 4
    V = torch.randn((64, n), dtype=torch.complex128, device="cuda")
    X = torch.randn((s, n), dtype=torch.complex128, device="cuda")
    H = LA.vhx(V, X)
    LA.sub_vh(V, H.contiguous(), X)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
