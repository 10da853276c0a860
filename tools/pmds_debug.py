import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2303_03964_b200 as P
rp, col = P.csr_build(10, np.arange(9, dtype=np.int32), np.arange(1, 10, dtype=np.int32))
with P.Layout(10, rp, col, np.zeros((10, 2), np.float32)) as L:
    print(L.pivot_mds(4, 1), L.layout())
