"""Dev tool: where does a single nonzero A[k][c] land in the tensor-core Gram?"""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1503_08366_b200 as gf

n = 384
for (k, c) in [(0, 0), (0, 1), (0, 4), (1, 0), (8, 0), (0, 130), (3, 5)]:
    A = np.zeros((512, n), np.float32)
    A[k, c] = 1.0
    A[k, 300] = 2.0   # a second column to create an off-diagonal entry (300, c)
    G = gf.build_projector(A).gram - np.eye(n)
    nz = np.argwhere(np.abs(G) > 1e-9)
    print((k, c), "expect", [(c, c, 1.0), (300, 300, 4.0), (300, c, 2.0)], "got",
          [(int(i), int(j), float(G[i, j])) for i, j in nz[:8]], "count", len(nz))
# random check of a full 128x256 tile
rng = np.random.default_rng(0)
A = rng.integers(-3, 4, size=(512, n)).astype(np.float32)
G = gf.build_projector(A).gram
ref = A.astype(np.float64).T @ A + np.eye(n)
print("max abs err", np.abs(G - ref).max(), "ref max", np.abs(ref).max())
d = np.abs(G - ref) > 1e-6
print("bad rows", np.unique(np.nonzero(d)[0])[:20], "bad cols", np.unique(np.nonzero(d)[1])[:20])
