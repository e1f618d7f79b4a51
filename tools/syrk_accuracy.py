"""Dev tool: tensor-core Gram error and build time vs the TMEM drain interval."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1503_08366_b200 as gf

A = np.random.default_rng(1).normal(size=(20000, 1300)).astype(np.float32)
A64 = A.astype(np.float64)
ref = A64.T @ A64 + np.eye(A.shape[1])
Abig = torch.randn(200000, 5000, device="cuda", dtype=torch.float32)
for kc in (4096, 1024, 512, 256, 128):
    os.environ["GF_SYRK_KCHUNK"] = str(kc)
    G = gf.build_projector(A).gram
    err = np.abs(G - ref).max() / np.abs(ref).max()
    ts = []
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        P = gf.build_projector(Abig)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        del P
    print(f"kchunk {kc:5d}: rel err {err:.2e}   build_projector 200000x5000: {min(ts):.4f} s")
os.environ["GF_GRAM_SIMT"] = "1"
G = gf.build_projector(A).gram
print("SIMT fp64-accumulate gram rel err", np.abs(G - ref).max() / np.abs(ref).max())
torch.cuda.synchronize(); t0 = time.perf_counter()
P = gf.build_projector(Abig); torch.cuda.synchronize()
print(f"SIMT build_projector 200000x5000: {time.perf_counter() - t0:.4f} s")
