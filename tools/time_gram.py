"""Dev tool: device time of the projector build phases (GF_VERBOSE_SETUP
lines) for prepare() on the device-drawn bench instance, per Gram split
(GF_SYRK: default pre-split f16 copy / f16 in-kernel converters / tf32), a few repetitions each."""
import os, sys
sys.path.insert(0, ".")
os.environ["GF_VERBOSE_SETUP"] = "1"
import numpy as np, torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances

m = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5_000
prob, _ = instances.tall_lasso(m, n, seed=0, dtype=np.float32, device=True)
torch.cuda.synchronize()
ref = None
for split in sys.argv[3].split(",") if len(sys.argv) > 3 else ("pre", "f16", "tf32", "pre", "f16", "tf32"):
    os.environ["GF_SYRK"] = split   # "pre" (any other value): pre-split copy when it fits
    print("split", split, flush=True)
    S = gf.prepare(prob)
    G = np.array(S.projector.gram)
    if ref is None:
        ref = G
    print(f"  max|G - G_first| / max|G| = {np.abs(G - ref).max() / np.abs(ref).max():.3e}", flush=True)
    del S
