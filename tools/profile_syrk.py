"""Dev tool: one fp32 Gram build (for ncu captures of the tensor-core SYRK)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1503_08366_b200 as gf
m = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
A = torch.randn(m, n, device="cuda", dtype=torch.float32)
P = gf.build_projector(A)
torch.cuda.synchronize()
print("ok")
