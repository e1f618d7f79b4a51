"""Dev tool: one fp64 prepare (C3 LP 50000 x 20000, device-drawn) for an ncu
capture of the DMMA Gram."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1503_08366_b200 as gf
from paper_1503_08366_b200 import instances
prob, _ = instances.generate(instances.GenSpec("lp", 50000, 20000, 0), device=True)
S = gf.prepare(prob)
torch.cuda.synchronize()
print("ok")
