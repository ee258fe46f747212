import sys, os
sys.path.insert(0, "/root/repo")
import torch, mf_inputs
import paper_2312_12732_b200 as mf
A, B = mf_inputs.device_pair("uniform", 64, 0)
with mf.Plan(mf.triples.get("strassen-winograd"), 1, 64) as p:
    for _ in range(3): C = p.dgemm(A, B)
    torch.cuda.synchronize()
print("ok")
