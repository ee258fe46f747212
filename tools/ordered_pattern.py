"""Where the ordered fold differs from the unfused reference (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MF_LEAF_SPLIT"] = "1"
import torch, mf_inputs
import paper_2312_12732_b200 as mf
from paper_2312_12732_b200 import triples
n = int(sys.argv[1]); t = triples.get("strassen-winograd")
A, B = mf_inputs.device_pair("uniform", n, 0)
two = os.environ.pop("MF_LEAF_2CTA", None)
with mf.Plan(t, 2, n) as p:
    ref = p.dgemm(A, B).clone()
if two:
    os.environ["MF_LEAF_2CTA"] = two
with mf.Plan(t, 2, n, fuse_postadd=1) as p:
    C = p.dgemm(A, B).clone()
d = (C != ref)
m = n // 4
print("mismatches", int(d.sum()))
bn = 64 if two and two != "0" else 128
tr = d.reshape(4, m // 128, 128, 4, m // bn, bn)
print("per tile row (all blocks):", tr.sum(dim=(0, 2, 3, 4, 5)).tolist())
print("per tile col:", tr.sum(dim=(0, 1, 2, 3, 5)).tolist())
print("per row in tile (mod 128):", tr.sum(dim=(0, 1, 3, 4, 5)).nonzero().flatten().tolist()[:64])
print("per col in tile:", tr.sum(dim=(0, 1, 2, 3, 4)).nonzero().flatten().tolist()[:64])
print("per block:", d.reshape(4, m, 4, m).sum(dim=(1, 3)).tolist())
