"""Ordered-fold probe: fused (fuse_postadd=1, 2) vs unfused C (flat K6, no
split-K tail), mismatch pattern and per-phase times.
    python tools/fused_probe.py [n] [levels] [triple] [alpha]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MF_LEAF_SPLIT", "1")
import torch  # noqa: E402
import mf_inputs  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402
from paper_2312_12732_b200 import triples  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
name = sys.argv[3] if len(sys.argv) > 3 else "strassen-winograd"
alpha = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
t = triples.get(name)
A, B = mf_inputs.device_pair("uniform", n, 0)
res = {}
two = os.environ.pop("MF_LEAF_2CTA", None)  # applied to the fused modes only
# the reference: one-CTA leaf, flat K6, no split tail
with mf.Plan(t, L, n) as p:
    os.environ["MF_MIX_GENERIC"] = "1"
with mf.Plan(t, L, n) as p:
    ref = p.dgemm(A, B, alpha=alpha).clone()
os.environ.pop("MF_MIX_GENERIC", None)
if two:
    os.environ["MF_LEAF_2CTA"] = two
for mode in (0, 1, 2):
    if mode == 0:
        os.environ["MF_MIX_GENERIC"] = "1"
    with mf.Plan(t, L, n, fuse_postadd=mode, profile=True) as p:
        C = p.dgemm(A, B, alpha=alpha)
        torch.cuda.synchronize()
        p.profile_read(reset=True)
        reps = 3
        for _ in range(reps):
            C = p.dgemm(A, B, alpha=alpha)
        torch.cuda.synchronize()
        ph = p.profile_read(reset=True)
        res[mode] = C.clone()
        print(mode, {k: round(v / reps, 3) if k != "calls" else v for k, v in ph.items()})
    os.environ.pop("MF_MIX_GENERIC", None)
print("vs one-CTA unfused reference: mode0", int((res[0] != ref).sum()), "mode1", int((res[1] != ref).sum()),
      "mode2 max|d|", float((res[2] - ref).abs().max()))
P = t.p ** L
m = n // P
d = (res[1] != res[0])
print("mismatches", int(d.sum()), "of", d.numel())
if d.any():
    blk = d.reshape(P, m, P, m).sum(dim=(1, 3))
    print("per C block:\n", blk.cpu().numpy())
    for i, j in d.nonzero()[:5].tolist():
        print(i, j, res[0][i, j].item(), res[1][i, j].item())
