"""Ordered fold (or, FUSE=0, the unfused leaf) against the unfused one-CTA
result, launch after launch: mismatch counts per launch and, with PATTERN=1,
where in the tile the first bad launch differs.  Second argument: a list of
modes, bit 1 = two CTAs per SM (MF_LEAF_2CTA=1).  The experiment build that
found the leaf's ring-release race had more bits (profiles/leaf_ring_race_r02.log).
    REPS=30 python tools/ordered_dbg.py 8192,16384 1,0
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MF_LEAF_SPLIT"] = "1"
import torch, mf_inputs
import paper_2312_12732_b200 as mf
from paper_2312_12732_b200 import triples
t = triples.get("strassen-winograd")
for n in [int(x) for x in sys.argv[1].split(",")]:
    A, B = mf_inputs.device_pair("uniform", n, 0)
    os.environ["MF_LEAF_2CTA"] = "0"
    os.environ.pop("MF_LEAF_DBG", None)
    with mf.Plan(t, int(os.environ.get("LEVELS", "2")), n) as p:
        ref = p.dgemm(A, B).clone()
    for dbg in [int(x) for x in sys.argv[2].split(",")]:
        os.environ["MF_LEAF_DBG"] = str(dbg)
        os.environ["MF_LEAF_2CTA"] = "1" if dbg & 1 else "0"
        bad = []
        with mf.Plan(t, int(os.environ.get("LEVELS", "2")), n, fuse_postadd=int(os.environ.get("FUSE", "1"))) as p:
            for _ in range(int(os.environ.get("REPS", "6"))):
                C = p.dgemm(A, B)
                torch.cuda.synchronize()
                d = C != ref
                bad.append(int(d.sum()))
                if bad[-1] and os.environ.get("PATTERN") and sum(b > 0 for b in bad) == 1:
                    m = n // 4
                    r = d.reshape(4, m // 128, 128, 4, m, ).sum(dim=(0, 1, 3, 4)).nonzero().flatten().tolist()
                    c = d.reshape(4, m, 4, m // 64, 64).sum(dim=(0, 1, 2, 3)).nonzero().flatten().tolist()
                    print(f"  rows in tile with mismatches: {r[:8]}..{r[-4:]} ({len(r)}), cols in tile: {len(c)}", flush=True)
                    print("  mismatching tiles (block, tm, tn):", (d.reshape(4, m // 128, 128, 4, m // 64, 64).sum(dim=(2, 5)) > 0).nonzero().tolist()[:12], flush=True)
        print(f"n={n} dbg={dbg}: launches {len(bad)}, bad launches {sum(b > 0 for b in bad)}, mismatches {sum(bad)} {bad if sum(bad) else ''}", flush=True)
