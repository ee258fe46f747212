"""Launch-to-launch determinism stress of the deterministic paths: K launches of
one plan on the same inputs, each result compared bitwise with the first (the
unfused path and the ordered fold are deterministic by construction; a race in
the leaf's ring or the fold's flags shows as a differing launch).
    python tools/determinism_stress.py [K]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mf_inputs  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 50
CASES = [  # (label, triple, levels, n, plan kwargs, env)
    ("SW2 n=16384 unfused (one CTA/SM)", "strassen-winograd", 2, 16384, {}, {}),
    ("SW2 n=16384 ordered fold (two CTAs/SM)", "strassen-winograd", 2, 16384, {"fuse_postadd": 1}, {}),
    ("SW3 n=8192 unfused (m=1024, two CTAs/SM)", "strassen-winograd", 3, 8192, {}, {}),
    ("SW1 n=4096 unfused (config 2, split-K tail)", "strassen-winograd", 1, 4096, {}, {}),
    ("LD1 n=13824 unfused", "laderman", 1, 13824, {}, {}),
    ("SW3 n=16384 ordered fold", "strassen-winograd", 3, 16384, {"fuse_postadd": 1}, {}),
]
for label, name, levels, n, kw, env in CASES:
    os.environ.update(env)
    A, B = mf_inputs.device_pair("uniform", n, 7)
    k = K if n <= 8192 else max(8, K // 4)
    t0 = time.time()
    with mf.Plan(mf.triples.get(name), levels, n, **kw) as p:
        ref = p.dgemm(A, B).clone()
        bad = []
        for i in range(k):
            if not torch.equal(p.dgemm(A, B), ref):
                bad.append(i)
    print(f"{label}: {k} launches, {len(bad)} differ {bad[:10]} ({time.time() - t0:.1f} s)", flush=True)
    del A, B, ref
    torch.cuda.empty_cache()
