"""Where a leaf tile's time goes outside the DMMA stream: per-CTA globaltimer
stamps (entry, first stage landed, end of k loop, end of epilogue) and the SM
id, from a diagnostic build of mf_leaf.cu with -DMF_LEAF_TRACE (not the
product build).  Build the diagnostic library into a copy of the package, e.g.

    nvcc ... -DMF_LEAF_TRACE -c mf_leaf.cu -o mf_leaf_trace.o   (flags as tools/build_mf.py)
    nvcc ... -shared -cudart static -o <copy>/paper_2312_12732_b200/libmf.so <other objs> mf_leaf_trace.o

and run this script from the copy.  Results: profiles/leaf_trace_r01.json.
"""
import ctypes, os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import mf_inputs
import paper_2312_12732_b200 as mf
lib = ctypes.CDLL(mf.LIB_PATH)
for n, L in ((16384, 2), (4096, 1), (16384, 3)):
    A, B = mf_inputs.device_pair("uniform", n, 0, device="cuda:0")
    C = torch.empty_like(A)
    with mf.Plan(mf.triples.get("strassen-winograd"), L, n, device=0) as p:
        for _ in range(2):
            p.dgemm(A, B, C)
        torch.cuda.synchronize()
        nt = 65536
        buf = np.zeros((nt, 5), dtype=np.uint64)
        assert lib.mf_debug_leaf_trace(buf.ctypes.data_as(ctypes.c_void_p), nt) == 0
    t = buf[buf[:, 0] > 0].astype(np.float64)
    ncta = len(t)
    t0 = t[:, 0].min()
    pro = t[:, 1] - t[:, 0]; loop = t[:, 2] - t[:, 1]; epi = t[:, 3] - t[:, 2]
    # gaps between consecutive CTAs on the same SM
    gaps = []
    for sm in np.unique(t[:, 4]):
        r = t[t[:, 4] == sm]
        r = r[np.argsort(r[:, 0])]
        gaps += list(r[1:, 0] - r[:-1, 3])
    gaps = np.array(gaps)
    span = t[:, 3].max() - t0
    out = {"n": n, "levels": L, "ctas": ncta, "span_ms": span / 1e6,
           "prologue_us": [float(np.median(pro)) / 1e3, float(np.mean(pro)) / 1e3],
           "kloop_us": [float(np.median(loop)) / 1e3, float(np.mean(loop)) / 1e3],
           "epilogue_us": [float(np.median(epi)) / 1e3, float(np.mean(epi)) / 1e3],
           "sm_gap_us": [float(np.median(gaps)) / 1e3, float(np.mean(gaps)) / 1e3, float(np.percentile(gaps, 95)) / 1e3]}
    print(json.dumps(out), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
