"""Small workloads touching every kernel path, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per call):
flattened + Kronecker-factored + generated + table-driven K4/K6, leaf BN=128/64
and the simple leaf, the small-problem cluster kernel, ragged and odd sizes,
bounded-workspace batches, host pipeline, level-by-level, sharded plans, the
ordered and bulk post-addition folds, two loopback ranks (broadcast, region
reduce-scatter)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mf_inputs  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402

T = mf.triples


def run(t, levels, n, **kw):
    A, B = mf_inputs.pair("int8", n, n)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    host_path = kw.pop("host", False)
    with mf.Plan(t, levels, n, **kw) as p:
        if host_path:
            C = p.dgemm_host(A, B)
        else:
            C = p.dgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    assert (C == exact).all(), (t.name if t else "classical", levels, n, kw)


run(None, 0, 256)                        # leaf BN=128/64 decided by wave model
run(None, 0, 33)                         # simple leaf (odd m)
run(T.STRASSEN_WINOGRAD, 1, 400)         # ragged m=200
run(T.STRASSEN_WINOGRAD, 2, 256)         # flattened fixed K4/K6
run(T.STRASSEN_WINOGRAD, 3, 256)         # Kronecker-factored K4/K6
run(T.LADERMAN, 1, 288)
run(T.LADERMAN, 2, 144)                  # factored, p=3
os.environ["MF_MIX_GENERIC"] = "1"
run(T.STRASSEN_WINOGRAD, 2, 256)         # plan-time generated K4/K6 (NVRTC)
os.environ["MF_MIX_NOJIT"] = "1"
run(T.STRASSEN_WINOGRAD, 2, 256)         # table-driven K4/K6 (grouped / term lists)
del os.environ["MF_MIX_NOJIT"]
del os.environ["MF_MIX_GENERIC"]
run(T.STRASSEN_WINOGRAD, 1, 64)          # small problem: one cluster launch (DMMA, DSMEM pushes)
run(T.LADERMAN, 1, 36)                   # small problem, fma leaf (m = 12)
run(T.STRASSEN_WINOGRAD, 2, 512, max_workspace=3 * 5 * 128 * 128 * 8)  # batches
run(T.STRASSEN_WINOGRAD, 2, 1024, host=True)   # host pipeline (regions, 4 streams)
run(T.STRASSEN_WINOGRAD, 2, 256, level_by_level=True)
n = 1024
A, B = mf_inputs.pair("int8", n, 1)
tot = np.zeros((n, n))
for r in range(3):                        # split sharding
    with mf.Plan(T.STRASSEN_WINOGRAD, 2, n, shard_rank=r, shard_count=3) as p:
        tot += p.dgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
assert (tot == (A.astype(np.int64) @ B.astype(np.int64))).all()
run(T.STRASSEN_WINOGRAD, 2, 512, fuse_postadd=1)   # ordered fold (flags, ticket order)
run(T.STRASSEN_WINOGRAD, 2, 400, fuse_postadd=1)   # ordered fold, ragged m=100 (scalar path)
run(T.STRASSEN_WINOGRAD, 2, 512, fuse_postadd=2)   # bulk-reduction fold
# two loopback ranks (threads): slab broadcasts of A, B under K4, region-wise
# reduce-scatter of C (MF_OUT_ROWSLAB), summation kernel
import threading  # noqa: E402
n = 1024
A, B = mf_inputs.pair("int8", n, 2)
comms = mf.loop_comm_create(2)
out = [None, None]


def rank(r):
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st), mf.Plan(T.STRASSEN_WINOGRAD, 2, n, comm=comms[r], shard_rank=r, shard_count=2,
                                        input_mode=mf.IN_ROOT, output_mode=mf.OUT_ROWSLAB) as p:
        C = p.dgemm(torch.from_numpy(A).cuda() if r == 0 else None,
                    torch.from_numpy(B).cuda() if r == 0 else None, stream=st)
        st.synchronize()
        out[r] = C.cpu().numpy()


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
for c in comms:
    mf.comm_destroy(c)
assert (np.concatenate(out) == (A.astype(np.int64) @ B.astype(np.int64))).all()
torch.cuda.synchronize()
print("sanitize smoke ok")
