"""Two mf_dgemm_host calls at n=16384 SW^2 (for an ncu launch list of the
host-buffer pipeline's region kernels)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402

n = 16384
Ah = torch.rand((n, n), dtype=torch.float64).pin_memory()
Bh = torch.rand((n, n), dtype=torch.float64).pin_memory()
Ch = torch.empty((n, n), dtype=torch.float64).pin_memory()
with mf.Plan(mf.triples.get("strassen-winograd"), 2, n, device=0) as p:
    for _ in range(2):
        p.dgemm_host_ptr(Ah.data_ptr(), n, Bh.data_ptr(), n, Ch.data_ptr(), n)
torch.cuda.synchronize()
print("ok")
