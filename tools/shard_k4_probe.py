"""K4/K6 phase times of an emulated shard (shard_rank r of N, no communicator:
the plan computes its partial C) -- the generated own-slot K4 vs the masked
compiled-in kernel (MF_SHARD_MASKED=1).

    python tools/shard_k4_probe.py [--n 16384] [--N 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import mf_inputs  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--N", type=int, default=8)
    a = ap.parse_args()
    A, B = mf_inputs.device_pair("uniform", a.n, 0, device="cuda:0")
    C = torch.empty_like(A)
    for r in (0, a.N // 2, a.N - 1):
        with mf.Plan(mf.triples.get("strassen-winograd"), 2, a.n, device=0, shard_rank=r,
                     shard_count=a.N, profile=True) as p:
            for _ in range(2):
                p.dgemm(A, B, C)
            torch.cuda.synchronize()
            p.profile_read(reset=True)
            for _ in range(5):
                p.dgemm(A, B, C)
            ph = p.profile_read(reset=True)
        print(json.dumps({"rank": r, "N": a.N, "masked": bool(os.environ.get("MF_SHARD_MASKED")),
                          **{k: round(ph[k] / ph["calls"], 3) for k in p.PHASES}}), flush=True)


if __name__ == "__main__":
    main()
