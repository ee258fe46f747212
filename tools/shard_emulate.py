"""Emulated product sharding on one GPU: every rank r of N runs its own plan
(shard_rank = r, shard_count = N, no communicator: the plan computes rank r's
partial C with the real kernels), timed with CUDA events.  max over ranks of
the per-rank step time = the compute part of an N-GPU step; the exchange (the
MF_IN_ROOT slab broadcasts of A and B and the reduce of C, overlapped region
by region in the real run) is NOT included -- its volumes per rank are
reported, not timed (one GPU has no NVLink peer).  SM clocks and throttle
reasons are sampled over the whole run (bench.Clocks).  Emulation, not a
multi-GPU measurement.

    python tools/shard_emulate.py [--n 16384] [--Ns 2,4,8]
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


def step_ms(plan, A, B, C, reps=3):
    for _ in range(2):
        plan.dgemm(A, B, C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.dgemm(A, B, C)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--Ns", default="2,4,8")
    ap.add_argument("--regions", type=int, default=0,
                    help="comm_regions of the real multi-GPU run (8 by default there); 0 = one launch")
    a = ap.parse_args()
    from bench import Clocks
    clocks = Clocks(0)
    clocks.start()
    n = a.n
    A, B = mf_inputs.device_pair("uniform", n, 0, device="cuda:0")
    C = torch.empty_like(A)
    t = mf.triples.get("strassen-winograd")
    with mf.Plan(t, a.levels, n, device=0) as p:
        t1 = step_ms(p, A, B, C)
    fl = 2.0 * n ** 3
    print(json.dumps({"n": n, "N": 1, "step_ms": t1, "tflops": fl / t1 / 1e9}), flush=True)
    for N in (int(x) for x in a.Ns.split(",")):
        per = []
        for r in range(N):
            with mf.Plan(t, a.levels, n, device=0, shard_rank=r, shard_count=N,
                         comm_regions=a.regions) as p:
                per.append(step_ms(p, A, B, C))
            torch.cuda.empty_cache()
        tmax = max(per)
        mat = 8.0 * n * n
        print(json.dumps({"n": n, "N": N, "regions": a.regions, "rank_ms": [round(x, 3) for x in per], "max_ms": tmax,
                          "tflops_compute_only": fl / tmax / 1e9,
                          "efficiency_vs_1gpu": t1 / (N * tmax),
                          "exchange_bytes_per_step": {"broadcast_A_B_from_root": 2 * mat,
                                                      "reduce_C_to_root": mat},
                          "timed": "compute only (every rank's real kernels, max over ranks)"}), flush=True)
    print(json.dumps({"clocks": clocks.stop()}), flush=True)


if __name__ == "__main__":
    main()
