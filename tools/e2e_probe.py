"""Where does the host-buffer stream lose time?  Times K consecutive
mf_dgemm_host_async calls (+ mf_host_sync) for several K, so the steady-state
per-step cost (slope) separates from the pipeline fill/drain (intercept), and
compares with device-resident mf_dgemm.

    python tools/e2e_probe.py [--n 16384] [--levels 2] [--ks 1,2,4,8,16]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import mf_inputs  # noqa: E402
import paper_2312_12732_b200 as mf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--triple", default="strassen-winograd")
    ap.add_argument("--ks", default="1,2,4,8,16")
    a = ap.parse_args()
    n = a.n
    A, B = mf_inputs.device_pair("uniform", n, 0, device="cuda:0")
    C = torch.empty_like(A)
    fl = 2.0 * n ** 3
    with mf.Plan(mf.triples.get(a.triple), a.levels, n, device=0) as plan:
        s = torch.cuda.current_stream()
        for _ in range(2):
            plan.dgemm(A, B, C)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(5):
            plan.dgemm(A, B, C)
        e1.record(s)
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"device_ms": dev_ms, "tflops": fl / dev_ms / 1e9}), flush=True)
        Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Bh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Ch = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        Ah.copy_(A); Bh.copy_(B)
        del A, B, C
        torch.cuda.empty_cache()
        args = (Ah.data_ptr(), n, Bh.data_ptr(), n, Ch.data_ptr(), n)
        plan.dgemm_host_async_ptr(*args)
        plan.host_sync()
        rows = []
        for k in [int(x) for x in a.ks.split(",")]:
            t0 = time.perf_counter()
            for _ in range(k):
                plan.dgemm_host_async_ptr(*args)
            plan.host_sync()
            dt = time.perf_counter() - t0
            rows.append((k, dt))
            print(json.dumps({"k": k, "total_ms": dt * 1e3, "ms_per_step": dt * 1e3 / k,
                              "tflops": fl * k / dt / 1e12}), flush=True)
        t0 = time.perf_counter()
        for _ in range(3):
            plan.dgemm_host_ptr(*args)
        dt = (time.perf_counter() - t0) / 3
        print(json.dumps({"sync_ms": dt * 1e3, "tflops": fl / dt / 1e12}), flush=True)
        if len(rows) >= 2:
            (k0, t0_), (k1, t1_) = rows[-2], rows[-1]
            slope = (t1_ - t0_) / (k1 - k0)
            print(json.dumps({"steady_ms_per_step": slope * 1e3, "fill_drain_ms": (t1_ - slope * k1) * 1e3,
                              "steady_tflops": fl / slope / 1e12}), flush=True)


if __name__ == "__main__":
    main()
