"""Error growth per recursion level (north_star: "error growth per level
reported as in the paper's error analysis"; PAPER.md L34-35, L97 promise it).

For uniform[-1,1) inputs, seeds s and s+1, the scaled error
max|C - C_ref| / (n * max|A| * max|B|) of mf_dgemm at 0..L levels of
Strassen-Winograd (L = 4, 5 through the level-by-level hybrids) and 1..2 of
Laderman, against two references:
  * the exact definition C_ij = sum_k A_ik B_kj evaluated in x87 extended
    precision (numpy longdouble, 64-bit mantissa) on a sampled 96 x 96 set of
    entries (random rows x random columns) -- the error of each method itself;
  * cuBLAS DGEMM over the whole matrix -- a classical fp64 product whose own
    error (~2e-16 max, ~1e-17 rms scaled) is the floor of that comparison.
Reported: max and RMS scaled error, and the growth ratio per added level.

    python tools/error_growth.py [--n 16384] [--seeds 0,1,2] > profiles/error_growth_r01.json
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


def extended_reference(A, B, rows, cols):
    """C_ij = sum_k A_ik B_kj on entries rows x cols, in extended precision."""
    import numpy as np
    Ar = A[rows].cpu().numpy().astype(np.longdouble)
    Bc = B[:, cols].cpu().numpy().astype(np.longdouble)
    return Ar @ Bc


def sampled_extended(ref, C, rows, cols, den):
    """max / rms scaled error of C on entries rows x cols against ref."""
    import numpy as np
    got = C[rows][:, cols].cpu().numpy().astype(np.longdouble)
    d = np.abs(got - ref)
    return float(d.max()) / den, float(np.sqrt((d * d).mean())) / den


def errors(C, Cref, den):
    mx, ss = 0.0, 0.0
    for r0 in range(0, C.shape[0], 2048):
        d = (C[r0:r0 + 2048] - Cref[r0:r0 + 2048]).abs()
        mx = max(mx, float(d.max()))
        ss += float((d * d).sum())
    return mx / den, (ss / C.numel()) ** 0.5 / den


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--seeds", default="0,1,2")
    a = ap.parse_args()
    out_rows = []
    cases = [("strassen-winograd", L, {}) for L in (0, 1, 2, 3)]
    cases += [("strassen-winograd", 4, {"level_by_level": True, "recurse_levels": 1})]
    if a.n % 32 == 0 and a.n >= 32768:
        cases += [("strassen-winograd", 5, {"level_by_level": True, "recurse_levels": 2})]
    n_ld = a.n if a.n % 9 == 0 else None
    if n_ld:
        cases += [("laderman", L, {}) for L in (1, 2)]
    for seed in (int(s) for s in a.seeds.split(",")):
        A, B = mf_inputs.device_pair("uniform", a.n, 2 * seed, device="cuda:0")
        Cref = torch.matmul(A, B)
        C = torch.empty_like(A)
        den = a.n * float(A.abs().max()) * float(B.abs().max())
        g = torch.Generator().manual_seed(1000 + seed)
        rows = torch.randperm(a.n, generator=g)[:96].sort().values.tolist()
        cols = torch.randperm(a.n, generator=g)[:96].sort().values.tolist()
        xref = extended_reference(A, B, rows, cols)
        for name, L, kw in cases:
            t = None if L == 0 else mf.triples.get(name)
            with mf.Plan(t, L, a.n, device=0, **kw) as p:
                p.dgemm(A, B, C)
                torch.cuda.synchronize()
            mx, rms = errors(C, Cref, den)
            xmx, xrms = sampled_extended(xref, C, rows, cols, den)
            out_rows.append({"triple": name if L else "classical (our levels=0 DGEMM)", "levels": L,
                             "n": a.n, "seed": seed, "max_scaled": mx, "rms_scaled": rms,
                             "ext_max_scaled": xmx, "ext_rms_scaled": xrms})
            print(json.dumps(out_rows[-1]), file=sys.stderr, flush=True)
        del A, B, C, Cref
        torch.cuda.empty_cache()
    # summary: median over seeds; growth = this level / the level below (same
    # family; level 0 is the classical product for both families)
    med = {}
    for r in out_rows:
        med.setdefault((r["triple"], r["levels"]), []).append(r)

    def median(rs, key):
        return sorted(r[key] for r in rs)[len(rs) // 2]
    out = []
    for (name, L), rs in med.items():
        o = {"triple": name, "levels": L, "n": a.n, "bound": 1e-13 * max(1, L)}
        for key in ("ext_max_scaled", "ext_rms_scaled", "max_scaled", "rms_scaled"):
            o[key + "_median"] = median(rs, key)
        o["within_bound"] = o["max_scaled_median"] <= o["bound"] and o["ext_max_scaled_median"] <= o["bound"]
        out.append(o)
    for o in out:
        below = [x for x in out if x["levels"] == o["levels"] - 1 and
                 (x["triple"] == o["triple"] or x["levels"] == 0)]
        o["growth_ext_rms_vs_level_below"] = (o["ext_rms_scaled_median"] / below[0]["ext_rms_scaled_median"]
                                              if below else None)
    print(json.dumps({"what": "scaled error per recursion level, uniform[-1,1) inputs, median over seeds; "
                              "ext_* against the definition in extended precision on 96x96 sampled "
                              "entries, the others against cuBLAS DGEMM over the whole matrix",
                      "seeds": a.seeds, "summary": out, "rows": out_rows}, indent=1))


if __name__ == "__main__":
    main()
