"""Bench: effective fp64 TFLOPS (2n^3/t) of the Matrix Flow hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mf|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (product-sharded, NCCL)

Workload (BASELINE.json metric / config 3): n = 16384 fp64, two-level
Strassen-Winograd executed as one level of the flattened <4,4,4;49> triple
(49 leaf products of 4096^3).  A step = one mf_dgemm call (pre-add A, pre-add
B, batched leaf DGEMM, post-add) on inputs already resident in HBM; inputs are
2.1 GB each (> 126 MB L2), so no L2 flush is needed between steps.  With N > 1
ranks the 49 products are sharded across ranks and the partial C is summed onto
rank 0 with NCCL (strong scaling: the same problem on N GPUs).

Printed (rank 0, one JSON line): value, ms_per_step, the leaf kernel's live
roofline, classical baselines in the same run (cuBLAS DGEMM and our own
levels=0 leaf), the max scaled error against cuBLAS, the end-to-end number
through mf_dgemm_host (host buffers, copies inside the timed region), the
clocks seen during the timed region and the CPU-oracle baseline.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective fp64 TFLOPS (2n^3/t) at n=16384 vs classic DGEMM; max scaled error"
UNIT = "TFLOPS"
CPU_SAMPLE_N = 4096  # reference-arm step: same triple and levels at n/4 (1/64 of the work)
CPU_BASELINE_N = 8192  # cpu_baseline leg: n/2 (1/8 of the work, ~15-20 s on 16 cores)


def cpu_sample_n(a, div=4, cap=CPU_SAMPLE_N):
    """n of a bounded oracle sample: n/div capped at `cap`, divisible by p^levels."""
    p = 1
    for part in a.triple.split("(x)"):
        p *= {"laderman": 3, "classical-p3": 3}.get(part, 2)
    p = p ** a.levels
    ns = min(max(a.n // div, p), cap)
    return max(p, ns - ns % p)


# BASELINE.json configs as presets: (n, triple, levels)
CONFIGS = {
    "c1-sw1-64": (64, "strassen-winograd", 1),
    "c2-sw1-4096": (4096, "strassen-winograd", 1),
    "c3-sw2-16384": (16384, "strassen-winograd", 2),      # the metric's config (default)
    "c3b-sw1-16384": (16384, "strassen-winograd", 1),
    "c4a-ld1-13824": (13824, "laderman", 1),
    "c4b-sw2-13824": (13824, "strassen-winograd", 2),     # <4,4,4;49> = SW (x) SW
    "c5-sw2-32768": (32768, "strassen-winograd", 2),      # config 5's problem (1-GPU leg)
    # deeper flattening at the same sizes (beyond the configs' level counts)
    "x-sw3-16384": (16384, "strassen-winograd", 3),
    "x-ld2-13824": (13824, "laderman", 2),
    "x-sw3-32768": (32768, "strassen-winograd", 3),
    # mixed chains <6,6,6;161>: 2-then-3 and 3-then-2
    "x-swld-13824": (13824, "strassen-winograd(x)laderman", 1),
    "x-ldsw-13824": (13824, "laderman(x)strassen-winograd", 1),
    # bounded workspace (NEXT-3): n where the all-products workspace does not fit in HBM
    "x-sw2-49152-bounded": (49152, "strassen-winograd", 2),
    # four levels: one level of SW run level by level, each of its 7 products a
    # flattened SW^3 child plan (343 leaves in one launch); mf_options.recurse_levels
    "x-sw4-16384-hybrid": (16384, "strassen-winograd", 4),
    "x-sw4-32768-hybrid": (32768, "strassen-winograd", 4),
    # five levels at n=32768: two levels one at a time (49 products), each a
    # flattened SW^3 child at n=8192 (m = 1024)
    "x-sw5-32768-hybrid": (32768, "strassen-winograd", 5),
}
# presets run level by level with this many recursive top levels
PRESET_RECURSE = {"x-sw4-16384-hybrid": 1, "x-sw4-32768-hybrid": 1, "x-sw5-32768-hybrid": 2}
# presets that need a workspace cap (GB): 49152^2 * 8 B = 19.3 GB per matrix;
# all 129 T/S/P blocks (1.2 GB each) would need 156 GB on top of A, B, C, C_ref
PRESET_WORKSPACE_GB = {"x-sw2-49152-bounded": 85.0}


def resolve_triple(mf, name):
    """A catalog name, or 'outer(x)inner' for a one-level mixed chain."""
    if "(x)" in name:
        o, i = name.split("(x)")
        return mf.triples.kron(mf.triples.get(o), mf.triples.get(i))
    return mf.triples.get(name)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=sorted(CONFIGS), default=None,
                    help="BASELINE config preset (overrides --n/--triple/--levels)")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mf", "reference"], default="mf")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--triple", default="strassen-winograd")
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-classical", action="store_true")
    ap.add_argument("--level-by-level", action="store_true",
                    help="ablation: the paper's recursion instead of the flattened triple")
    ap.add_argument("--max-workspace-gb", type=float, default=0.0,
                    help="cap the plan workspace (bounded schedule); 0 = unlimited")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip timing the variants (same n: one more level; fused post-addition)")
    ap.add_argument("--recurse-levels", type=int, default=0,
                    help="with --level-by-level: top levels run one at a time (0 = all but the "
                         "last); the rest run as one flattened child plan")
    ap.add_argument("--leaf", choices=["dmma", "cublas", "simple"], default="dmma",
                    help="leaf GEMM: our TMA+DMMA kernel (default) or the cuBLAS ablation")
    ap.add_argument("--comm-regions", type=int, default=0,
                    help="sharded runs: row regions whose C rows are reduced while the next "
                         "region computes (0 = library default)")
    ap.add_argument("--input-mode", choices=["root", "replicated"], default="root",
                    help="sharded runs: A and B on rank 0 only, broadcast by row slabs inside "
                         "the timed step (default), or already replicated on every rank")
    ap.add_argument("--fuse", type=int, nargs="?", const=1, default=0, choices=[0, 1, 2],
                    help="fold the post-additions into the leaf epilogue (mf_options.fuse_postadd): "
                         "1 = ordered fold (bitwise the unfused result), 2 = bulk f64 reductions")
    a = ap.parse_args()
    if a.config:
        a.n, a.triple, a.levels = CONFIGS[a.config]
        if a.config in PRESET_WORKSPACE_GB and not a.max_workspace_gb:
            a.max_workspace_gb = PRESET_WORKSPACE_GB[a.config]
        if a.config in PRESET_RECURSE:
            a.level_by_level, a.recurse_levels = True, PRESET_RECURSE[a.config]
    return a


def workload_name(a):
    mode = "level by level" if getattr(a, "level_by_level", False) else "flattened"
    if getattr(a, "level_by_level", False) and getattr(a, "recurse_levels", 0):
        r = a.recurse_levels
        mode = (f"{r} top level(s) one at a time, each product a flattened "
                f"{a.levels - r}-level child")
    if getattr(a, "fuse", 0):
        mode += (", post-additions folded into the leaf epilogue in ascending q (ordered fold)"
                 if a.fuse == 1 else ", post-additions fused by bulk f64 reductions into C")
    if getattr(a, "leaf", "dmma") != "dmma":
        mode += f", {a.leaf} leaf (ablation)"
    return f"n={a.n} fp64, {a.levels}-level {a.triple} ({mode}, {_rank(a) ** a.levels} leaf products)"


def ceiling(levels):
    """north_star: scaled error <= 1e-13 per recursion level used (tests/bounds.py)."""
    return 1e-13 * max(1, levels)


def model_guard(levels):
    """10x the measured error model ~1e-16 * 2^L (profiles/error_growth_r01.json)."""
    return 10 * 1e-16 * 2.0 ** max(1, levels)


def step_roofline(a, n, ms, world, peak):
    R = _rank(a)
    p = 1
    for part in a.triple.split("(x)"):
        p *= {"laderman": 3, "classical-p3": 3}.get(part, 2)
    alg = (R / p ** 3) ** a.levels * 2.0 * n ** 3  # R^L (n/p^L)^3 multiply-adds x 2
    eff = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
    alg_tf = alg / (ms * 1e-3) / 1e12
    return {"effective_tflops": eff, "algorithmic_tflops": alg_tf, "n_gpus": world,
            "peak_tflops": peak * world, "effective_frac_of_peak": eff / (peak * world),
            "algorithmic_frac_of_peak": alg_tf / (peak * world),
            "note": "algorithmic = the leaf multiplications the method performs, R^L * 2 (n/p^L)^3, "
                    "per second of the whole step (additions and exchange included)"}


def launches_per_step(a):
    """Our kernels per mf_dgemm: K4, K4, K5, K6 per flattened level (K6 folded
    into K5 with --fuse); level by level: the top level's K4, K4, K6 around R
    child calls."""
    if a.levels == 0:
        return 1
    if (a.n <= 64 and _rank(a) ** a.levels <= 64 and not a.fuse and not a.level_by_level
            and a.leaf == "dmma" and not a.max_workspace_gb and not os.environ.get("MF_TINY_OFF")):
        return 1  # the whole level as one cluster launch (mf_tiny.cu)
    flat = 3 if a.fuse else 4
    if not a.level_by_level or a.levels < 2:
        return flat
    r = a.recurse_levels if 0 < a.recurse_levels < a.levels else a.levels - 1
    count = flat
    for _ in range(r):
        count = 3 + _rank(a) * count
    return count


def _rank(a):
    ranks = {"strassen-winograd": 7, "paper-strassen": 7, "strassen-1969": 7, "laderman": 23,
             "classical-p2": 8, "classical-p3": 27}
    r = 1
    for part in a.triple.split("(x)"):
        r *= ranks[part]
    return r


def config(a, world):
    return {"workload": workload_name(a), "preset": a.config, "n": a.n, "triple": a.triple,
            "levels": a.levels, "max_workspace_gb": a.max_workspace_gb or None,
            "leaf_products": _rank(a) ** a.levels, "inputs": "uniform[-1,1) fp64, seeds 0/1",
            "l2": ("inputs larger than L2 (8n^2 = %.1f GB per matrix); no flush" % (8 * a.n ** 2 / 1e9)
                   if 8 * a.n ** 2 > 126e6 else "inputs fit in L2 (%.1f MB per matrix); not flushed"
                   % (8 * a.n ** 2 / 1e6)),
            "parallelism": (f"product-sharded x{world}: "
                            + ("A, B on rank 0 only, broadcast by row slabs under K4 inside the "
                               "timed step" if getattr(a, "input_mode", "root") == "root"
                               else "A, B replicated before the timed step")
                            + "; partial C reduced onto rank 0 region by region (NCCL)")
            if world > 1 else "single GPU"}


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        time.sleep(0.3)

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.15)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def fp64_peak():
    """Measured FP64 DMMA peak (tools/peaks_fp64.cu on this pool's B200, committed
    under profiles/).  MEASURED_PEAKS.json carries no FP64 figure."""
    path = os.path.join(ROOT, "profiles", "peaks_fp64.json")
    with open(path) as f:
        d = json.load(f)
    return float(d["dmma_tflops"]), "measured: tools/peaks_fp64.cu DMMA m8n8k4, profiles/peaks_fp64.json"


def leaf_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_leaf.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    return None


def oracle_triple(a):
    import oracle
    parts = [oracle.catalog(x) for x in a.triple.split("(x)")]
    t = parts[0]
    for x in parts[1:]:
        t = oracle.kron(t, x)
    return t


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(a):
    """The oracle (or_fmm: plain C interpreter of Eq. "strassen", OpenMP over
    rows) on the host cores: same triple and levels at n/2 (<= CPU_BASELINE_N),
    about 10-30 s of CPU work."""
    import numpy as np
    import mf_inputs
    import oracle
    n = cpu_sample_n(a, div=2, cap=CPU_BASELINE_N)
    A, B = mf_inputs.pair("uniform", n, 0)
    t = oracle_triple(a)
    # load the library and start its OpenMP pool (~1 s in a process that
    # imported torch) outside the timed region
    oracle.classical(A[:64, :64], B[:64, :64])
    t0 = time.perf_counter()
    oracle.fmm(A, B, t, a.levels)
    dt = time.perf_counter() - t0
    nc = min(n, 4096)  # O3, the plain classical loop, on the same cores
    t0 = time.perf_counter()
    oracle.classical(A[:nc, :nc], B[:nc, :nc])
    dtc = time.perf_counter() - t0
    return {"value": 2.0 * n ** 3 / dt / 1e12, "unit": UNIT, "cores": oracle.num_threads(),
            "kind": "oracle", "cpu_model": _cpu_model(),
            "classical_o3": {"n": nc, "seconds": dtc, "value": 2.0 * nc ** 3 / dtc / 1e12,
                             "unit": UNIT},
            "sample": f"or_fmm({a.triple}, levels={a.levels}) full call at n={n} "
                      f"({(n / a.n) ** 3:.4g} of the n={a.n} work), {dt:.2f} s; value = 2n^3/t at n={n}",
            "seconds": dt}


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, each step one bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import mf_inputs
    import oracle
    n = cpu_sample_n(a)
    A, B = mf_inputs.pair("uniform", n, 0)
    t = oracle_triple(a)
    for _ in range(a.warmup):
        oracle.fmm(A, B, t, a.levels)
    times = []
    for _ in range(a.steps):
        t0 = time.perf_counter()
        oracle.fmm(A, B, t, a.levels)
        times.append(time.perf_counter() - t0)
    dt = sum(times) / len(times)
    value = 2.0 * n ** 3 / dt / 1e12
    sample = (f"or_fmm({a.triple}, levels={a.levels}) full call at n={n} per step "
              f"({(n / a.n) ** 3:.4g} of the n={a.n} work); value = 2n^3/t at n={n}")
    emit({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config(a, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


# ------------------------------------------------------------------ output
_JSON_FD = None


def _claim_stdout():
    """Route fd 1 to stderr for the whole run (NCCL, torch or libraries may print
    banners) and keep the real stdout for the one JSON line."""
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def emit(obj):
    line = (json.dumps(obj) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(line.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, line)


# ------------------------------------------------------------------ main arm
def main():
    _claim_stdout()
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import torch.distributed as dist
    import mf_inputs
    import paper_2312_12732_b200 as mf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    # MF_BENCH_DIST=1 runs the distributed path even at world size 1 (process
    # group, NCCL communicator through libmf, reduce of C, max-over-ranks
    # timing) -- the multi-GPU plumbing, checkable on a single GPU
    distributed = world > 1 or os.environ.get("MF_BENCH_DIST") == "1"
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
        obj = [mf.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = mf.nccl_comm_create(obj[0], rank, world)

    n = a.n
    triple = resolve_triple(mf, a.triple)
    in_root = a.input_mode == "root"
    plan = mf.Plan(triple, a.levels, n, device=local, shard_rank=rank, shard_count=world,
                   comm=comm, profile=True, level_by_level=a.level_by_level,
                   max_workspace=int(a.max_workspace_gb * 1e9), fuse_postadd=a.fuse,
                   recurse_levels=a.recurse_levels, leaf=a.leaf, comm_regions=a.comm_regions,
                   input_mode=mf.IN_ROOT if in_root else mf.IN_REPLICATED)
    info = plan.info()
    stream = torch.cuda.current_stream()
    # MF_IN_ROOT (sharded default): only rank 0 holds A and B; the step itself
    # broadcasts them (the input exchange is inside the timed step)
    feeds = rank == 0 or not in_root or comm is None
    A, B = mf_inputs.device_pair("uniform", n, 0, device=f"cuda:{local}") if feeds else (None, None)
    C = torch.empty((n, n), dtype=torch.float64, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up, then K timed steps ----
    for _ in range(a.warmup):
        plan.dgemm(A, B, C)
    barrier()
    plan.profile_read(reset=True)
    clocks = Clocks(local)
    clocks.start()
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    evs[0].record(stream)
    for i in range(a.steps):
        plan.dgemm(A, B, C)
        evs[i + 1].record(stream)
    barrier()
    clk = clocks.stop()
    ms = evs[0].elapsed_time(evs[-1]) / a.steps
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
    ms_median = statistics.median(step_ms)
    phases = plan.profile_read(reset=True)
    if distributed:
        t = torch.tensor([ms, ms_median], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_median = float(t[0].item()), float(t[1].item())
    value = 2.0 * n ** 3 / (ms * 1e-3) / 1e12

    # ---- roofline of the dominant kernel (K5 leaf), live over the timed region ----
    shard = plan.products()["shard"]
    m = info["leaf_n"]
    r0s, r1s = plan.shard_rows()  # this rank's row slab of the split leftover products
    my_prods = sum(1 for s in shard if s == rank) + sum(1 for s in shard if s == -1) * (r1s - r0s) / m
    leaf_ms = phases["leaf"] / max(1, phases["calls"])
    leaf_flops = my_prods * 2.0 * m ** 3
    if a.level_by_level:  # the leaf phase holds the whole sub-recursion of each product
        R, p = _rank(a), triple.p
        leaf_flops = R ** a.levels * 2.0 * (n // p ** a.levels) ** 3
    peak, peak_src = fp64_peak()
    achieved = leaf_flops / (leaf_ms * 1e-3) / 1e12
    # the leaf's algorithmic DRAM bytes: every distinct operand block (materialised
    # slot or aliased input block) read once, every product written once
    pr = plan.products()
    mine = [q for q, sh in enumerate(shard) if sh == rank or sh == -1]
    alg_bytes = None
    if not a.level_by_level:
        blk = 8.0 * m * m
        ops_a = {(int(pr["a_src"][q]), int(pr["a_idx"][q])) for q in mine}
        ops_b = {(int(pr["b_src"][q]), int(pr["b_idx"][q])) for q in mine}
        alg_bytes = (len(ops_a) + len(ops_b) + len(mine)) * blk
    kernel = {"dmma": "leaf_dmma_kernel (K5)", "cublas": "cublasDgemmBatched leaf (ablation)",
              "simple": "leaf_simple_kernel (ablation)"}[a.leaf]
    # ncu's leaf DRAM bytes (profiles/ncu_leaf.json) were captured on the default
    # workload: reported only for it
    default_wl = (a.n == 16384 and a.levels == 2 and a.triple == "strassen-winograd"
                  and not a.fuse and not a.level_by_level and a.leaf == "dmma" and world == 1)
    traffic = leaf_traffic() if default_wl else None
    roofline = {"bound": "tensor", "kernel": kernel, "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_src, "flops_per_launch": leaf_flops, "ms_per_launch": leaf_ms,
                "phase_ms_per_step": {k: phases[k] / max(1, phases["calls"]) for k in plan.PHASES},
                "leaf_share_of_step": leaf_ms / ms,
                "algorithmic_bytes": alg_bytes,
                "traffic_over_algorithmic": traffic / alg_bytes if traffic and alg_bytes else None,
                "traffic_note": ("ncu DRAM bytes of the leaf (profiles/ncu_leaf.json) over its "
                                 "algorithmic bytes: B panels are re-read once per 8-tile-row "
                                 "group because a 134 MB operand block does not stay in the "
                                 "126 MB L2; the kernel is DMMA-bound at ~3% of HBM bandwidth "
                                 "(DESIGN.md §5)")}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "ms_per_step_median": ms_median,
           "value_median": 2.0 * n ** 3 / (ms_median * 1e-3) / 1e12,
           "config": config(a, world), "clocks": clk,
           "gpu_launches": launches_per_step(a) * a.steps,
           "roofline": roofline,
           # the whole step against the FP64 tensor roofline of all N GPUs:
           # effective rate, and the algorithmic rate (the multiplications the method
           # performs, R^L 2 m^3 per product) -- the "without credit" fraction
           "step_roofline": step_roofline(a, n, ms, world, peak)}

    # ---- accuracy (north_star: the scaled error against the definition
    # C_ij = sum_k A_ik B_kj, in extended precision on sampled entries; and
    # against cuBLAS DGEMM over the whole matrix), and the classical baselines
    # timed interleaved with the fast step ----
    if rank == 0:
        import numpy as np
        Cref = torch.empty_like(C)
        torch.matmul(A, B, out=Cref)
        torch.cuda.synchronize()
        den = n * float(A.abs().max()) * float(B.abs().max())
        err = 0.0
        for r0 in range(0, n, 2048):  # row slabs: no n x n temporary
            err = max(err, float((C[r0:r0 + 2048] - Cref[r0:r0 + 2048]).abs().max()))
        rng = np.random.Generator(np.random.PCG64(2024))
        ns = min(n, 96)
        rows = np.sort(rng.choice(n, ns, replace=False))
        cols = np.sort(rng.choice(n, ns, replace=False))
        ri = torch.from_numpy(rows).to(dev)
        ci = torch.from_numpy(cols).to(dev)
        ref = (A[ri].cpu().numpy().astype(np.longdouble) @ B[:, ci].cpu().numpy().astype(np.longdouble))
        got = C[ri][:, ci].cpu().numpy().astype(np.longdouble)
        err_ext = float(np.abs(got - ref).max()) / den
        out["max_scaled_error"] = err_ext
        out["max_scaled_error_vs_cublas"] = err / den
        out["error_reference"] = (f"max_scaled_error: |C - C_def| / (n max|A| max|B|) on {ns}x{ns} "
                                  "sampled entries, C_def = sum_k A_ik B_kj in x87 extended precision "
                                  "(the definition); max_scaled_error_vs_cublas: over the whole "
                                  "matrix against cuBLAS DGEMM (includes cuBLAS's own ~2e-16)")
        out["error_bound"] = ceiling(a.levels)
        out["error_model_guard"] = model_guard(a.levels)
        if not a.no_classical and world == 1:
            # K rounds of (fast step, cuBLAS DGEMM, our levels=0 DGEMM), each
            # timed by its own events on the stream, clocks sampled throughout
            with mf.Plan(None, 0, n, device=local) as p0:
                legs = {"fast": lambda: plan.dgemm(A, B, C),
                        "cublas": lambda: torch.matmul(A, B, out=Cref),
                        "levels0": lambda: p0.dgemm(A, B, Cref)}
                for fn in legs.values():
                    fn()
                torch.cuda.synchronize()
                clk2 = Clocks(local)
                clk2.start()
                ev = {k: [] for k in legs}
                for _ in range(a.steps):
                    for k, fn in legs.items():
                        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e_a.record(stream)
                        fn()
                        e_b.record(stream)
                        ev[k].append((e_a, e_b))
                torch.cuda.synchronize()
                clk_il = clk2.stop()
                med = {k: statistics.median(x.elapsed_time(y) for x, y in v) for k, v in ev.items()}
            fl = 2.0 * n ** 3 / 1e12
            t_cublas, t_leaf0 = med["cublas"], med["levels0"]
            out["classical"] = {"cublas_dgemm_tflops": fl / (t_cublas * 1e-3), "cublas_ms": t_cublas,
                                "mf_levels0_tflops": fl / (t_leaf0 * 1e-3), "mf_levels0_ms": t_leaf0,
                                "fast_ms_interleaved": med["fast"],
                                "what": f"medians over {a.steps} interleaved rounds of (fast step, "
                                        "cuBLAS DGEMM, our levels=0 DGEMM), each timed by CUDA events",
                                "clocks": clk_il}
            out["speedup_vs_cublas"] = t_cublas / med["fast"]
            def timeit(fn, st=stream):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(st)
                for _ in range(a.steps):
                    fn()
                s1.record(st)
                torch.cuda.synchronize()
                return s0.elapsed_time(s1) / a.steps
            if n <= 4096:  # launch-bound sizes: the same step replayed as a CUDA graph
                gs = torch.cuda.Stream()
                with mf.Plan(triple, a.levels, n, device=local, graph=True,
                             level_by_level=a.level_by_level, recurse_levels=a.recurse_levels,
                             fuse_postadd=a.fuse, leaf=a.leaf) as pg, torch.cuda.stream(gs):
                    t_graph = timeit(lambda: pg.dgemm(A, B, C, stream=gs), gs)
                out["graph"] = {"ms_per_step": t_graph, "value": fl / (t_graph * 1e-3), "unit": UNIT,
                                "what": "mf_options.graph: the same launches replayed as one "
                                        "CUDA graph per step (no profiling events)"}
        del Cref

    # ---- end to end through the C ABI with host buffers (every rank: its
    # replicated host inputs in, the NCCL reduce inside, C back; max over ranks) ----
    if not a.no_e2e:
        # N > 1 with host buffers: every rank holds the host inputs and copies only
        # its 1/N row slab over its own PCIe link; NCCL all-gathers the rest (one
        # host link carrying all of A and B would bound the step at N = 8)
        slab_e2e = distributed and world > 1 and n % world == 0
        eplan = plan
        if slab_e2e:
            eplan = mf.Plan(triple, a.levels, n, device=local, shard_rank=rank, shard_count=world,
                            comm=comm, level_by_level=a.level_by_level,
                            max_workspace=int(a.max_workspace_gb * 1e9), fuse_postadd=a.fuse,
                            recurse_levels=a.recurse_levels, leaf=a.leaf, comm_regions=a.comm_regions,
                            input_mode=mf.IN_REPLICATED)
            if not feeds:
                A, B = mf_inputs.device_pair("uniform", n, 0, device=f"cuda:{local}")
        Ch = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        if feeds or slab_e2e:
            Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
            Bh = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
            Ah.copy_(A); Bh.copy_(B)
            args = (Ah.data_ptr(), n, Bh.data_ptr(), n, Ch.data_ptr(), n)
        else:  # MF_IN_ROOT: the other ranks pass no host inputs
            args = (None, n, None, n, Ch.data_ptr(), n)
        del A, B, C
        torch.cuda.empty_cache()

        def e2e_time(call, sync):
            call(*args)  # warm-up
            sync()
            barrier()
            t0 = time.perf_counter()
            for _ in range(a.steps):
                call(*args)
            sync()
            dt = (time.perf_counter() - t0) / a.steps
            if distributed:
                t = torch.tensor([dt], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t.item())
            return dt
        # a stream of K products through mf_dgemm_host_async (call k+1's copies
        # under call k's compute), and single synchronous calls
        dt = e2e_time(eplan.dgemm_host_async_ptr, eplan.host_sync)
        dts = e2e_time(eplan.dgemm_host_ptr, lambda: None)
        if eplan is not plan:
            eplan.close()
        out["e2e"] = {"value": 2.0 * n ** 3 / dt / 1e12, "unit": UNIT, "ms_per_step": dt * 1e3,
                      "h2d_bytes_per_step": 2 * 8 * n * n, "d2h_bytes_per_step": 8 * n * n,
                      "api": "mf_dgemm_host_async x K steps + mf_host_sync (pinned host A, B, C; "
                             "every step's H2D + compute + D2H inside the timed region; consecutive "
                             "steps overlap copies with compute"
                             + (("; product-sharded: each rank copies its 1/N row slab of A and B "
                                 "over its own PCIe link and NCCL all-gathers the rest over NVLink"
                                 if slab_e2e or not in_root else
                                 "; product-sharded: rank 0 copies A and B in and broadcasts them "
                                 "by row slabs over NVLink under the other ranks' K4 and leaf")
                                + ", the NCCL reduce of C runs inside, C returns to rank 0's host "
                                  "buffer)" if distributed else ")"),
                      "sync": {"value": 2.0 * n ** 3 / dts / 1e12, "ms_per_step": dts * 1e3,
                               "api": "mf_dgemm_host: one synchronous call per step"}}
        out["gpu_launches_e2e_per_step"] = launches_per_step(a)

    # ---- variants at the same n, same run: one more recursion level (deeper
    # flattening), and the post-additions folded into the leaf epilogue ----
    if rank == 0 and world == 1 and not a.no_variants and a.triple == "strassen-winograd" \
            and a.levels == 2 and not a.level_by_level and not a.fuse and a.n % 8 == 0:
        torch.cuda.empty_cache()
        Av, Bv = mf_inputs.device_pair("uniform", n, 0, device=f"cuda:{local}")
        Cv = torch.empty((n, n), dtype=torch.float64, device=dev)
        Cr = torch.matmul(Av, Bv)
        den = n * float(Av.abs().max()) * float(Bv.abs().max())
        out["variants"] = []
        # the unfused SW^2 result on these inputs (flat K6; no split-K tail, which
        # sums its pieces' k ranges separately): the ordered fold equals it bitwise
        Cu = torch.empty((n, n), dtype=torch.float64, device=dev)
        os.environ["MF_LEAF_SPLIT"] = "1"
        plan.dgemm(Av, Bv, Cu)
        torch.cuda.synchronize()
        del os.environ["MF_LEAF_SPLIT"]
        ordered = ("post-additions folded into the leaf epilogue in ascending q (ordered fold: "
                   "bitwise the unfused result; no P workspace)")
        for label, levels, kw in (
                (f"n={n} fp64, 3-level strassen-winograd (flattened <8,8,8;343>)", 3, {}),
                (f"n={n} fp64, 3-level strassen-winograd, {ordered}", 3, {"fuse_postadd": 1}),
                (f"n={n} fp64, 3-level strassen-winograd, post-additions fused by bulk f64 "
                 "reductions into C (two CTAs per SM; order not fixed; no P workspace)", 3,
                 {"fuse_postadd": 2}),
                (f"n={n} fp64, 4-level strassen-winograd (one level by level, each of its 7 "
                 "products a flattened <8,8,8;343> child: 2401 leaves)", 4,
                 {"level_by_level": True, "recurse_levels": 1}),
                (f"n={n} fp64, 2-level strassen-winograd, {ordered}", 2, {"fuse_postadd": 1}),
                (f"n={n} fp64, 2-level strassen-winograd, post-additions fused by bulk f64 "
                 "reductions into C (two CTAs per SM; order not fixed; no P workspace)", 2,
                 {"fuse_postadd": 2}),
                (f"n={n} fp64, 2-level strassen-winograd with cuBLAS-batched leaves (ablation: "
                 "same K4/K6, cublasDgemmBatched leaf)", 2, {"leaf": "cublas"})):
            if n % (2 ** levels):
                continue
            with mf.Plan(triple, levels, n, device=local, **kw) as pv:
                for _ in range(a.warmup):
                    pv.dgemm(Av, Bv, Cv)
                torch.cuda.synchronize()
                v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                v0.record(stream)
                for _ in range(a.steps):
                    pv.dgemm(Av, Bv, Cv)
                v1.record(stream)
                torch.cuda.synchronize()
                vms = v0.elapsed_time(v1) / a.steps
                ws = pv.info()["workspace_bytes"]
            errv = float((Cv - Cr).abs().max()) / den
            row = {"workload": label, "value": 2.0 * n ** 3 / (vms * 1e-3) / 1e12, "unit": UNIT,
                   "ms_per_step": vms, "max_scaled_error_vs_cublas": errv,
                   "error_bound": ceiling(levels), "workspace_gb": ws / 1e9,
                   "speedup_vs_cublas": (out.get("classical", {}).get("cublas_ms", 0) / vms) or None}
            if kw.get("fuse_postadd") == 1 and levels == 2:
                row["bitwise_equal_unfused"] = bool(torch.equal(Cv, Cu))
            out["variants"].append(row)
        del Av, Bv, Cv, Cr, Cu

    if rank == 0 and world == 1 and not a.no_cpu:
        out["cpu_baseline"] = cpu_baseline(a)

    plan.close()
    if comm is not None:
        mf.comm_destroy(comm)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        emit(out)


if __name__ == "__main__":
    main()
