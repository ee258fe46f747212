"""bench.py's reference arm (the CPU oracle) on the CPU: one JSON line with the
contract's keys (metric/value/unit/.../impl/cpu_baseline/e2e)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--n", "512", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, check=True).stdout
    lines = [l for l in out.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["n"] == 512 and d["config"]["levels"] == 2


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--n", "256", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env, check=True)
    assert out.stdout.strip() == ""


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _args(mod, *argv):
    old = sys.argv
    try:
        sys.argv = ["bench.py", *argv]
        return mod.parse()
    finally:
        sys.argv = old


def test_bench_presets_and_launch_counts():
    """Host-side bench logic: presets resolve to BASELINE's configs, the kernel
    launch count claimed per step (gpu_launches) follows the plan shape, and
    the oracle sample sizes stay divisible by p^levels."""
    b = _bench_module()
    a = _args(b)
    assert (a.n, a.triple, a.levels) == (16384, "strassen-winograd", 2)   # the metric's config
    assert b.launches_per_step(a) == 4                                     # K4, K4, K5, K6
    assert b._rank(a) ** a.levels == 49
    a = _args(b, "--config", "c1-sw1-64")
    assert b.launches_per_step(a) == 1                                     # one cluster launch
    a = _args(b, "--config", "c4a-ld1-13824")
    assert (a.n, a.triple, a.levels) == (13824, "laderman", 1) and b._rank(a) == 23
    a = _args(b, "--config", "x-sw4-16384-hybrid")
    assert a.level_by_level and a.recurse_levels == 1
    assert b.launches_per_step(a) == 3 + 7 * 4                             # parent + 7 children
    a = _args(b, "--config", "x-sw5-32768-hybrid")
    assert b.launches_per_step(a) == 3 + 7 * (3 + 7 * 4)
    a = _args(b, "--fuse")
    assert b.launches_per_step(a) == 3                                     # K6 in the epilogue
    a = _args(b, "--config", "x-swld-13824")
    assert b._rank(a) == 161
    for cfg in b.CONFIGS:
        a = _args(b, "--config", cfg)
        p = 1
        for part in a.triple.split("(x)"):
            p *= 3 if part == "laderman" else 2
        assert a.n % p ** a.levels == 0, cfg
        ns = b.cpu_sample_n(a)
        assert ns % p ** a.levels == 0 and 0 < ns <= max(a.n // 4, p ** a.levels), cfg
        assert "n=" in b.workload_name(a)
