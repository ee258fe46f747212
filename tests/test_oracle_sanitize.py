"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY.md
§5: memory and UB checking of the C code that pins the GPU path).

tests/oracle_sanitize.c drives every oracle/ entry point (catalog, Kronecker,
Brent check, classical, recursion interpreter with alpha and strided views,
pre/post-additions, Freivalds, sampled entries) on small integer inputs with
exact expected values; it is compiled together with oracle/oracle.c with
-fsanitize=address,undefined -fno-sanitize-recover=all, so any out-of-bounds
access, leak or undefined operation fails the run.  CPU only."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_oracle_under_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_sanitize")
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-fopenmp", "-ffp-contract=off",
           "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer",
           os.path.join(ROOT, "oracle", "oracle.c"), os.path.join(ROOT, "tests", "oracle_sanitize.c"),
           "-o", exe, "-lm"]
    subprocess.check_call(cmd)
    env = dict(os.environ, OMP_NUM_THREADS="2",
               ASAN_OPTIONS="detect_leaks=1:abort_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "oracle sanitize ok" in r.stdout
