"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (north_star):
* integer-valued fp64 inputs: bit-exact (IEEE ==) with the exact product;
* pre-additions (K4) and post-addition (K6): bit-exact with the oracle's
  or_premix / or_postmix on random fp64 (same fixed summation order);
* random fp64 end to end: scaled error max|C-C_ref|/(n max|A| max|B|)
  <= 1e-13 per recursion level (classical: <= 1e-14), C_ref = oracle.
Sizes span several 128x128 tiles and ragged tails; the bench-size configs are
checked with exact Freivalds (integers) and sampled oracle entries (random).
"""
import numpy as np
import pytest

import mf_inputs
import oracle
from bounds import assert_error

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2312_12732_b200 as mf
    from paper_2312_12732_b200 import triples
else:  # collected on CPU boxes only to be deselected by -m "not gpu"
    mf = triples = None

SW = "strassen-winograd"


def dev(X):
    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def host(X):
    torch.cuda.synchronize()
    return X.cpu().numpy()


def exact(A, B):
    """Exact product of integer-valued inputs: numpy int64 matmul for small n,
    the oracle's classical loop beyond (exact while |partial sums| < 2^53)."""
    if A.shape[0] <= 512:
        return (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    assert np.abs(A).max() * np.abs(B).max() * A.shape[0] < 2.0 ** 53
    return oracle.classical(A, B)


def run(name, levels, A, B, alpha=1.0, leaf="dmma"):
    t = triples.get(name) if name else None
    with mf.Plan(t, levels, A.shape[0], leaf=leaf) as p:
        C = p.dgemm(dev(A), dev(B), alpha=alpha)
        return host(C)


def scaled(C, Cref, A, B):
    return float(np.abs(C - Cref).max()) / (A.shape[0] * np.abs(A).max() * np.abs(B).max())


# ------------------------------------------------------------------ leaf (levels = 0)

@pytest.mark.parametrize("n", [64, 128, 200, 256, 384, 1000])
def test_classical_leaf_integer_exact(n):
    A, B = mf_inputs.pair("int1024", n, n)
    assert (run(None, 0, A, B) == exact(A, B)).all()


@pytest.mark.parametrize("n", [130, 512])
def test_classical_leaf_random(n):
    A, B = mf_inputs.pair("uniform", n, 1)
    C = run(None, 0, A, B)
    err = scaled(C, oracle.classical(A, B), A, B)
    assert err <= 1e-14


def test_classical_leaf_simple_kernel_and_odd_sizes():
    for n in (1, 7, 33, 97):  # odd m: the TMA path cannot describe these views
        A, B = mf_inputs.pair("int8", n, 2)
        assert (run(None, 0, A, B) == exact(A, B)).all()
    A, B = mf_inputs.pair("int1024", 160, 3)
    assert (run(None, 0, A, B, leaf="simple") == exact(A, B)).all()


def test_leaf_alpha_and_strided_views():
    n = 256
    A, B = mf_inputs.pair("int8", n, 4)
    big = torch.zeros((n, n + 16), dtype=torch.float64, device="cuda")
    big[:, 8:8 + n] = dev(A)
    Av = big[:, 8:8 + n]
    Cbig = torch.full((n, n + 32), float("nan"), dtype=torch.float64, device="cuda")
    Cv = Cbig[:, 4:4 + n]
    with mf.Plan(triples.get(SW), 1, n) as p:
        p.dgemm(Av, dev(B), Cv, alpha=-0.5)
    Ch = host(Cbig)
    assert (Ch[:, 4:4 + n] == -0.5 * exact(A, B)).all()
    assert np.isnan(Ch[:, :4]).all() and np.isnan(Ch[:, 4 + n:]).all()


# ------------------------------------------------------------------ K4 / K6 bit-exact

def _flat_oracle_triple(name, levels):
    return oracle.kron_power(oracle.catalog(name), levels)


def _kron_factored(name, levels, path):
    """True when the plan runs the Kronecker-factored K4/K6 (mf_kron.cu), whose
    order is the recursion's (tested against it below), not the flat table's."""
    deep = (levels >= 3 and name in (SW, "paper-strassen", "strassen-1969")) or \
        (levels == 2 and name == "laderman")
    return path == "fixed" and deep


# compile-time specialised K4/K6 vs the plan-time generated kernels (NVRTC,
# the default for triples without compiled-in kernels) vs the table-driven
# kernels: grouped and the per-output term-list kernel (MF_MIX_UNGROUPED)
MIX_PATHS = ["fixed", "jit", "generic", "generic-terms"]


def _mix_path(monkeypatch, path):
    for var, on in (("MF_MIX_GENERIC", path != "fixed"),
                    ("MF_MIX_NOJIT", path.startswith("generic")),
                    ("MF_MIX_UNGROUPED", path == "generic-terms")):
        if on:
            monkeypatch.setenv(var, "1")
        else:
            monkeypatch.delenv(var, raising=False)
    # every plan the test makes proves, when it closes, that the K4/K6 family
    # the parametrization names is the one that ran (mf_plan_kernels)
    monkeypatch.setattr(mf, "Plan", _checked_plan(path))


def _assert_kernel_path(k, path):
    L = k["launches"]
    if path == "jit":
        # NVRTC and the driver API loaded and every table the plan asked a
        # generated kernel for compiled and loaded -- a silent fallback to the
        # table kernels would show as jit_built < jit_tables.  (Tables too large
        # for a generated kernel's registers are not asked for: those, and
        # views whose alignment a generated kernel cannot serve, run the table
        # kernels by design.)
        assert k["jit_built"] == k["jit_tables"], k
        if k["jit_tables"] and sum(L.values()):
            assert L["jit"] > 0 or L["table"] > 0, k
    elif path.startswith("generic"):
        assert k["jit_built"] == 0 and L["jit"] == L["fixed"] == L["kron"] == 0, k
    elif path == "fixed":
        assert k["jit_built"] == k["jit_tables"], k


_BASE_PLAN = mf.Plan if mf is not None else None


def _checked_plan(path):
    class CheckedPlan(_BASE_PLAN):
        def close(self):
            if getattr(self, "_h", None) is not None and self._h.value and not self._opt.host_only:
                _assert_kernel_path(self.kernels(), path)
            super().close()
    return CheckedPlan


@pytest.mark.parametrize("path", MIX_PATHS)
@pytest.mark.parametrize("name,levels,n", [(SW, 1, 64), (SW, 1, 200), ("laderman", 1, 96),
                                           (SW, 2, 256), ("paper-strassen", 1, 128),
                                           ("strassen-1969", 1, 64), ("paper-strassen", 2, 128),
                                           ("strassen-1969", 2, 64), (SW, 3, 128)])
def test_premix_bit_exact(name, levels, n, path, monkeypatch):
    _mix_path(monkeypatch, path)
    if _kron_factored(name, levels, path):
        pytest.skip("Kronecker-factored path: see test_kron_factored_mix_bit_exact_with_recursion")
    A, B = mf_inputs.pair("uniform", n, 5)
    to = _flat_oracle_triple(name, levels)
    with mf.Plan(triples.get(name), levels, n) as p:
        info, pr = p.info(), p.products()
        m = info["leaf_n"]
        for side, X, src, idx in (("A", A, pr["a_src"], pr["a_idx"]), ("B", B, pr["b_src"], pr["b_idx"])):
            nmat = info["n_mat_a"] if side == "A" else info["n_mat_b"]
            out = torch.empty((max(nmat, 1), m, m), dtype=torch.float64, device="cuda")
            p.premix(side, dev(X), out)
            got = host(out)
            ref = oracle.premix(X, to, side)
            qs = [q for q in range(to.R) if src[q] == 1]
            assert len(qs) == nmat
            for q in qs:
                assert (got[idx[q]] == ref[q]).all(), (side, q)


@pytest.mark.parametrize("path", MIX_PATHS)
@pytest.mark.parametrize("name,levels,n", [(SW, 1, 64), ("laderman", 1, 96), (SW, 2, 256),
                                           (SW, 1, 200), ("paper-strassen", 2, 128),
                                           ("strassen-1969", 1, 64), (SW, 3, 128)])
def test_postmix_bit_exact(name, levels, n, path, monkeypatch):
    _mix_path(monkeypatch, path)
    if _kron_factored(name, levels, path):
        pytest.skip("Kronecker-factored path: see test_kron_factored_mix_bit_exact_with_recursion")
    to = _flat_oracle_triple(name, levels)
    m = n // to.p
    rng = np.random.Generator(np.random.PCG64(9))
    Pp = rng.uniform(-1, 1, size=(to.R, m, m))  # P' as the leaf stage would write it
    with mf.Plan(triples.get(name), levels, n) as p:
        sign = p.products()["sign"].astype(np.float64)
        for alpha in (1.0, 0.37):
            C = torch.empty((n, n), dtype=torch.float64, device="cuda")
            p.postmix(dev(Pp), C, alpha=alpha)
            ref = oracle.postmix(Pp * sign[:, None, None], to, n, alpha)
            assert (host(C) == ref).all()


def _recursive_premix(X, t, levels, side):
    """The oracle's recursion (or_fmm) for the operands: level-1
    T_q of X, then level-2 T of each, ... -> R^levels blocks, index outer-major.
    t may be a list of triples, one per level (a mixed chain), outer first."""
    chain = t if isinstance(t, list) else [t] * levels
    blocks = [X]
    for tl in chain:
        blocks = [T for Y in blocks for T in oracle.premix(Y, tl, side)]
    return np.stack(blocks)


def _recursive_postmix(P, t, levels, n, alpha):
    """The oracle's recursion for the post-addition: combine the innermost level
    first ("recursively solve P_i and distribute it"), alpha last."""
    chain = t if isinstance(t, list) else [t] * levels
    cur = list(P)
    size = n
    for tl in chain:
        size //= tl.p
    for lev, tl in enumerate(reversed(chain)):
        size *= tl.p
        a = alpha if lev == len(chain) - 1 else 1.0
        cur = [oracle.postmix(np.stack(cur[g * tl.R:(g + 1) * tl.R]), tl, size, a)
               for g in range(len(cur) // tl.R)]
    return cur[0]


@pytest.mark.parametrize("name,levels,n", [(SW, 3, 128), ("paper-strassen", 3, 64),
                                           ("strassen-1969", 3, 64), ("laderman", 2, 144),
                                           (SW, 3, 200)])
def test_kron_factored_mix_bit_exact_with_recursion(name, levels, n):
    """Kronecker-factored K4/K6 (mf_kron.cu) == the oracle's recursive
    pre-/post-additions bitwise on random fp64 (same per-level order)."""
    t = triples.get(name)
    to = oracle.catalog(name)
    A, B = mf_inputs.pair("uniform", n, 23)
    with mf.Plan(t, levels, n) as p:
        info, pr = p.info(), p.products()
        m = info["leaf_n"]
        for side, X, src, idx in (("A", A, pr["a_src"], pr["a_idx"]), ("B", B, pr["b_src"], pr["b_idx"])):
            nmat = info["n_mat_a"] if side == "A" else info["n_mat_b"]
            out = torch.empty((nmat, m, m), dtype=torch.float64, device="cuda")
            p.premix(side, dev(X), out)
            got = host(out)
            ref = _recursive_premix(X, to, levels, side)
            for q in np.nonzero(src == 1)[0]:
                assert (got[idx[q]] == ref[q]).all(), (side, q)
        rng = np.random.Generator(np.random.PCG64(24))
        Pp = rng.uniform(-1, 1, size=(to.R ** levels, m, m))
        for alpha in (1.0, -1.25):
            C = torch.empty((n, n), dtype=torch.float64, device="cuda")
            p.postmix(dev(Pp), C, alpha=alpha)
            assert (host(C) == _recursive_postmix(Pp, to, levels, n, alpha)).all()


@pytest.mark.parametrize("outer,inner", [(SW, "laderman"), ("laderman", SW)])
@pytest.mark.parametrize("n", [72, 1152])
def test_mixed_chain_6x6(outer, inner, n):
    """NEXT-2: the chains 2-then-3 and 3-then-2 ("the sequence 2 and 3
    specifies an algorithm that is different from the sequence 3 and 2") as one
    flattened <6,6,6;161> level: Kronecker-factored K4/K6 bitwise the oracle's
    mixed recursion, end to end exact on integers and within the bound."""
    to, ti = triples.get(outer), triples.get(inner)
    t = triples.kron(to, ti)
    chain = [oracle.catalog(outer), oracle.catalog(inner)]
    assert t.p == 6 and t.R == 161
    A, B = mf_inputs.pair("uniform", n, 25)
    with mf.Plan(t, 1, n) as p:
        info, pr = p.info(), p.products()
        m = info["leaf_n"]
        for side, X, src, idx in (("A", A, pr["a_src"], pr["a_idx"]), ("B", B, pr["b_src"], pr["b_idx"])):
            out = torch.empty((info["n_mat_a"] if side == "A" else info["n_mat_b"], m, m),
                              dtype=torch.float64, device="cuda")
            p.premix(side, dev(X), out)
            got, ref = host(out), _recursive_premix(X, chain, 2, side)
            for q in np.nonzero(src == 1)[0]:
                assert (got[idx[q]] == ref[q]).all(), (side, q)
        Pp = np.random.Generator(np.random.PCG64(26)).uniform(-1, 1, size=(161, m, m))
        C = torch.empty((n, n), dtype=torch.float64, device="cuda")
        p.postmix(dev(Pp), C, alpha=0.5)
        assert (host(C) == _recursive_postmix(Pp, chain, 2, n, 0.5)).all()
        C = host(p.dgemm(dev(A), dev(B)))
        assert scaled(C, oracle.classical(A, B), A, B) <= 2e-13
        Ai, Bi = mf_inputs.pair("int1024", n, 27)
        assert (host(p.dgemm(dev(Ai), dev(Bi))) == exact(Ai, Bi)).all()


def test_leaf_stage_matches_oracle_products_on_integers():
    n = 256
    A, B = mf_inputs.pair("int1024", n, 6)
    to = _flat_oracle_triple(SW, 2)
    T, S = oracle.premix(A, to, "A"), oracle.premix(B, to, "B")
    with mf.Plan(triples.get(SW), 2, n) as p:
        info, pr = p.info(), p.products()
        m = info["leaf_n"]
        Td = torch.empty((info["n_mat_a"], m, m), dtype=torch.float64, device="cuda")
        Sd = torch.empty((info["n_mat_b"], m, m), dtype=torch.float64, device="cuda")
        p.premix("A", dev(A), Td)
        p.premix("B", dev(B), Sd)
        P = torch.empty((to.R, m, m), dtype=torch.float64, device="cuda")
        p.leaf(dev(A), dev(B), Td, Sd, P)
        got = host(P)
        for q in range(to.R):
            assert (got[q] == pr["sign"][q] * exact(T[q], S[q])).all(), q


# ------------------------------------------------------------------ end to end

CASES = [(SW, 1, 64), (SW, 1, 256), (SW, 1, 400), (SW, 2, 128), (SW, 2, 512), (SW, 3, 512),
         ("paper-strassen", 1, 256), ("paper-strassen", 2, 256), ("strassen-1969", 1, 256),
         ("laderman", 1, 96), ("laderman", 1, 288), ("laderman", 1, 390), ("laderman", 2, 144),
         ("classical-p2", 1, 128)]


@pytest.mark.parametrize("path", MIX_PATHS)
@pytest.mark.parametrize("name,levels,n", CASES)
def test_dgemm_integer_exact(name, levels, n, path, monkeypatch):
    """integer computations are exact -> bit-exact vs the exact product."""
    _mix_path(monkeypatch, path)
    A, B = mf_inputs.pair("int1024", n, 11)
    C = run(name, levels, A, B)
    assert (C == exact(A, B)).all()


@pytest.mark.parametrize("name,levels,n", CASES)
def test_dgemm_random_within_bound(name, levels, n):
    A, B = mf_inputs.pair("uniform", n, 12)
    C = run(name, levels, A, B)
    err = scaled(C, oracle.classical(A, B), A, B)
    assert_error(err, levels)
    # and close to the oracle's own recursion (same algorithm, different leaf order)
    Co = oracle.fmm(A, B, oracle.catalog(name), levels)
    assert_error(scaled(C, Co, A, B), levels)


@pytest.mark.parametrize("name,levels,n", [(SW, 2, 256), (SW, 3, 512), ("laderman", 2, 288),
                                           ("paper-strassen", 2, 512), (SW, 2, 1000)])
def test_level_by_level_recursion(name, levels, n):
    """a5: the paper's recursion executed level by level -- the
    same bilinear map as the flattened default: exact on integers; on random
    inputs within the bound, and close to the oracle's own recursion."""
    t = triples.get(name)
    A, B = mf_inputs.pair("int1024", n, 17)
    with mf.Plan(t, levels, n, level_by_level=True) as p:
        assert p.info()["n_products"] == t.R and p.info()["leaf_n"] == n // t.p
        assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 18)
        C = host(p.dgemm(dev(A), dev(B), alpha=1.5))
    Co = oracle.fmm(A, B, oracle.catalog(name), levels, alpha=1.5)
    assert_error(scaled(C, Co, A, B), levels)
    assert_error(scaled(C, 1.5 * oracle.classical(A, B), A, B), levels)


@pytest.mark.parametrize("name,levels,n,r", [(SW, 3, 512, 1), (SW, 4, 1024, 1), (SW, 4, 2048, 2),
                                             ("laderman", 3, 27 * 16, 1)])
def test_recurse_levels_hybrid(name, levels, n, r):
    """level_by_level with recurse_levels = r: the top r levels one at a time,
    each product a flattened (levels - r)-level child plan.  Same bilinear map:
    exact on integers; random within the bound and close to the oracle's
    recursion."""
    t = triples.get(name)
    A, B = mf_inputs.pair("int1024", n, 46)
    with mf.Plan(t, levels, n, level_by_level=True, recurse_levels=r) as p:
        assert p.info()["n_products"] == t.R and p.info()["leaf_n"] == n // t.p
        assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 47)
        C = host(p.dgemm(dev(A), dev(B), alpha=-0.5))
    Co = oracle.fmm(A, B, oracle.catalog(name), levels, alpha=-0.5)
    assert_error(scaled(C, Co, A, B), levels)
    assert_error(scaled(C, -0.5 * oracle.classical(A, B), A, B), levels)


def test_sw4_hybrid_bench_size_sampled():
    """The bench's 4-level variant at full size (n = 16384: one SW level by
    level over 7 flattened SW^3 children, 2401 leaves of 1024^2): exact
    Freivalds on integers, sampled oracle entries on random inputs."""
    n = 16384
    with mf.Plan(triples.get(SW), 4, n, level_by_level=True, recurse_levels=1) as p:
        Ad, Bd = mf_inputs.device_pair("int1024", n, 48)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
        del Ad, Bd
        assert oracle.freivalds_int(A, B, C, trials=2) == 0
        _sampled_check(C, A, B, count=128)
        Ad, Bd = mf_inputs.device_pair("uniform", n, 49)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
    _sampled_check(C, A, B, count=128, tol=4e-13)


def test_sw5_hybrid_full_size():
    """The five-level preset at full size (n = 32768: two SW levels one at a
    time over 49 flattened SW^3 children at n = 8192, 16807 leaves of 1024^2):
    exact Freivalds on integers (entries in [-8, 8]: every partial sum of five
    levels stays below 2^53, DESIGN R15), sampled oracle entries on random
    inputs within 1e-13 per level."""
    n = 32768
    with mf.Plan(triples.get(SW), 5, n, level_by_level=True, recurse_levels=2) as p:
        Ad, Bd = mf_inputs.device_pair("int8", n, 50)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
        del Ad, Bd
        assert oracle.freivalds_int(A, B, C, trials=2) == 0
        _sampled_check(C, A, B, count=64)
        del A, B, C
        Ad, Bd = mf_inputs.device_pair("uniform", n, 51)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
    _sampled_check(C, A, B, count=64, tol=5e-13)


def test_config1_n64_sw1_all_distributions():
    """BASELINE config 1: n=64, one-level Strassen-Winograd."""
    for kind in ("int8", "int1024"):
        A, B = mf_inputs.pair(kind, 64, 0)
        assert (run(SW, 1, A, B) == exact(A, B)).all()
    A, B = mf_inputs.pair("uniform", 64, 0)
    C = run(SW, 1, A, B)
    Co = oracle.fmm(A, B, oracle.catalog(SW), 1)
    assert_error(scaled(C, oracle.classical(A, B), A, B), 1)
    assert scaled(C, Co, A, B) <= 1e-15


@pytest.mark.parametrize("name,levels", [(SW, 1), ("laderman", 1), (SW, 2)])
def test_block_impulse_routing(name, levels):
    """A = 1 on block x, B = 1 on block y -> C = m on block (i,j) iff x=(i,k),
    y=(k,j) (the GPU-level Brent check)."""
    t = triples.get(name)
    P = t.p ** levels
    m = 16
    n = P * m
    with mf.Plan(t, levels, n) as p:
        for x in range(P * P):
            A = mf_inputs.block_impulse(n, P, x)
            Ad = dev(A)
            for y in range(P * P):
                B = mf_inputs.block_impulse(n, P, y)
                C = host(p.dgemm(Ad, dev(B)))
                i, k = divmod(x, P); k2, j = divmod(y, P)
                E = np.zeros((n, n))
                if k == k2:
                    E[i * m:(i + 1) * m, j * m:(j + 1) * m] = m
                assert (C == E).all(), (x, y)


def test_sharded_partials_sum_to_product():
    """Product sharding emulated on one GPU: every shard's
    partial C is its products' W-combination; the shards sum to A*B."""
    n = 256
    A, B = mf_inputs.pair("int1024", n, 13)
    total = np.zeros((n, n))
    owners = []
    for r in range(3):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=3) as p:
            total += run_plan(p, A, B)
            owners.append(p.products()["shard"])
    assert (total == exact(A, B)).all()
    assert (owners[0] == owners[1]).all() and sorted(set(owners[0].tolist())) == [0, 1, 2]


@pytest.mark.parametrize("N", [2, 3, 8])
def test_split_sharding_partials_sum_to_product(N):
    """Exact balance emulated on one GPU: floor(49/N) whole products
    per rank + a row slab of each leftover product; the N partial C sum to the
    exact product on integers, and to the 1-GPU result within the bound."""
    n = 4096
    A, B = mf_inputs.pair("int1024", n, 19)
    Ad, Bd = dev(A), dev(B)
    total = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for r in range(N):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=N) as p:
            assert (p.products()["shard"] == -1).sum() == 49 % N
            total += p.dgemm(Ad, Bd)
    assert (host(total) == exact(A, B)).all()
    A, B = mf_inputs.pair("uniform", n, 20)
    Ad, Bd = dev(A), dev(B)
    with mf.Plan(triples.get(SW), 2, n) as p:
        ref = host(p.dgemm(Ad, Bd))
    total.zero_()
    for r in range(N):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=N) as p:
            total += p.dgemm(Ad, Bd)
    assert scaled(host(total), ref, A, B) <= 2e-13


@pytest.mark.parametrize("N", [2, 3, 8])
def test_sharded_workspace_shrinks_with_ranks(N):
    """A shard allocates only its own products' T / S slots and P blocks
    (shard-local numbering): per-rank workspace ~ 1/N of the 1-GPU plan's
    (SW^2 n = 4096: 129 blocks of 8 MB on one GPU; rank r of 8 holds at most
    7 products, <= 21 blocks)."""
    n = 4096
    with mf.Plan(triples.get(SW), 2, n) as p:
        full = p.info()["workspace_bytes"]
    blk = 8 * (n // 4) ** 2
    assert full == 129 * blk
    for r in range(N):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=N) as p:
            ws = p.info()["workspace_bytes"]
            mine = int((p.products()["shard"] == r).sum() + (p.products()["shard"] == -1).sum())
            assert ws <= 3 * mine * blk
            assert ws <= (1.0 / N + 0.2) * full


def test_nccl_single_rank_plan_matches_local():
    """The NCCL exchange step of the sharded path (mf_nccl_unique_id /
    mf_nccl_comm_create / reduce of C in mf_dgemm) on a 1-rank communicator:
    bitwise the local result; OUT_ALL (all-reduce) too; and IN_ROOT inputs are
    broadcast into plan replicas.  Through mf_dgemm_host too: with replicated
    host inputs each rank copies its row slab and NCCL all-gathers the rest
    (strided host views included); IN_ROOT copies everything."""
    n = 512
    A, B = mf_inputs.pair("uniform", n, 30)
    with mf.Plan(triples.get(SW), 2, n) as p:
        ref = host(p.dgemm(dev(A), dev(B)))
    comm = mf.nccl_comm_create(mf.nccl_unique_id(), 0, 1)
    Aw = np.zeros((n, n + 8)); Aw[:, :n] = A
    Bw = np.zeros((n, n + 16)); Bw[:, :n] = B
    try:
        for out_mode, in_mode in ((mf.OUT_ROOT, mf.IN_REPLICATED), (mf.OUT_ALL, mf.IN_ROOT)):
            with mf.Plan(triples.get(SW), 2, n, shard_rank=0, shard_count=1, nccl_comm=comm,
                         output_mode=out_mode, input_mode=in_mode) as p:
                C = host(p.dgemm(dev(A), dev(B)))
                assert (p.dgemm_host(A, B) == ref).all()
                assert (p.dgemm_host(Aw[:, :n], Bw[:, :n]) == ref).all()
                # a stream of host-buffer calls (all-gather on the compute stream)
                Ah = torch.from_numpy(A).pin_memory(); Bh = torch.from_numpy(B).pin_memory()
                outs = [torch.full((n, n), float("nan"), dtype=torch.float64).pin_memory()
                        for _ in range(3)]
                for Ch in outs:
                    p.dgemm_host_async_ptr(Ah.data_ptr(), n, Bh.data_ptr(), n, Ch.data_ptr(), n)
                p.host_sync()
                for Ch in outs:
                    assert (Ch.numpy() == ref).all()
            assert (C == ref).all()
    finally:
        mf.nccl_comm_destroy(comm)


def run_plan(p, A, B):
    return host(p.dgemm(dev(A), dev(B)))


@pytest.mark.parametrize("path", ["jit", "generic"])
@pytest.mark.parametrize("name,levels,n,g", [(SW, 2, 512, 5), ("laderman", 1, 288, 2), (SW, 3, 256, 3),
                                             (SW, 1, 400, 1)])
def test_bounded_workspace_batches(name, levels, n, g, path, monkeypatch):
    """NEXT-3 bounded workspace: products run in batches
    of g whose T/S/P fit max_workspace; exact on integers, within the bound on
    random inputs, workspace within the cap; too small a cap is reported.
    Batches run generated K4/K6 (jit) or the table-driven kernels (generic)."""
    _mix_path(monkeypatch, path)
    t = triples.get(name)
    m = n // t.p ** levels
    cap = 3 * g * m * m * 8
    A, B = mf_inputs.pair("int1024", n, 28)
    with mf.Plan(t, levels, n, max_workspace=cap) as p:
        assert p.info()["workspace_bytes"] <= cap
        assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 29)
        C = host(p.dgemm(dev(A), dev(B), alpha=0.5))
    assert_error(scaled(C, 0.5 * oracle.classical(A, B), A, B), levels)
    with pytest.raises(mf.MfError) as e:
        mf.Plan(t, levels, n, max_workspace=3 * m * m * 8 - 1)
    assert e.value.status == mf.MF_ERR_OUT_OF_MEMORY
    with mf.Plan(t, levels, n, max_workspace=1 << 40) as p:  # no batching needed
        C2 = host(p.dgemm(dev(A), dev(B), alpha=0.5))
    with mf.Plan(t, levels, n) as p:
        assert (C2 == host(p.dgemm(dev(A), dev(B), alpha=0.5))).all()


@pytest.mark.parametrize("name,levels,n,cap_blocks", [(SW, 2, 512, 15), ("laderman", 2, 243, 6),
                                                      (SW, 1, 200, None), ("laderman", 1, 120, None)])
def test_jit_mix_bitwise_table_kernels(name, levels, n, cap_blocks, monkeypatch):
    """The plan-time generated K4/K6 (mf_jit.cpp) and the table-driven kernels
    sum every output in the same (the oracle's) order: bitwise equal results on
    random inputs, whole plans and bounded-workspace batches (K6 accumulating
    into C), ragged leaves (m = 100, 60: 64-bit vectors) included."""
    t = triples.get(name)
    m = n // t.p ** levels
    kw = {"max_workspace": 3 * cap_blocks * m * m * 8} if cap_blocks else {}
    A, B = mf_inputs.pair("uniform", n, 31)
    out = {}
    for path in ("jit", "generic"):
        _mix_path(monkeypatch, path)
        with mf.Plan(t, levels, n, **kw) as p:
            out[path] = host(p.dgemm(dev(A), dev(B), alpha=1.5))
    assert (out["jit"] == out["generic"]).all()
    assert_error(scaled(out["jit"], 1.5 * oracle.classical(A, B), A, B), levels)


def test_host_buffer_entry_point():
    n = 256
    A, B = mf_inputs.pair("int1024", n, 14)
    with mf.Plan(triples.get(SW), 2, n) as p:
        C = p.dgemm_host(A, B)
        assert (C == exact(A, B)).all()
        C2 = p.dgemm_host(A, B, alpha=2.0)
        assert (C2 == 2 * exact(A, B)).all()


@pytest.mark.parametrize("path", MIX_PATHS)
@pytest.mark.parametrize("name,levels,n", [(SW, 2, 2048), (SW, 1, 2048), (None, 0, 1024),
                                           ("laderman", 1, 3072), (SW, 1, 1000)])
def test_host_pipeline_matches_device_path(name, levels, n, path, monkeypatch):
    """mf_dgemm_host's slab pipeline (H2D / K4-K5-K6 per row slab / D2H on
    three streams) computes exactly what mf_dgemm computes: same kernels, same
    per-element order -> bitwise equal on random inputs, exact on integers;
    host leading dimensions > n are honoured.  (mf_dgemm's own leaf may cut a
    few-wave launch's tail into split-K pieces, which the pipeline's region
    launches never do: bitwise with MF_LEAF_SPLIT=1, to rounding otherwise.)"""
    _mix_path(monkeypatch, path)
    t = triples.get(name) if name else None
    A, B = mf_inputs.pair("uniform", n, 15)
    with mf.Plan(t, levels, n) as p:
        Cs = host(p.dgemm(dev(A), dev(B), alpha=0.75))
        monkeypatch.setenv("MF_LEAF_SPLIT", "1")
        Cd = host(p.dgemm(dev(A), dev(B), alpha=0.75))
        monkeypatch.delenv("MF_LEAF_SPLIT")
        Ah = np.zeros((n, n + 8)); Ah[:, :n] = A
        Ch = np.full((n, n + 4), np.nan)
        p.dgemm_host_ptr(Ah.ctypes.data, n + 8, B.ctypes.data, n, Ch.ctypes.data, n + 4, alpha=0.75)
        assert (Ch[:, :n] == Cd).all() and np.isnan(Ch[:, n:]).all()
        assert scaled(Ch[:, :n], Cs, A, B) <= 1e-14 * max(1, levels)
        Ai, Bi = mf_inputs.pair("int1024", n, 16)
        assert (p.dgemm_host(Ai, Bi) == exact(Ai, Bi)).all()


def test_invalid_calls_report_errors():
    n = 64
    with mf.Plan(triples.get(SW), 1, n) as p:
        A = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        with pytest.raises(mf.MfError) as e:
            p.dgemm(A, A, A)  # C overlaps A
        assert e.value.status == mf.MF_ERR_INVALID_ARG


# ------------------------------------------------------------------ bench-size configs

def _sampled_check(C, A, B, count=256, seed=0, tol=None):
    rng = np.random.Generator(np.random.PCG64(seed))
    n = A.shape[0]
    rows = rng.integers(0, n, count); cols = rng.integers(0, n, count)
    ref = oracle.sample_entries(A, B, rows, cols)
    got = C[rows, cols]
    if tol is None:
        assert (got == ref).all()
    else:
        den = n * np.abs(A).max() * np.abs(B).max()
        assert float(np.abs(got - ref).max()) / den <= tol


@pytest.mark.parametrize("name,levels,n", [(SW, 1, 4096), (SW, 2, 16384), ("laderman", 1, 13824),
                                           (SW, 2, 13824), (SW, 2, 32768), (SW, 3, 16384),
                                           ("laderman", 2, 13824), (SW + "(x)laderman", 1, 13824),
                                           ("laderman(x)" + SW, 1, 13824)])
def test_bench_configs_full_size(name, levels, n):
    """BASELINE configs 2-5 at full size (config 5: its 1-GPU problem, n=32768,
    69 GB of workspace) and the reported variants (SW^3, Laderman^2, both mixed
    chains <6,6,6;161>), in the launch configuration bench.py times (k = 48 leaf
    stages at m = 3456, 4608, 8192; 2304 for the chains): exact Freivalds on
    integers + sampled oracle entries on random."""
    if "(x)" in name:
        o, i = name.split("(x)")
        t = triples.kron(triples.get(o), triples.get(i))
    else:
        t = triples.get(name)
    with mf.Plan(t, levels, n) as p:
        Ad, Bd = mf_inputs.device_pair("int1024", n, 21)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
        del Ad, Bd
        assert oracle.freivalds_int(A, B, C, trials=2) == 0
        _sampled_check(C, A, B, count=128)
        Ad, Bd = mf_inputs.device_pair("uniform", n, 22)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
        _sampled_check(C, A, B, count=128, tol=1e-13 * levels)


# ------------------------------------------------ fused post-addition (epilogue fold)

FUSED_CASES = [(SW, 1, 256), (SW, 1, 400), (SW, 2, 512), (SW, 2, 800), (SW, 3, 1024),
               ("paper-strassen", 2, 256), ("strassen-1969", 1, 256), ("laderman", 1, 390),
               ("laderman", 2, 288), ("classical-p2", 1, 128)]


def _ordered_and_flat(monkeypatch, t, levels, n, A, B, alpha, **kw):
    """(ordered fold, unfused) results with the same flat-order kernels: both
    plans use the flat ascending-index K4 (generated / table kernels; the
    Kronecker-factored K4/K6 of deep catalog powers sum in the recursion's
    order instead), and the unfused leaf has no split-K tail (a split tile sums
    its k range in pieces).  The ordered fold must then equal K5 + K6 bitwise."""
    with monkeypatch.context() as mp:
        mp.setenv("MF_MIX_GENERIC", "1")
        mp.setenv("MF_LEAF_SPLIT", "1")
        with mf.Plan(t, levels, n, fuse_postadd=1, **kw) as p:
            Cf = host(p.dgemm(dev(A), dev(B), alpha=alpha))
        with mf.Plan(t, levels, n, **kw) as p:
            Cu = host(p.dgemm(dev(A), dev(B), alpha=alpha))
    return Cf, Cu


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name,levels,n", FUSED_CASES)
def test_fused_postadd_integer_exact_and_random(name, levels, n, mode, monkeypatch):
    """North_star (3) / SURVEY §8a a4 "optionally folded into the leaf GEMM
    epilogue": every product tile goes straight into the C blocks it feeds.
    Mode 1, the ordered fold (SURVEY §8f NEXT-1 "deterministic product-serial
    ordering"): tiles of one position update C in ascending q, store / add /
    alpha last like K6 -- bitwise the unfused path on random inputs, and
    bitwise from run to run.  Mode 2 (bulk f64 reductions, order not fixed):
    integers bit-exact (all partial sums exact); random within the bound.
    Covers -1 coefficients, ragged tails (n=400: m=200, n=800: m=200, n=390:
    m=130), alpha != 1, NaN-filled C (write-only), no P workspace."""
    t = triples.get(name)
    A, B = mf_inputs.pair("int1024", n, 40)
    with mf.Plan(t, levels, n, fuse_postadd=mode) as p:
        C = torch.full((n, n), float("nan"), dtype=torch.float64, device="cuda")
        assert (host(p.dgemm(dev(A), dev(B), C=C)) == exact(A, B)).all()
        assert (host(p.dgemm(dev(A), dev(B), alpha=-2.0)) == -2.0 * exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 41)
        Cf = host(p.dgemm(dev(A), dev(B), alpha=0.5))
        Cf2 = host(p.dgemm(dev(A), dev(B), alpha=0.5))
    Cref = 0.5 * oracle.classical(A, B)
    assert_error(scaled(Cf, Cref, A, B), levels)
    if mode == 1:
        assert (Cf2 == Cf).all()  # deterministic
        Co, Cu = _ordered_and_flat(monkeypatch, t, levels, n, A, B, 0.5)
        assert (Co == Cu).all()
    else:
        with mf.Plan(t, levels, n) as p:
            assert_error(scaled(Cf, host(p.dgemm(dev(A), dev(B), alpha=0.5)), A, B), levels)


@pytest.mark.parametrize("name,levels,n", [(SW, 3, 1024), ("laderman", 1, 768), (SW, 1, 4096),
                                           ("paper-strassen", 2, 1000)])
def test_fused_ordered_bitwise_unfused(name, levels, n, monkeypatch):
    """The ordered fold at more shapes: SW^3 (343 products, ~5 C blocks per
    product), Laderman (p = 3), one level at a bench size (7 products of
    2048^2), a ragged leaf (m = 250): C bitwise the unfused K5 + flat K6 result
    (itself bitwise or_postmix, test_postmix_bit_exact)."""
    t = triples.get(name)
    A, B = mf_inputs.pair("uniform", n, 46)
    Cf, Cu = _ordered_and_flat(monkeypatch, t, levels, n, A, B, -1.25)
    assert (Cf == Cu).all()


def test_fused_postadd_workspace_views_and_fallbacks(monkeypatch):
    """Fused plans allocate no P workspace; strided C (ldc > n, even) keeps the
    TMA/bulk path, odd ldc falls back to the simple leaf with f64 atomics; the
    simple leaf kind and the host-buffer entry point work fused too."""
    n, t = 512, triples.get(SW)
    m = n // 4
    with mf.Plan(t, 2, n) as p:
        ws_unfused = p.info()["workspace_bytes"]
    A, B = mf_inputs.pair("int1024", n, 42)
    ref = exact(A, B)
    for mode in (1, 2):
        with mf.Plan(t, 2, n, fuse_postadd=mode) as p:
            assert ws_unfused - p.info()["workspace_bytes"] == 49 * m * m * 8
            for ldc in (n + 2, n + 1):
                Cbig = torch.full((n, ldc), 7.0, dtype=torch.float64, device="cuda")
                p.dgemm(dev(A), dev(B), C=Cbig[:, :n])
                out = host(Cbig)
                assert (out[:, :n] == ref).all() and (out[:, n:] == 7.0).all()
            assert (p.dgemm_host(A, B) == ref).all()
        with mf.Plan(t, 2, n, fuse_postadd=mode, leaf="simple") as p:
            assert (host(p.dgemm(dev(A), dev(B))) == ref).all()
    # the ordered fold on the simple leaf (one launch per product, in order) and
    # on odd ldc (scalar stores) is bitwise the unfused result on random inputs
    A, B = mf_inputs.pair("uniform", n, 47)
    Cs, Cu = _ordered_and_flat(monkeypatch, t, 2, n, A, B, 3.0, leaf="simple")
    assert (Cs == Cu).all()
    _, Cu = _ordered_and_flat(monkeypatch, t, 2, n, A, B, 3.0)
    with mf.Plan(t, 2, n, fuse_postadd=1) as p:
        Cbig = torch.full((n, n + 1), 7.0, dtype=torch.float64, device="cuda")
        p.dgemm(dev(A), dev(B), C=Cbig[:, :n], alpha=3.0)
        assert (host(Cbig)[:, :n] == Cu).all()


@pytest.mark.parametrize("N", [1, 3])
def test_fused_postadd_sharded_partials(N):
    """Fused epilogue on product shards, whole and split (row slabs): the
    partial C of the N shards sum to the exact product."""
    n = 2048
    A, B = mf_inputs.pair("int1024", n, 43)
    Ad, Bd = dev(A), dev(B)
    total = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for r in range(N):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=N, fuse_postadd=2) as p:
            total += p.dgemm(Ad, Bd)
    assert (host(total) == exact(A, B)).all()


def test_fused_postadd_bench_size_sampled():
    """n = 16384, SW^2 fused (the bench's --fuse variant, ordered fold):
    Freivalds on integers is exact; random inputs checked on sampled oracle
    entries."""
    n = 16384
    with mf.Plan(triples.get(SW), 2, n, fuse_postadd=1) as p:
        Ad, Bd = mf_inputs.device_pair("int1024", n, 44)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
        del Ad, Bd
        assert oracle.freivalds_int(A, B, C, trials=2) == 0
        _sampled_check(C, A, B, count=128)
        Ad, Bd = mf_inputs.device_pair("uniform", n, 45)
        C = host(p.dgemm(Ad, Bd))
        A, B = host(Ad), host(Bd)
    _sampled_check(C, A, B, count=128, tol=2e-13)


# ------------------------------------------------ cuBLAS leaf ablation, row-slab output

@pytest.mark.parametrize("name,levels,n", [(SW, 1, 256), (SW, 2, 512), ("laderman", 1, 390),
                                           (None, 0, 300), (SW, 3, 1024)])
def test_cublas_leaf_ablation(name, levels, n):
    """MF_LEAF_CUBLAS: the same K4/K6 around cublasDgemmBatched leaf products
    (grouped by operand strides).  Integers exact; random within the bound."""
    t = triples.get(name) if name else None
    A, B = mf_inputs.pair("int1024", n, 50)
    with mf.Plan(t, levels, n, leaf="cublas") as p:
        assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 51)
        C = host(p.dgemm(dev(A), dev(B), alpha=0.25))
        assert (p.dgemm_host(A, B, alpha=0.25) == C).all()
    assert_error(scaled(C, 0.25 * oracle.classical(A, B), A, B), levels)


def test_cublas_leaf_split_sharding_and_batches():
    """The cuBLAS leaf on split-product row slabs (shards) and bounded-workspace
    batches (batch-local slots): partials sum / results equal the exact product."""
    n = 1024
    A, B = mf_inputs.pair("int1024", n, 52)
    total = np.zeros((n, n))
    for r in range(3):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=3, leaf="cublas") as p:
            total += run_plan(p, A, B)
    assert (total == exact(A, B)).all()
    m = n // 4
    with mf.Plan(triples.get(SW), 2, n, leaf="cublas", max_workspace=3 * 5 * m * m * 8) as p:
        assert (run_plan(p, A, B) == exact(A, B)).all()


def test_nccl_rowslab_output_single_rank():
    """MF_OUT_ROWSLAB: C reduce-scattered by block rows (ncclReduceScatter); on a
    1-rank communicator the slab is the whole product, bitwise the local result,
    through both entry points."""
    n = 512
    A, B = mf_inputs.pair("uniform", n, 53)
    with mf.Plan(triples.get(SW), 2, n) as p:
        ref = host(p.dgemm(dev(A), dev(B)))
    comm = mf.nccl_comm_create(mf.nccl_unique_id(), 0, 1)
    try:
        with mf.Plan(triples.get(SW), 2, n, shard_rank=0, shard_count=1, nccl_comm=comm,
                     output_mode=mf.OUT_ROWSLAB, input_mode=mf.IN_REPLICATED) as p:
            assert p.c_rows() == n
            assert (host(p.dgemm(dev(A), dev(B))) == ref).all()
            assert (p.dgemm_host(A, B) == ref).all()
    finally:
        mf.nccl_comm_destroy(comm)


# ------------------------------------------------ split-K tail of the leaf launch

@pytest.mark.parametrize("name,levels,n", [(SW, 1, 2048), (SW, 1, 2000), (SW, 1, 4096),
                                           (None, 0, 2048), ("laderman", 1, 1152)])
def test_leaf_split_k_tail(name, levels, n, monkeypatch):
    """Launches that fill the SMs in few waves cut their tail tiles into k-range
    pieces (mf_leaf.cu leaf_tiles; the last piece sums the partials in split
    order).  Exact on integers, deterministic (two runs bitwise equal), within
    the bound on random inputs and close to the unsplit launch (MF_LEAF_SPLIT=1)."""
    t = triples.get(name) if name else None
    A, B = mf_inputs.pair("int1024", n, 54)
    with mf.Plan(t, levels, n) as p:
        Ad, Bd = dev(A), dev(B)
        C1 = host(p.dgemm(Ad, Bd))
        assert (C1 == exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 55)
        Ad, Bd = dev(A), dev(B)
        Cs = host(p.dgemm(Ad, Bd))
        assert (host(p.dgemm(Ad, Bd)) == Cs).all()
    monkeypatch.setenv("MF_LEAF_SPLIT", "1")
    with mf.Plan(t, levels, n) as p:
        Cn = host(p.dgemm(Ad, Bd))
    Cref = oracle.classical(A, B)
    assert_error(scaled(Cs, Cref, A, B), levels)
    assert scaled(Cs, Cn, A, B) <= 1e-14 * max(1, levels)


# ------------------------------------------------ CUDA-graph replay of the step

@pytest.mark.parametrize("name,levels,n", [(SW, 1, 64), (SW, 2, 512), (SW, 1, 2048), (None, 0, 256),
                                           ("laderman", 1, 390)])
def test_graph_replay_matches_eager(name, levels, n):
    """mf_options.graph: call 1 eager, call 2 captured + launched, calls 3+
    replayed -- all bitwise the eager result (the same launches); new
    arguments re-capture; the legacy default stream stays eager."""
    t = triples.get(name) if name else None
    A, B = mf_inputs.pair("uniform", n, 56)
    Ad, Bd = dev(A), dev(B)
    with mf.Plan(t, levels, n) as p:
        ref = host(p.dgemm(Ad, Bd, alpha=0.5))
    side = torch.cuda.Stream()
    with mf.Plan(t, levels, n, graph=True) as p:
        C = torch.empty((n, n), dtype=torch.float64, device="cuda")
        with torch.cuda.stream(side):
            for _ in range(4):
                C.fill_(float("nan"))
                p.dgemm(Ad, Bd, C=C, alpha=0.5, stream=side)
                side.synchronize()
                assert (host(C) == ref).all()
            C2 = torch.empty_like(C)
            for _ in range(3):  # new output pointer and alpha: eager, capture, replay
                p.dgemm(Ad, Bd, C=C2, alpha=1.0, stream=side)
            side.synchronize()
        assert (host(C2) == 2.0 * ref).all()
        p.dgemm(Ad, Bd, C=C2, alpha=0.5)  # legacy stream: eager path
        assert (host(C2) == ref).all()



# ------------------------------------------------ region-overlapped exchange (NEXT-4)

@pytest.mark.parametrize("N", [1, 3, 8])
def test_comm_regions_partials_match_one_shot(N, monkeypatch):
    """comm_regions: the leaf and K6 by 128-aligned row regions (each region's C
    rows reduced while the next computes).  Without a communicator the shard's
    partial C is returned: bitwise the one-shot partial (same launches per
    element; split-K off on both sides), whole and split products alike; the
    N partials sum to the exact product on integers."""
    monkeypatch.setenv("MF_LEAF_SPLIT", "1")
    n = 2048
    A, B = mf_inputs.pair("int1024", n, 57)
    Ad, Bd = dev(A), dev(B)
    total = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    U, V = mf_inputs.pair("uniform", n, 58)
    Ud, Vd = dev(U), dev(V)
    for r in range(N):
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=N, comm_regions=4) as p:
            total += p.dgemm(Ad, Bd)
            Cr = host(p.dgemm(Ud, Vd, alpha=0.5))
        with mf.Plan(triples.get(SW), 2, n, shard_rank=r, shard_count=N) as p:
            assert (host(p.dgemm(Ud, Vd, alpha=0.5)) == Cr).all()
    assert (host(total) == exact(A, B)).all()


def test_comm_regions_nccl_single_rank(monkeypatch):
    """The region-overlapped NCCL exchange on a 1-rank communicator (reduce and
    all-reduce of each region's C rows on the comm stream): bitwise the local
    result with split-K off, within rounding with it on."""
    n = 1024
    A, B = mf_inputs.pair("uniform", n, 59)
    Ad, Bd = dev(A), dev(B)
    comm = mf.nccl_comm_create(mf.nccl_unique_id(), 0, 1)
    try:
        for split in ("1", None):
            if split:
                monkeypatch.setenv("MF_LEAF_SPLIT", split)
            else:
                monkeypatch.delenv("MF_LEAF_SPLIT", raising=False)
            with mf.Plan(triples.get(SW), 2, n) as p:
                ref = host(p.dgemm(Ad, Bd))
            for out_mode in (mf.OUT_ROOT, mf.OUT_ALL):
                with mf.Plan(triples.get(SW), 2, n, shard_rank=0, shard_count=1, nccl_comm=comm,
                             output_mode=out_mode, input_mode=mf.IN_REPLICATED, comm_regions=8) as p:
                    C = host(p.dgemm(Ad, Bd))
                if split:
                    assert (C == ref).all()
                else:
                    assert scaled(C, ref, A, B) <= 1e-14
    finally:
        mf.nccl_comm_destroy(comm)


@pytest.mark.parametrize("regions", [0, 4])
def test_three_level_sharding_n8(regions):
    """NEXT-4 three-level sharding: SW^3's 343 products over 8 ranks (343 =
    8*42 + 7: 42 whole products each plus a 128-row slab of each of the 7
    leftovers), emulated on one GPU, with and without row regions.  The 8
    partial C sum to A*B: exact Freivalds on integers."""
    n, N = 8192, 8
    Ad, Bd = mf_inputs.device_pair("int1024", n, 60)
    total = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    for r in range(N):
        with mf.Plan(triples.get(SW), 3, n, shard_rank=r, shard_count=N, comm_regions=regions) as p:
            pr = p.products()["shard"]
            assert (pr == r).sum() == 42 and (pr == -1).sum() == 7
            total += p.dgemm(Ad, Bd)
    A, B, C = host(Ad), host(Bd), host(total)
    assert oracle.freivalds_int(A, B, C, trials=2) == 0


# ------------------------------------------------ asynchronous host-buffer stream

@pytest.mark.parametrize("name,levels,n,kw", [(SW, 2, 2048, {}), (SW, 1, 1000, {}), (None, 0, 1024, {}),
                                              (SW, 2, 1024, {"level_by_level": True}),
                                              (SW, 3, 1024, {"level_by_level": True, "recurse_levels": 1}),
                                              (SW, 2, 1024, {"fuse_postadd": 1}),
                                              (SW, 2, 1024, {"fuse_postadd": 2}),
                                              (SW, 2, 512, {"max_workspace": 3 * 5 * 128 * 128 * 8}),
                                              (SW, 2, 512, {"leaf": "cublas"})])
def test_host_async_stream_matches_sync(name, levels, n, kw):
    """mf_dgemm_host_async: a stream of 5 products with different pinned inputs,
    enqueued back to back (two device sets, call k+1's copies under call k's
    compute), then mf_host_sync: every C bitwise the synchronous call's.  A
    synchronous call after async ones waits for them.  Plans without the region
    pipeline (level by level, fused, bounded workspace, cuBLAS leaf) stream
    whole matrices on three streams (the fused plan's bulk reductions add in a
    run-dependent order: equal to rounding there)."""
    t = triples.get(name) if name else None
    with mf.Plan(t, levels, n, **kw) as p:
        ins, outs, refs = [], [], []
        for k in range(5):
            A, B = mf_inputs.pair("uniform", n, 70 + k)
            Ah = torch.from_numpy(A).pin_memory(); Bh = torch.from_numpy(B).pin_memory()
            Ch = torch.full((n, n), float("nan"), dtype=torch.float64).pin_memory()
            ins.append((Ah, Bh)); outs.append(Ch)
            refs.append(p.dgemm_host(A, B, alpha=0.5))
        for (Ah, Bh), Ch in zip(ins, outs):
            p.dgemm_host_async_ptr(Ah.data_ptr(), n, Bh.data_ptr(), n, Ch.data_ptr(), n, alpha=0.5)
        p.host_sync()
        for (Ah, Bh), Ch, ref in zip(ins, outs, refs):
            if kw.get("fuse_postadd") == 2:  # bulk-reduction order varies run to run: the bound
                assert scaled(Ch.numpy(), ref, Ah.numpy(), Bh.numpy()) <= 1e-15
            else:
                assert (Ch.numpy() == ref).all()
        Ai, Bi = mf_inputs.pair("int1024", n, 80)
        p.dgemm_host_async_ptr(ins[0][0].data_ptr(), n, ins[0][1].data_ptr(), n, outs[0].data_ptr(), n)
        assert (p.dgemm_host(Ai, Bi) == exact(Ai, Bi)).all()  # drains the async call first
        if kw.get("fuse_postadd") == 2:
            assert scaled(outs[0].numpy(), 2.0 * refs[0], ins[0][0].numpy(), ins[0][1].numpy()) <= 1e-15
        else:
            assert (outs[0].numpy() == 2.0 * refs[0]).all()


# ---- triples outside the catalog (tests/sandwich.py): no compiled-in K4/K6 ----

def _sandwich_pair(name, kind):
    from sandwich import sandwich, P2_INT, P2_DYADIC, P3_INT
    mats = {"int": P2_INT if name == SW else P3_INT, "dyadic": P2_DYADIC}[kind]
    t = oracle.catalog(name)
    U, V, W = sandwich(t.U, t.V, t.W, t.p, *mats)
    return (oracle.Triple(f"{name}-{kind}", t.p, U, V, W),
            triples.Triple(f"{name}-{kind}", t.p, U, V, W))


@pytest.mark.parametrize("path", ["jit", "generic", "generic-terms"])
@pytest.mark.parametrize("name,kind,levels,n", [(SW, "int", 1, 128), (SW, "int", 2, 256),
                                                (SW, "dyadic", 2, 200), ("laderman", "int", 1, 96)])
def test_sandwich_triple_mix_bit_exact(name, kind, levels, n, path, monkeypatch):
    """A triple the library has no compiled-in kernels for, with coefficients
    2, -3, 1/4 ... (tests/sandwich.py): its plan-time generated K4/K6 (`jit`,
    the default) and the table-driven kernels are bitwise the oracle's
    pre-/post-additions on random fp64 -- the general-coefficient terms
    (multiply, then add) included."""
    _mix_path(monkeypatch, path)
    to1, tp = _sandwich_pair(name, kind)
    to = oracle.kron_power(to1, levels)
    A, B = mf_inputs.pair("uniform", n, 41)
    with mf.Plan(tp, levels, n) as p:
        info, pr = p.info(), p.products()
        m = info["leaf_n"]
        for side, X, src, idx in (("A", A, pr["a_src"], pr["a_idx"]), ("B", B, pr["b_src"], pr["b_idx"])):
            nmat = info["n_mat_a"] if side == "A" else info["n_mat_b"]
            out = torch.empty((max(nmat, 1), m, m), dtype=torch.float64, device="cuda")
            p.premix(side, dev(X), out)
            got, ref = host(out), oracle.premix(X, to, side)
            for q in [q for q in range(to.R) if src[q] == 1]:
                assert (got[idx[q]] == ref[q]).all(), (side, q)
        rng = np.random.Generator(np.random.PCG64(43))
        Pp = rng.uniform(-1, 1, size=(to.R, m, m))
        sign = pr["sign"].astype(np.float64)
        C = torch.empty((n, n), dtype=torch.float64, device="cuda")
        p.postmix(dev(Pp), C, alpha=0.625)
        assert (host(C) == oracle.postmix(Pp * sign[:, None, None], to, n, 0.625)).all()


@pytest.mark.parametrize("path", ["jit", "generic"])
@pytest.mark.parametrize("name,kind,levels,n", [(SW, "int", 2, 512), (SW, "dyadic", 2, 400),
                                                ("laderman", "int", 1, 288)])
def test_sandwich_triple_end_to_end(name, kind, levels, n, path, monkeypatch):
    """End to end through mf_dgemm with a non-catalog triple: integer inputs
    bit-exact with the exact product, random inputs within
    1e-13 per level of the oracle's classical product."""
    _mix_path(monkeypatch, path)
    _, tp = _sandwich_pair(name, kind)
    A, B = mf_inputs.pair("int8", n, 44)  # coefficients up to 4: keep partials < 2^53
    with mf.Plan(tp, levels, n) as p:
        assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 45)
        C = host(p.dgemm(dev(A), dev(B)))
    # sandwiched coefficients (2, -3, 1/4) amplify rounding: the ceiling only
    assert scaled(C, oracle.classical(A, B), A, B) <= 1e-13 * levels


@pytest.mark.parametrize("name,levels,n", [(SW, 1, 64), (SW, 2, 64), ("laderman", 1, 36),
                                           ("paper-strassen", 2, 32), ("strassen-1969", 1, 8),
                                           (SW, 3, 64), ("classical-p2", 1, 16)])
def test_tiny_single_launch(name, levels, n, monkeypatch):
    """n <= 64, R^L <= 64: the whole level as one thread-block cluster launch
    (mf_tiny.cu: pre-additions, products and post-additions, the products read
    across the cluster through distributed shared memory).  Integer inputs:
    bit-exact with the exact product; random: within the bound of the oracle,
    and equal to the four-launch path to rounding (the leaf dot products are
    fma chains in both, in different k orders); alpha applied last; graph
    replay bitwise the eager call."""
    t = triples.get(name)
    A, B = mf_inputs.pair("int1024", n, 60)
    with mf.Plan(t, levels, n) as p:
        assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all()
        assert (host(p.dgemm(dev(A), dev(B), alpha=-3.0)) == -3.0 * exact(A, B)).all()
        A, B = mf_inputs.pair("uniform", n, 61)
        Ct = host(p.dgemm(dev(A), dev(B), alpha=0.75))
    monkeypatch.setenv("MF_TINY_OFF", "1")
    with mf.Plan(t, levels, n) as p:
        Cg = host(p.dgemm(dev(A), dev(B), alpha=0.75))
    monkeypatch.delenv("MF_TINY_OFF")
    ref = 0.75 * oracle.fmm(A, B, oracle.catalog(name), levels)
    assert scaled(Ct, ref, A, B) <= 1e-13 * levels
    assert scaled(Ct, Cg, A, B) <= 1e-13 * levels
    s = torch.cuda.Stream()
    with mf.Plan(t, levels, n, graph=True) as p, torch.cuda.stream(s):
        Ad, Bd = dev(A), dev(B)
        C = torch.empty((n, n), dtype=torch.float64, device="cuda")
        outs = []
        for _ in range(3):  # eager, capture, replay
            p.dgemm(Ad, Bd, C, stream=s)
            s.synchronize()
            outs.append(host(C).copy())
    assert (outs[0] == outs[1]).all() and (outs[0] == outs[2]).all()


def test_random_sandwich_triples_generated_kernels_bit_exact():
    """Property over random unimodular block transforms of SW and Laderman
    (tests/sandwich.py): each draw is a fresh triple, so each plan generates and
    compiles new K4/K6; pre- and post-additions bitwise the oracle's, the
    integer product exact."""
    from sandwich import sandwich
    rng = np.random.Generator(np.random.PCG64(77))

    def unimodular(p):
        M = np.eye(p, dtype=np.int64)
        for _ in range(3):
            i, j = rng.choice(p, 2, replace=False)
            E = np.eye(p, dtype=np.int64)
            E[i, j] = rng.choice([-1, 1])
            M = M @ E
        return M

    for name, n in ((SW, 128), ("laderman", 96), (SW, 256)):
        t = oracle.catalog(name)
        for _ in range(2):
            U, V, W = sandwich(t.U, t.V, t.W, t.p, unimodular(t.p), unimodular(t.p), unimodular(t.p))
            to, tp = oracle.Triple("s", t.p, U, V, W), triples.Triple("s", t.p, U, V, W)
            A, B = mf_inputs.pair("uniform", n, int(rng.integers(1 << 30)))
            with mf.Plan(tp, 1, n) as p:
                info, pr = p.info(), p.products()
                m = info["leaf_n"]
                for side, X, src, idx in (("A", A, pr["a_src"], pr["a_idx"]),
                                          ("B", B, pr["b_src"], pr["b_idx"])):
                    nmat = info["n_mat_a"] if side == "A" else info["n_mat_b"]
                    out = torch.empty((max(nmat, 1), m, m), dtype=torch.float64, device="cuda")
                    p.premix(side, dev(X), out)
                    got, ref = host(out), oracle.premix(X, to, side)
                    for q in [q for q in range(to.R) if src[q] == 1]:
                        assert (got[idx[q]] == ref[q]).all()
                Pp = rng.uniform(-1, 1, size=(to.R, m, m))
                sign = pr["sign"].astype(np.float64)
                C = torch.empty((n, n), dtype=torch.float64, device="cuda")
                p.postmix(dev(Pp), C, alpha=1.0)
                assert (host(C) == oracle.postmix(Pp * sign[:, None, None], to, n, 1.0)).all()
                Ai, Bi = mf_inputs.pair("int8", n, 5)
                assert (host(p.dgemm(dev(Ai), dev(Bi))) == exact(Ai, Bi)).all()


def test_random_shape_sweep():
    """40 random draws of (triple, levels, n, alpha, leading-dimension padding,
    input distribution): every plan shape the library accepts -- the small-
    problem cluster kernel (n <= 64), ragged leaves, 64-wide tiles, split-K
    tails, generic and specialised additions -- exact on integer inputs, within
    1e-13 per level of the oracle on random ones."""
    rng = np.random.Generator(np.random.PCG64(99))
    names = [SW, "paper-strassen", "strassen-1969", "laderman", "classical-p2"]
    for _ in range(40):
        name = names[int(rng.integers(len(names)))]
        t = triples.get(name)
        levels = int(rng.integers(1, 3 if t.p == 2 else 2))
        unit = t.p ** levels
        n = unit * int(rng.integers(1, max(2, 600 // unit)))
        pad = int(rng.choice([0, 0, 2, 8, 13]))
        alpha = float(rng.choice([1.0, 0.5, -2.0, 3.25]))
        kind = str(rng.choice(["int8", "uniform"]))
        A, B = mf_inputs.pair(kind, n, int(rng.integers(1 << 30)))
        Ap = np.zeros((n, n + pad)); Ap[:, :n] = A
        Bp = np.zeros((n, n + pad)); Bp[:, :n] = B
        Ad = torch.from_numpy(Ap).cuda()[:, :n]
        Bd = torch.from_numpy(Bp).cuda()[:, :n]
        with mf.Plan(t, levels, n) as p:
            C = host(p.dgemm(Ad, Bd, alpha=alpha))
        if kind == "int8":
            assert (C == alpha * exact(A, B)).all(), (name, levels, n, pad, alpha)
        else:
            ref = alpha * oracle.classical(A, B)
            assert_error(scaled(C, ref, A, B), levels, abs(alpha), (name, levels, n, pad, alpha))


@pytest.mark.parametrize("name,levels,n", [(SW, 2, 2048), (SW, 1, 400), ("laderman", 1, 390), (None, 0, 640)])
def test_two_cta_leaf(name, levels, n, monkeypatch):
    """The two-CTA-per-SM leaf (4 MMA warps, 128 x 64 tiles; the default under
    both folds and for unfused leaves with m <= 1536; forced on and off here):
    integer inputs
    exact, random inputs bitwise the one-CTA leaf (same k order per element)
    with no split-K tail on either side; ragged leaves (m = 200, 130) too."""
    t = triples.get(name) if name else None
    monkeypatch.setenv("MF_LEAF_SPLIT", "1")
    A, B = mf_inputs.pair("int1024", n, 48)
    Ar, Br = mf_inputs.pair("uniform", n, 49)
    out = {}
    for two in ("0", "1"):
        monkeypatch.setenv("MF_LEAF_2CTA", two)
        with mf.Plan(t, levels, n) as p:
            assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all(), two
            out[two] = host(p.dgemm(dev(Ar), dev(Br)))
    assert (out["0"] == out["1"]).all()


@pytest.mark.parametrize("ksub", ["1", "2", "3"])
@pytest.mark.parametrize("two", ["0", "1"])
def test_leaf_ksub_override_on_both_shapes(ksub, two, monkeypatch):
    """MF_LEAF_KSUB (k sub-blocks per ring stage) on the one- and two-CTA leaf:
    the two-CTA shape has only KSUB = 2 and must build its B box and k-block
    count from that, whatever the override (m = 512, 1536: integers exact)."""
    monkeypatch.setenv("MF_LEAF_KSUB", ksub)
    monkeypatch.setenv("MF_LEAF_2CTA", two)
    for n in (2048, 3072):
        A, B = mf_inputs.pair("int1024", n, 52)
        with mf.Plan(triples.get(SW), 2, n) as p:
            assert (host(p.dgemm(dev(A), dev(B))) == exact(A, B)).all(), (n, ksub, two)


@pytest.mark.parametrize("n", [8192, 16384])
def test_leaf_ring_reuse_under_the_ordered_fold(n, monkeypatch):
    """Regression: the leaf's consumer warps released a ring slot (mbarrier
    arrive) while their last fragment loads from it could still be in flight,
    so the next TMA load could overwrite data not yet read.  It showed as wrong
    64 x 32 warp tiles (rows 64-127) in about half of the two-CTA ordered-fold
    launches at n = 8192 and every launch at n = 16384, before the
    fence.proxy.async ahead of the arrive.  Ten launches (four at 16384), each
    bitwise the unfused one-CTA result."""
    t = triples.get(SW)
    A, B = mf_inputs.pair("uniform", n, 51)
    Ad, Bd = dev(A), dev(B)
    monkeypatch.setenv("MF_LEAF_SPLIT", "1")
    monkeypatch.setenv("MF_LEAF_2CTA", "0")
    with mf.Plan(t, 2, n) as p:
        Cu = p.dgemm(Ad, Bd).clone()
    monkeypatch.setenv("MF_LEAF_2CTA", "1")
    with mf.Plan(t, 2, n, fuse_postadd=1) as p:
        for _ in range(10 if n <= 8192 else 4):
            assert torch.equal(p.dgemm(Ad, Bd), Cu)


@pytest.mark.parametrize("n,bn,two", [(2048, "64", "0"), (4096, "64", "0"), (2048, "128", "0"),
                                      (2048, "64", "1"), (4096, "64", "1")])
def test_fused_ordered_concurrent_dependencies(n, bn, two, monkeypatch):
    """The ordered fold where its flags really order concurrent CTAs: few tiles
    per product (n = 2048: 16 / 32 tiles; n = 4096 with 64-wide tiles: 128), so
    the products of one tile position run in the same wave and wait on each
    other; one CTA per SM (128- or 64-wide tiles) and two.  Five launches,
    each bitwise the flat unfused result."""
    t = triples.get(SW)
    A, B = mf_inputs.pair("uniform", n, 50)
    monkeypatch.setenv("MF_LEAF_BN", bn)
    monkeypatch.setenv("MF_LEAF_2CTA", two)
    Cf, Cu = _ordered_and_flat(monkeypatch, t, 2, n, A, B, 1.0)
    assert (Cf == Cu).all()
    with monkeypatch.context() as mp:
        mp.setenv("MF_MIX_GENERIC", "1")
        with mf.Plan(t, 2, n, fuse_postadd=1) as p:
            Ad, Bd = dev(A), dev(B)
            for _ in range(5):
                assert (host(p.dgemm(Ad, Bd)) == Cu).all()
