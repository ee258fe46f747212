"""Pins for the CPU oracle (oracle/): checked against what the paper and the
mathematics fix, never against the oracle itself or the CUDA path.

Pins:
* the paper's printed matrices (tests/golden/paper_strassen.txt) and its
  worked expansions C0 = P3+P5, C3 = P0+P6;
* exact Brent equations for every triple, and the product
  counts of PAPER.md L271-278 for Kronecker compositions;
* classical product: SPEC.md L92's worked example, identities, and exact
  integer products from numpy's int64 matmul (an independent library routine);
* the recursion interpreter: brute force at n = p^L with scalar leaves, integer
  exactness ("integer computations are correct, always"),
  error bounds against an extended-precision library product;
* Freivalds/sampled-entry helpers detect a planted error.
"""
import os

import numpy as np
import pytest

import oracle
import mf_inputs

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_strassen.txt")


def load_golden():
    sections, cur = {}, None
    with open(GOLDEN) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if line.startswith("["):
                cur = line.strip("[]")
                sections[cur] = []
            else:
                sections[cur].append(line.split())
    return sections


def exact_product(A, B):
    """Exact integer product via numpy int64 matmul (values well below 2^63)."""
    return (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)


# ---------------------------------------------------------------- catalog / Brent

def test_paper_strassen_matches_printed_matrices():
    g = load_golden()
    a = np.array([[int(v) for v in r[1:]] for r in g["a"]], dtype=float)
    b = np.array([[int(v) for v in r[1:]] for r in g["b"]], dtype=float)
    labels = [r[0] for r in g["ct"]]
    ct = np.array([[int(v) for v in r[1:]] for r in g["ct"]], dtype=float)
    W = np.zeros_like(ct)
    for lab, row in zip(labels, ct):
        W[int(lab[1:])] = row
    t = oracle.catalog("paper-strassen")
    assert (t.U == a).all() and (t.V == b).all() and (t.W == W).all()


def test_printed_row_labels_are_needed():
    """Reading R1: with the printed labels C0,C2,C1,C3 the triple is exact;
    read naively as C0,C1,C2,C3 it violates 8 of the 64 Brent equations."""
    g = load_golden()
    t = oracle.catalog("paper-strassen")
    ct = np.array([[int(v) for v in r[1:]] for r in g["ct"]], dtype=float)
    naive = oracle.Triple("naive", 2, t.U, t.V, ct)
    assert oracle.brent_check(t) == (0, None)
    bad, _ = oracle.brent_check(naive)
    assert bad == 8


@pytest.mark.parametrize("name,p,R", [("paper-strassen", 2, 7), ("strassen-winograd", 2, 7),
                                      ("strassen-1969", 2, 7), ("laderman", 3, 23),
                                      ("classical-p2", 2, 8), ("classical-p3", 3, 27)])
def test_catalog_brent_exact(name, p, R):
    t = oracle.catalog(name)
    assert (t.p, t.R) == (p, R)
    assert oracle.brent_check(t) == (0, None)
    # no dead products
    assert (np.abs(t.U).sum(0) > 0).all() and (np.abs(t.V).sum(0) > 0).all()


def test_mutated_strassen_fails_only_on_c3():
    """W[3][0] 1 -> 0 breaks exactly the C3 (z=3) equations."""
    t = oracle.catalog("paper-strassen")
    W = t.W.copy()
    assert W[3, 0] == 1
    W[3, 0] = 0
    bad_t = oracle.Triple("mut", 2, t.U, t.V, W)
    bad, first = oracle.brent_check(bad_t)
    assert bad > 0 and first[2] == 3
    # brute-force list of failing z indices
    fails = set()
    for x in range(4):
        for y in range(4):
            for z in range(4):
                s = (bad_t.U[x] * bad_t.V[y] * bad_t.W[z]).sum()
                i, k = divmod(x, 2); k2, j = divmod(y, 2); i2, j2 = divmod(z, 2)
                if s != int(k == k2 and i == i2 and j == j2):
                    fails.add(z)
    assert fails == {3}


def test_worked_expansions():
    """C0 = P3+P5 = A1*B2 + A0*B0 (matrix reading, R2) and
    C3 = P0+P6 = (A2-A3)*B1 + A3*(B1+B3)."""
    g = load_golden()
    t = oracle.catalog("paper-strassen")
    for row in g["worked"]:
        i = int(row[0][1:])
        used = sorted(int(v[1:]) for v in row[1:])
        assert sorted(np.nonzero(t.W[i])[0].tolist()) == used
        assert all(t.W[i, q] == 1 for q in used)
    # P5 = A0*B0, P3 = A1*B2 (column 3 of b selects B2, not the prose's B3)
    assert np.nonzero(t.U[:, 5])[0].tolist() == [0] and np.nonzero(t.V[:, 5])[0].tolist() == [0]
    assert np.nonzero(t.U[:, 3])[0].tolist() == [1] and np.nonzero(t.V[:, 3])[0].tolist() == [2]
    # P0 = (A2 - A3) * B1, P6 = A3 * (B1 + B3)
    assert t.U[:, 0].tolist() == [0, 0, 1, -1] and t.V[:, 0].tolist() == [0, 1, 0, 0]
    assert t.U[:, 6].tolist() == [0, 0, 0, 1] and t.V[:, 6].tolist() == [0, 1, 0, 1]
    # numerically, on scalars: C0 = A0B0 + A1B2 and C3 = A2B1 + A3B3
    A = np.array([[2.0, 3.0], [5.0, 7.0]]); B = np.array([[11.0, 13.0], [17.0, 19.0]])
    C = oracle.fmm(A, B, t, 1)
    assert C[0, 0] == 2 * 11 + 3 * 17 and C[1, 1] == 5 * 13 + 7 * 19


def test_kron_counts_match_paper():
    """factor -> products 4->49, 6->161 (both orders),
    9->529, 12->1127; compositions are exact."""
    g = load_golden()
    counts = {int(a): int(b) for a, b in g["counts"]}
    SW = oracle.catalog("strassen-winograd")
    LD = oracle.catalog("laderman")
    cases = {4: [oracle.kron(SW, SW)], 6: [oracle.kron(SW, LD), oracle.kron(LD, SW)],
             9: [oracle.kron(LD, LD)], 12: [oracle.kron(oracle.kron(SW, SW), LD)]}
    for p, ts in cases.items():
        for t in ts:
            assert (t.p, t.R) == (p, counts[p])
            if p <= 9:
                assert oracle.brent_check(t) == (0, None)
    assert counts[2] == SW.R and counts[3] == LD.R


def test_kron_p12_brent():
    t = oracle.kron(oracle.kron(oracle.catalog("strassen-winograd"),
                                oracle.catalog("strassen-winograd")), oracle.catalog("laderman"))
    assert oracle.brent_check(t) == (0, None)


def test_kron_of_classical_is_classical_p4_up_to_permutation():
    """classical-p2 (x) classical-p2 = classical-p4 up to a column permutation."""
    c2 = oracle.catalog("classical-p2")
    k = oracle.kron(c2, c2)
    # classical-p4 built from Eq. (recursion)'s definition directly
    p = 4
    cols = set()
    for q in range(k.R):
        x = int(np.nonzero(k.U[:, q])[0][0]); y = int(np.nonzero(k.V[:, q])[0][0])
        z = int(np.nonzero(k.W[:, q])[0][0])
        i, kk = divmod(x, p); k2, j = divmod(y, p); i2, j2 = divmod(z, p)
        assert kk == k2 and i == i2 and j == j2
        cols.add((i, j, kk))
    assert len(cols) == 64


# ---------------------------------------------------------------- classical (O3)

def test_classical_spec_example():
    """[[1,2],[3,4]]*[[5,6],[7,8]] = [[19,22],[43,50]]."""
    C = oracle.classical(np.array([[1.0, 2], [3, 4]]), np.array([[5.0, 6], [7, 8]]))
    assert C.tolist() == [[19, 22], [43, 50]]


def test_classical_identity_and_integers():
    A = mf_inputs.uniform(37, 3)
    I = np.eye(37)
    assert (oracle.classical(I, A) == A).all() and (oracle.classical(A, I) == A).all()
    A, B = mf_inputs.pair("int1024", 97, 5)
    assert (oracle.classical(A, B) == exact_product(A, B)).all()


def test_classical_k_ascending_single_rounding_order():
    """Each C[i][j] is the k-ascending sum of separately rounded products:
    compare against an explicit Python loop on a tiny random case."""
    A, B = mf_inputs.pair("uniform", 6, 11)
    C = oracle.classical(A, B)
    for i in range(6):
        for j in range(6):
            acc = 0.0
            for k in range(6):
                acc = acc + float(A[i, k]) * float(B[k, j])
            assert C[i, j] == acc


def test_classical_close_to_extended_precision():
    A, B = mf_inputs.pair("uniform", 128, 1)
    ref = A.astype(np.longdouble) @ B.astype(np.longdouble)
    err = np.abs(oracle.classical(A, B) - ref).max() / 128
    assert err < 128 * 2.0 ** -53


# ---------------------------------------------------------------- interpreter (O4)

def tiny_exact(n, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.integers(-9, 10, (n, n)).astype(float), rng.integers(-9, 10, (n, n)).astype(float))


@pytest.mark.parametrize("name,levels", [("strassen-winograd", 1), ("paper-strassen", 1),
                                         ("strassen-1969", 1), ("laderman", 1),
                                         ("strassen-winograd", 2), ("strassen-winograd", 3),
                                         ("laderman", 2), ("classical-p2", 2)])
def test_fmm_brute_force_scalar_leaves(name, levels):
    """n = p^L: every leaf is a scalar product; result equals the exact product."""
    t = oracle.catalog(name)
    n = t.p ** levels
    for seed in range(5):
        A, B = tiny_exact(n, seed)
        assert (oracle.fmm(A, B, t, levels) == exact_product(A, B)).all()


@pytest.mark.parametrize("outer,inner", [("strassen-winograd", "laderman"),
                                         ("laderman", "strassen-winograd"),
                                         ("strassen-winograd", "strassen-winograd"),
                                         ("paper-strassen", "paper-strassen")])
def test_fmm_flattened_brute_force(outer, inner):
    """One level of a Kronecker-flattened triple at n = p_o*p_i (scalar leaves)."""
    t = oracle.kron(oracle.catalog(outer), oracle.catalog(inner))
    for seed in range(3):
        A, B = tiny_exact(t.p, seed)
        assert (oracle.fmm(A, B, t, 1) == exact_product(A, B)).all()


@pytest.mark.parametrize("n,name,levels", [(12, "strassen-winograd", 2), (24, "strassen-winograd", 3),
                                           (36, "laderman", 2), (48, "strassen-winograd", 4),
                                           (64, "strassen-winograd", 1), (128, "strassen-winograd", 2),
                                           (72, "laderman", 1)])
def test_fmm_integer_exact(n, name, levels):
    """integer computations are exact."""
    t = oracle.catalog(name)
    A, B = mf_inputs.pair("int1024", n, 7)
    assert (oracle.fmm(A, B, t, levels) == exact_product(A, B)).all()


def test_fmm_flattened_equals_recursive_on_integers():
    """kron(t,t) at one level is the two-level algorithm."""
    SW = oracle.catalog("strassen-winograd")
    F44 = oracle.kron_power(SW, 2)
    A, B = mf_inputs.pair("int1024", 64, 3)
    C1 = oracle.fmm(A, B, F44, 1)
    C2 = oracle.fmm(A, B, SW, 2)
    assert (C1 == C2).all() and (C1 == exact_product(A, B)).all()


def test_block_impulse_routing():
    """A = 1 on block x, B = 1 on block y: C = m*1 on block (i,j) iff
    x=(i,k), y=(k,j); zero elsewhere (SURVEY.md §8c block-impulse pin)."""
    t = oracle.catalog("laderman")
    P, m = 3, 2
    n = P * m
    for x in range(9):
        for y in range(9):
            A = mf_inputs.block_impulse(n, P, x)
            B = mf_inputs.block_impulse(n, P, y)
            C = oracle.fmm(A, B, t, 1)
            i, k = divmod(x, P); k2, j = divmod(y, P)
            E = np.zeros((n, n))
            if k == k2:
                E[i * m:(i + 1) * m, j * m:(j + 1) * m] = m
            assert (C == E).all()


def test_fmm_alpha_applied_last():
    """C = alpha*A*B: alpha is applied once after the W-sum."""
    t = oracle.catalog("strassen-winograd")
    A, B = mf_inputs.pair("int8", 32, 2)
    assert (oracle.fmm(A, B, t, 1, alpha=3.0) == 3.0 * exact_product(A, B)).all()
    A, B = mf_inputs.pair("uniform", 32, 2)
    C1 = oracle.fmm(A, B, t, 1)
    assert (oracle.fmm(A, B, t, 1, alpha=-0.7) == -0.7 * C1).all()


def test_fmm_indivisible():
    with pytest.raises(ValueError):
        oracle.fmm(np.zeros((10, 10)), np.zeros((10, 10)), oracle.catalog("laderman"), 1)


@pytest.mark.parametrize("name,levels", [("strassen-winograd", 1), ("strassen-winograd", 2),
                                         ("laderman", 1)])
def test_fmm_random_error_bound(name, levels):
    """north_star: max scaled error <= 1e-13 per level, vs extended precision."""
    t = oracle.catalog(name)
    n = 144 if t.p == 3 else 128
    A, B = mf_inputs.pair("uniform", n, 0)
    ref = A.astype(np.longdouble) @ B.astype(np.longdouble)
    C = oracle.fmm(A, B, t, levels)
    err = float(np.abs(C - ref).max()) / n
    assert 0 < err <= 1e-13 * levels
    assert err < 1e-15  # actual magnitude is ~1e-16 (SURVEY.md verified fact 7)


def test_error_grows_with_levels():
    """median error of L=2 >= L=1 >= classical (n=64, seed 42)."""
    SW = oracle.catalog("strassen-winograd")
    rng_seeds = range(42, 42 + 30)
    errs = {0: [], 1: [], 2: []}
    for s in rng_seeds:
        A, B = mf_inputs.pair("uniform", 64, s)
        ref = A.astype(np.longdouble) @ B.astype(np.longdouble)
        for L in (0, 1, 2):
            C = oracle.classical(A, B) if L == 0 else oracle.fmm(A, B, SW, L)
            errs[L].append(float(np.abs(C - ref).max()))
    med = {L: np.median(v) for L, v in errs.items()}
    assert med[2] >= med[1] >= med[0]
    assert max(max(v) for v in errs.values()) <= 1e-10


def test_premix_postmix_compose_to_fmm():
    """One level split into its steps: postmix(classical(T_q, S_q)) == fmm(...) bitwise."""
    t = oracle.catalog("strassen-winograd")
    A, B = mf_inputs.pair("uniform", 48, 9)
    T = oracle.premix(A, t, "A")
    S = oracle.premix(B, t, "B")
    P = np.stack([oracle.classical(T[q], S[q]) for q in range(t.R)])
    assert (oracle.postmix(P, t, 48) == oracle.fmm(A, B, t, 1)).all()
    # premix on integers equals the defining block sums
    A = mf_inputs.integers(8, 1)
    T = oracle.premix(A, t, "A")
    blocks = [A[:4, :4], A[:4, 4:], A[4:, :4], A[4:, 4:]]
    for q in range(t.R):
        assert (T[q] == sum(t.U[k, q] * blocks[k] for k in range(4))).all()


@pytest.mark.parametrize("name", ["strassen-winograd", "laderman"])
@pytest.mark.parametrize("alpha", [3.0, -0.7, 0.1, -1.0, 0.0])
def test_postmix_alpha_applied_once_after_the_sum(name, alpha):
    """or_postmix's alpha branch (C = alpha*A*B; reading R8:
    alpha once, after the W-sum).  Pins: (1) integer-valued P: equals alpha
    times the block sums C_i = sum_q W[i][q] P_q done in exact int64
    arithmetic; (2) random P: equals alpha * postmix(alpha=1) bitwise, while
    applying alpha to every term (a plausible mistake) rounds differently --
    the test shows it can tell the two apart; (3) alpha = 0 gives zeros."""
    t = oracle.catalog(name)
    p, R = t.p, t.R
    m = 12
    n = p * m
    rng = np.random.Generator(np.random.PCG64(77))
    Pi = rng.integers(-1000, 1001, size=(R, m, m)).astype(np.float64)
    C = oracle.postmix(Pi, t, n, alpha)
    Wi = t.W.astype(np.int64)
    for i in range(p * p):
        blk = C[(i // p) * m:(i // p + 1) * m, (i % p) * m:(i % p + 1) * m]
        exact = sum(Wi[i, q] * Pi[q].astype(np.int64) for q in range(R))
        assert (blk == alpha * exact.astype(np.float64)).all()
    Pr = rng.uniform(-1, 1, size=(R, m, m))
    C1 = oracle.postmix(Pr, t, n, 1.0)
    Ca = oracle.postmix(Pr, t, n, alpha)
    assert (Ca == alpha * C1).all()
    if alpha in (0.1, -0.7):
        per_term = np.zeros((n, n))
        for i in range(p * p):
            acc = None
            for q in range(R):
                if t.W[i, q] != 0:
                    term = alpha * (t.W[i, q] * Pr[q])
                    acc = term if acc is None else acc + term
            per_term[(i // p) * m:(i // p + 1) * m, (i % p) * m:(i % p + 1) * m] = acc
        assert (per_term != Ca).any()
    if alpha == 0.0:
        assert (Ca == 0).all()


# ---------------------------------------------------------------- large-n helpers (O7)

def test_freivalds_detects_planted_error():
    A, B = mf_inputs.pair("int1024", 96, 4)
    C = exact_product(A, B)
    assert oracle.freivalds_int(A, B, C) == 0
    C[17, 33] += 1
    assert oracle.freivalds_int(A, B, C) > 0
    assert oracle.freivalds_int(A + 0.5, B, C) == -1


def test_sample_entries_match_classical():
    A, B = mf_inputs.pair("uniform", 64, 8)
    C = oracle.classical(A, B)
    rows = np.array([0, 5, 63, 17]); cols = np.array([3, 63, 0, 17])
    assert (oracle.sample_entries(A, B, rows, cols) == C[rows, cols]).all()


# ---- triples outside the catalog (tests/sandwich.py): general coefficients ----

def _sandwiched(name, mats):
    from sandwich import sandwich
    t = oracle.catalog(name)
    return oracle.Triple(f"{name}-sandwich", t.p, *sandwich(t.U, t.V, t.W, t.p, *mats))


def test_sandwich_triples_valid():
    """A sandwich X A Y^-1, Y B Z^-1 of a valid triple is valid (tests/sandwich.py):
    the integer ones pass the exact Brent check with coefficients up to 3 in
    magnitude; the dyadic one (coefficients 1/4, 1/2, 4) is refused by the
    integer check but reproduces exact products on scalar leaves (brute force,
    n = p) and on integer matrices through two levels -- the interpreter's
    general-coefficient terms (multiply, then add) are exercised."""
    from sandwich import P2_INT, P2_DYADIC, P3_INT
    rng = np.random.Generator(np.random.PCG64(77))
    for name, mats, integral in (("strassen-winograd", P2_INT, True), ("laderman", P3_INT, True),
                                 ("strassen-winograd", P2_DYADIC, False)):
        s = _sandwiched(name, mats)
        coefs = np.unique(np.concatenate([s.U.ravel(), s.V.ravel(), s.W.ravel()]))
        assert np.abs(coefs).max() >= 2
        if integral:
            assert oracle.brent_check(s) == (0, None)
        else:
            with pytest.raises(ValueError):
                oracle.brent_check(s)
        for _ in range(10):
            A = rng.integers(-9, 10, (s.p, s.p)).astype(np.float64)
            B = rng.integers(-9, 10, (s.p, s.p)).astype(np.float64)
            assert (oracle.fmm(A, B, s, 1) == A @ B).all()
        n = s.p * s.p * 8
        A = rng.integers(-1024, 1025, (n, n)).astype(np.float64)
        B = rng.integers(-1024, 1025, (n, n)).astype(np.float64)
        assert (oracle.fmm(A, B, s, 2) == oracle.classical(A, B)).all()
    # a corrupted sandwich fails the exact check
    s = _sandwiched("strassen-winograd", P2_INT)
    W = s.W.copy()
    W[0, 0] += 1
    assert oracle.brent_check(oracle.Triple("bad", 2, s.U, s.V, W))[0] > 0


def test_random_sandwiches_stay_valid():
    """Property: for random unimodular X, Y, Z (products of elementary integer
    matrices), the sandwich of a valid triple is valid -- exact Brent check,
    and the interpreter reproduces exact products on scalar leaves.  A dropped
    or mis-indexed term anywhere in or_brent_check / or_fmm's combination
    code would break one of these on some draw."""
    from sandwich import sandwich
    rng = np.random.Generator(np.random.PCG64(2024))

    def unimodular(p):
        M = np.eye(p, dtype=np.int64)
        for _ in range(3):
            i, j = rng.choice(p, 2, replace=False)
            E = np.eye(p, dtype=np.int64)
            E[i, j] = rng.choice([-1, 1])
            M = M @ E
        return M

    for name in ("strassen-winograd", "laderman", "strassen-1969"):
        t = oracle.catalog(name)
        for _ in range(6):
            s = oracle.Triple("s", t.p, *sandwich(t.U, t.V, t.W, t.p, unimodular(t.p),
                                                  unimodular(t.p), unimodular(t.p)))
            assert oracle.brent_check(s) == (0, None)
            A = rng.integers(-9, 10, (t.p, t.p)).astype(np.float64)
            B = rng.integers(-9, 10, (t.p, t.p)).astype(np.float64)
            assert (oracle.fmm(A, B, s, 1) == A @ B).all()
