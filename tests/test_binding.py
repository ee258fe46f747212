"""CPU-side checks of the boundary (no GPU compute): libmf.so loads, exports
every entry point include/mf.h declares, and mf_plan's host-side validation
(exact Brent check, divisibility, arguments) answers with the documented
status codes.  Also: the product catalog equals the oracle's."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2312_12732_b200 as mf
from paper_2312_12732_b200 import triples

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mf.h")).read()
    return sorted(set(re.findall(r"^(?:mf_status|const char\*)\s+(mf_\w+)\s*\(", src, re.M)))


def test_library_exports_every_header_symbol():
    names = header_functions()
    assert len(names) >= 14
    lib = ctypes.CDLL(mf.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(mf.EXPORTS)


def test_version():
    assert "sm_100a" in mf.version()


@pytest.mark.parametrize("name", list(triples.CATALOG))
def test_product_catalog_matches_oracle(name):
    t = triples.get(name)
    o = oracle.catalog(name)
    assert t.p == o.p and t.R == o.R
    assert (t.U == o.U).all() and (t.V == o.V).all() and (t.W == o.W).all()


def _plan_status(p, R, U, V, W, levels, n, **kw):
    h = ctypes.c_void_p()
    opt = mf.mf_options()
    opt.struct_size = ctypes.sizeof(mf.mf_options)
    opt.device = -1
    for k, v in kw.items():
        setattr(opt, k, v)
    args = [np.ascontiguousarray(x, dtype=np.float64) if x is not None else None for x in (U, V, W)]
    st = mf._lib.mf_plan(ctypes.byref(h), p, R, *[a.ctypes.data if a is not None else None
                                                    for a in args], levels, n, ctypes.byref(opt))
    assert not h.value or st == 0
    return st, mf._lib.mf_last_error().decode()


def test_plan_rejects_bad_triple_with_first_violation():
    t = triples.PAPER_STRASSEN
    W = t.W.copy()
    W[3, 0] = 0  # SPEC.md L193 mutation
    st, msg = _plan_status(2, 7, t.U, t.V, W, 1, 64)
    assert st == mf.MF_ERR_BAD_TRIPLE and "Brent" in msg
    # the printed (unlabelled) c^t row order is also rejected (reading R1)
    Wn = t.W[[0, 2, 1, 3]]
    st, msg = _plan_status(2, 7, t.U, t.V, Wn, 1, 64)
    assert st == mf.MF_ERR_BAD_TRIPLE and "8 of 64" in msg


def test_plan_rejects_dead_product():
    t = triples.STRASSEN_WINOGRAD
    U = np.concatenate([t.U, np.zeros((4, 1))], 1)
    V = np.concatenate([t.V, np.ones((4, 1))], 1)
    W = np.concatenate([t.W, np.zeros((4, 1))], 1)
    st, msg = _plan_status(2, 8, U, V, W, 1, 64)
    assert st == mf.MF_ERR_BAD_TRIPLE and "all-zero" in msg


def test_plan_rejects_indivisible_and_bad_args():
    t = triples.LADERMAN
    st, msg = _plan_status(3, 23, t.U, t.V, t.W, 1, 100)
    assert st == mf.MF_ERR_INDIVISIBLE and "100" in msg and "p = 3" in msg
    t = triples.STRASSEN_WINOGRAD
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 1002)  # 1002 % 4 != 0
    assert st == mf.MF_ERR_INDIVISIBLE
    st, _ = _plan_status(2, 7, t.U, t.V, t.W, -1, 64)
    assert st == mf.MF_ERR_INVALID_ARG
    st, _ = _plan_status(2, 7, t.U, t.V, t.W, 1, 0)
    assert st == mf.MF_ERR_INVALID_ARG
    st, _ = _plan_status(2, 7, None, None, None, 1, 64)
    assert st == mf.MF_ERR_INVALID_ARG
    st, _ = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, shard_rank=3, shard_count=2)
    assert st == mf.MF_ERR_INVALID_ARG


def test_plan_rejects_non_dyadic_coefficients():
    t = triples.STRASSEN_WINOGRAD
    U = t.U.copy() / 3.0
    st, _ = _plan_status(2, 7, U, t.V, t.W, 1, 64)
    assert st == mf.MF_ERR_UNSUPPORTED


def test_plan_accepts_dyadic_rescaling_up_to_device():
    """U/2, W*2 is the same bilinear map; the exact dyadic Brent check accepts it
    (the plan then fails only for lack of a GPU here, or succeeds on one)."""
    t = triples.STRASSEN_WINOGRAD
    st, msg = _plan_status(2, 7, t.U / 2, t.V, t.W * 2, 1, 64)
    assert st in (mf.MF_OK, mf.MF_ERR_CUDA, mf.MF_ERR_OUT_OF_MEMORY), msg


@pytest.mark.parametrize("name,levels,nmat", [("strassen-winograd", 1, 4), ("strassen-winograd", 2, 40),
                                              ("laderman", 1, 14), ("paper-strassen", 1, 4)])
def test_host_only_plan_classification(name, levels, nmat):
    """mf_plan step 5 on the host: single +-1 columns alias (SURVEY App. A:
    SW 4 T + 4 S materialised, SW^2 40 + 40, Laderman 14 + 14)."""
    t = triples.get(name)
    p = mf.Plan(t, levels, t.p ** levels * 8, host_only=True)
    info = p.info()
    assert info["n_products"] == t.R ** levels and info["workspace_bytes"] == 0
    assert info["n_mat_a"] == nmat and info["n_mat_b"] == nmat
    pr = p.products()
    assert (pr["a_src"] == 1).sum() == nmat and (pr["shard"] == 0).all()
    # aliased operands carry their block index, materialised ones a dense slot index
    assert sorted(pr["a_idx"][pr["a_src"] == 1].tolist()) == list(range(nmat))
    buf = np.zeros(16)
    st = mf._lib.mf_dgemm(p._h, 1.0, buf.ctypes.data, 4, buf.ctypes.data, 4, buf.ctypes.data, 4, None)
    assert st == mf.MF_ERR_INVALID_ARG and "host-only" in mf._lib.mf_last_error().decode()


def test_host_only_sharding_balanced():
    p = mf.Plan(triples.STRASSEN_WINOGRAD, 2, 64, shard_rank=0, shard_count=8, host_only=True)
    sh = p.products()["shard"]
    counts = np.bincount(sh, minlength=8)
    assert counts.sum() == 49 and counts.max() - counts.min() <= 1
    assert (np.diff(sh) >= 0).all()  # contiguous ranges


@pytest.mark.parametrize("N", [2, 3, 5, 8])
def test_host_only_split_sharding_exact_balance(N):
    """49 products on N ranks = floor(49/N) whole products each plus a
    row slab of every leftover product; the slabs tile [0, m) exactly once."""
    n = 4096
    m = n // 4
    slabs, whole = [], []
    for r in range(N):
        p = mf.Plan(triples.STRASSEN_WINOGRAD, 2, n, shard_rank=r, shard_count=N, host_only=True)
        sh = p.products()["shard"]
        whole.append(int((sh == r).sum()))
        assert int((sh == -1).sum()) == 49 % N
        slabs.append(p.shard_rows())
    assert whole == [49 // N] * N
    assert slabs[0][0] == 0 and slabs[-1][1] == m
    assert all(slabs[i][1] == slabs[i + 1][0] for i in range(N - 1))
    assert all(a % 128 == 0 for a, _ in slabs)


def test_product_kron_matches_oracle_kron():
    """triples.kron (product side) and or_kron (oracle) agree for the mixed chains
    of PAPER.md L275-278 (6 = 2x3 and 3x2 as 7*23 products)."""
    for o, i in (("strassen-winograd", "laderman"), ("laderman", "strassen-winograd"),
                 ("strassen-winograd", "strassen-winograd")):
        a = triples.kron(triples.get(o), triples.get(i))
        b = oracle.kron(oracle.catalog(o), oracle.catalog(i))
        assert a.p == b.p and a.R == b.R
        assert (a.U == b.U).all() and (a.V == b.V).all() and (a.W == b.W).all()


def test_fused_postadd_option_validation():
    """mf_options.fuse_postadd (include/mf.h): needs levels >= 1 and the flattened
    path; recurse_levels must be >= 0; all checked before any device work."""
    t = triples.STRASSEN_WINOGRAD
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 0, 64, fuse_postadd=1, host_only=1)
    assert st == mf.MF_ERR_UNSUPPORTED and "levels" in msg
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 64, fuse_postadd=1, level_by_level=1, host_only=1)
    assert st == mf.MF_ERR_UNSUPPORTED and "level_by_level" in msg
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 64, level_by_level=1, recurse_levels=-1,
                           host_only=1)
    assert st == mf.MF_ERR_INVALID_ARG and "recurse_levels" in msg
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 64, comm_regions=-2, host_only=1)
    assert st == mf.MF_ERR_INVALID_ARG and "comm_regions" in msg
    p = mf.Plan(t, 2, 64, fuse_postadd=True, host_only=True)
    assert p.info()["n_products"] == 49
    p.close()
    # the ordered fold (1) is for unsharded plans; sharded plans take the
    # bulk-reduction fold (2); other values are refused
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 64, fuse_postadd=1, shard_count=2, host_only=1)
    assert st == mf.MF_ERR_UNSUPPORTED and "ordered" in msg
    p = mf.Plan(t, 2, 64, fuse_postadd=2, shard_count=2, shard_rank=1, host_only=True)
    p.close()
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 64, fuse_postadd=3, host_only=1)
    assert st == mf.MF_ERR_INVALID_ARG and "fuse_postadd" in msg


def test_output_mode_and_leaf_validation():
    """MF_OUT_ROWSLAB needs n % shard_count == 0; unknown modes/leaf kinds and
    fuse_postadd with the cuBLAS leaf are rejected on the host."""
    t = triples.STRASSEN_WINOGRAD
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, output_mode=mf.OUT_ROWSLAB, shard_count=3,
                           host_only=1)
    assert st == mf.MF_ERR_INVALID_ARG and "ROWSLAB" in msg
    st, _ = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, output_mode=mf.OUT_ROWSLAB, shard_count=4,
                         host_only=1)
    assert st == mf.MF_OK
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, output_mode=7, host_only=1)
    assert st == mf.MF_ERR_INVALID_ARG and "output_mode" in msg
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, leaf=9, host_only=1)
    assert st == mf.MF_ERR_INVALID_ARG and "leaf" in msg
    st, msg = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, leaf=mf.LEAF_CUBLAS, fuse_postadd=1,
                           host_only=1)
    assert st == mf.MF_ERR_UNSUPPORTED


def test_jit_generator_compiles_without_gpu():
    """mf_jit_compile_check (include/mf.h): the plan-time K4/K6 generator emits
    CUDA that NVRTC compiles for sm_100a here, on the GPU-less box -- the
    output-major shape for a pre-addition (16 inputs held, 256-bit vectors) and
    the input-major shape for a post-addition (16 accumulators, 128-bit);
    tables too large for registers are refused, not miscompiled."""
    import numpy as np
    from paper_2312_12732_b200 import triples
    sw = triples.get("strassen-winograd")
    f = triples.kron(sw, sw)
    U = np.array(f.U, dtype=float).reshape(16, 49)
    W = np.array(f.W, dtype=float).reshape(16, 49)
    mat = [q for q in range(49) if np.count_nonzero(U[:, q]) != 1]
    try:
        vw, nb = mf.jit_compile_check(U[:, mat].T, 4, 0)
    except mf.MfError as e:
        if "NVRTC not available" in str(e):
            pytest.skip("no NVRTC in this image")
        raise
    assert vw == 4 and nb > 0
    vw, nb = mf.jit_compile_check(W, 0, 4)
    assert vw == 2 and nb > 0
    # a non-unit coefficient (hex literal, exact) and alpha paths compile too
    vw, _ = mf.jit_compile_check(np.array([[0.5, -3.0, 1.0]]), 0, 0)
    assert vw == 4
    big = np.ones((80, 80))
    with pytest.raises(mf.MfError) as e:
        mf.jit_compile_check(big, 0, 0)
    assert e.value.status == mf.MF_ERR_UNSUPPORTED


def test_plan_accepts_sandwiched_triples():
    """mf_plan's own Brent check (include/mf.h: exact for integer, dyadic-exact
    for dyadic coefficients) accepts triples outside the catalog with general
    coefficients (tests/sandwich.py) and rejects a corrupted one."""
    from sandwich import sandwich, P2_INT, P2_DYADIC, P3_INT
    for name, mats in (("strassen-winograd", P2_INT), ("strassen-winograd", P2_DYADIC),
                       ("laderman", P3_INT)):
        t = triples.get(name)
        U, V, W = sandwich(t.U, t.V, t.W, t.p, *mats)
        s = triples.Triple(f"{name}-sandwich", t.p, U, V, W)
        for levels in (1, 2):
            p = mf.Plan(s, levels, t.p ** levels * 8, host_only=True)
            assert p.info()["n_products"] == t.R ** levels
            p.close()
        W = W.copy()
        W[0, 0] += 1
        with pytest.raises(mf.MfError) as e:
            mf.Plan(triples.Triple("bad", t.p, U, V, W), 1, t.p * 8, host_only=True)
        assert e.value.status == mf.MF_ERR_BAD_TRIPLE


@pytest.mark.parametrize("levels,shards", [(4, 1), (4, 8), (5, 3)])
def test_flattened_plan_beyond_mask_capacity(levels, shards):
    """Flattened plans with more than 576 products (SW^4: 2401, SW^5: 16807)
    plan, report their products and close cleanly (the specialised kernels'
    product mask holds 576 bits; larger plans must not touch it)."""
    t = triples.STRASSEN_WINOGRAD
    n = 2 ** levels * 8
    p = mf.Plan(t, levels, n, host_only=True, shard_count=shards, shard_rank=shards - 1)
    info = p.info()
    assert info["n_products"] == 7 ** levels
    sh = p.products()["shard"]
    assert sh.max() == shards - 1 and (sh >= -1).all()
    p.close()


def test_brent_check_rejects_coefficients_beyond_exact_range():
    """Dyadic coefficients whose scaled products could overflow the exact
    __int128 check are refused (MF_ERR_UNSUPPORTED), not silently wrapped."""
    t = triples.STRASSEN_WINOGRAD
    # each entry passes on its own (|x 2^d| <= 1e6), but a 2^-30 entry scales the
    # whole matrix by 2^30, so 9e5 becomes ~2^50 and U'V'W' ~2^150
    U, V, W = (x * 9e5 for x in (t.U, t.V, t.W))
    for M in (U, V, W):
        M[M == 0] = 2.0 ** -30
    st, msg = _plan_status(2, 7, U, V, W, 1, 64, host_only=1)
    assert st == mf.MF_ERR_UNSUPPORTED and "exact Brent" in msg


def test_loop_comm_handles_and_plan_validation():
    """mf_loop_comm_create hands out one handle per in-process rank; a plan
    with a communicator must shard as rank r of N (host-side checks only)."""
    comms = mf.loop_comm_create(4)
    try:
        assert [mf.comm_info(c) for c in comms] == [
            {"rank": r, "nranks": 4, "kind": "loopback"} for r in range(4)]
        t = triples.STRASSEN_WINOGRAD
        p = mf.Plan(t, 2, 512, host_only=True, comm=comms[2], shard_rank=2, shard_count=4)
        assert (p.products()["shard"] == 2).sum() == 12
        p.close()
        st, msg = _plan_status(2, 7, t.U, t.V, t.W, 2, 512, comm=comms[2].value, shard_rank=1,
                               shard_count=4, host_only=1)
        assert st == mf.MF_ERR_INVALID_ARG and "communicator" in msg
        bogus = (ctypes.c_uint32 * 16)()
        st, msg = _plan_status(2, 7, t.U, t.V, t.W, 1, 64, comm=ctypes.addressof(bogus), host_only=1)
        assert st == mf.MF_ERR_INVALID_ARG and "mf_loop_comm_create" in msg
        with pytest.raises(mf.MfError):
            mf.loop_comm_create(17)
    finally:
        for c in comms:
            mf.comm_destroy(c)
    mf.comm_destroy(None)


@pytest.mark.parametrize("outer,inner", [("strassen-winograd", "laderman"),
                                         ("laderman", "strassen-winograd"),
                                         ("paper-strassen", "strassen-1969")])
def test_triple_kron_abi_matches_oracle(outer, inner):
    """mf_triple_kron (the C caller's way to plan a mixed chain, PAPER.md
    L303-313) equals the oracle's independent or_kron, and the result passes
    mf_plan's exact Brent check."""
    U, V, W = mf.triple_kron(triples.get(outer), triples.get(inner))
    o = oracle.kron(oracle.catalog(outer), oracle.catalog(inner))
    assert (U == o.U).all() and (V == o.V).all() and (W == o.W).all()
    t = triples.kron(triples.get(outer), triples.get(inner))
    p = mf.Plan(t, 1, t.p * 8, host_only=True)
    assert p.info()["n_products"] == t.R
    p.close()
