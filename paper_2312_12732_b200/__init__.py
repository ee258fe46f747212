"""B200-native Matrix Flow hot path (arXiv 2312.12732): Python binding of libmf.so.

Argument marshalling only: every step of the path (pre-additions K4, batched
leaf DGEMM K5, post-addition K6, NCCL reduction) runs inside libmf.so.  The C
ABI is include/mf.h; the names here mirror it.  PyTorch supplies device
memory, streams and process groups.  There is no fallback: if libmf.so is
missing this import fails.

    import torch, paper_2312_12732_b200 as mf
    plan = mf.Plan(mf.triples.STRASSEN_WINOGRAD, levels=2, n=16384)
    C = plan.dgemm(A, B)              # A, B: cuda float64, row-major
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import triples

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmf.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python tools/build_mf.py` "
                      "(the CUDA path has no fallback)")

_lib = ctypes.CDLL(LIB_PATH)

MF_OK, MF_ERR_INVALID_ARG, MF_ERR_INDIVISIBLE, MF_ERR_BAD_TRIPLE = 0, 1, 2, 3
MF_ERR_OUT_OF_MEMORY, MF_ERR_CUDA, MF_ERR_NCCL, MF_ERR_UNSUPPORTED = 4, 5, 6, 7
STATUS_NAMES = {0: "MF_OK", 1: "MF_ERR_INVALID_ARG", 2: "MF_ERR_INDIVISIBLE",
                3: "MF_ERR_BAD_TRIPLE", 4: "MF_ERR_OUT_OF_MEMORY", 5: "MF_ERR_CUDA",
                6: "MF_ERR_NCCL", 7: "MF_ERR_UNSUPPORTED"}
LEAF_DMMA, LEAF_SIMPLE, LEAF_CUBLAS = 0, 1, 2
IN_ROOT, IN_REPLICATED = 0, 1
OUT_ROOT, OUT_ALL, OUT_ROWSLAB = 0, 1, 2

EXPORTS = ("mf_plan", "mf_dgemm", "mf_dgemm_host", "mf_destroy", "mf_last_error", "mf_plan_info",
           "mf_plan_products", "mf_premix", "mf_leaf", "mf_postmix", "mf_nccl_unique_id",
           "mf_nccl_comm_create", "mf_nccl_comm_destroy", "mf_version", "mf_profile_read",
           "mf_plan_shard_rows", "mf_dgemm_host_async", "mf_host_sync", "mf_jit_compile_check",
           "mf_loop_comm_create", "mf_comm_info", "mf_comm_destroy", "mf_plan_kernels",
           "mf_triple_kron", "mf_plan_exchange")
COMM_NCCL, COMM_LOOPBACK = 0, 1


class mf_options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_int32), ("device", ctypes.c_int32),
                ("leaf", ctypes.c_int32), ("shard_rank", ctypes.c_int32),
                ("shard_count", ctypes.c_int32), ("comm", ctypes.c_void_p),
                ("input_mode", ctypes.c_int32), ("output_mode", ctypes.c_int32),
                ("profile", ctypes.c_int32), ("host_only", ctypes.c_int32),
                ("level_by_level", ctypes.c_int32), ("max_workspace", ctypes.c_int64),
                ("fuse_postadd", ctypes.c_int32), ("graph", ctypes.c_int32),
                ("comm_regions", ctypes.c_int32), ("recurse_levels", ctypes.c_int32)]


_P, _D, _I32, _I64 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int64
_lib.mf_plan.argtypes = [ctypes.POINTER(_P), _I32, _I32, _P, _P, _P, _I32, _I64,
                         ctypes.POINTER(mf_options)]
_lib.mf_dgemm.argtypes = [_P, _D, _P, _I64, _P, _I64, _P, _I64, _P]
_lib.mf_dgemm_host.argtypes = [_P, _D, _P, _I64, _P, _I64, _P, _I64, _P]
_lib.mf_dgemm_host_async.argtypes = [_P, _D, _P, _I64, _P, _I64, _P, _I64, _P]
_lib.mf_host_sync.argtypes = [_P]
_lib.mf_destroy.argtypes = [_P]
_lib.mf_last_error.argtypes = []
_lib.mf_last_error.restype = ctypes.c_char_p
_lib.mf_version.restype = ctypes.c_char_p
_lib.mf_plan_info.argtypes = [_P, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(_I64),
                              ctypes.POINTER(_I64), ctypes.POINTER(_I32), ctypes.POINTER(_I32)]
_lib.mf_plan_products.argtypes = [_P] * 7
_lib.mf_plan_shard_rows.argtypes = [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]
_lib.mf_plan_kernels.argtypes = [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), _P]
_lib.mf_plan_exchange.argtypes = [_P] * 10 + [_I64, ctypes.POINTER(_I64)]
_lib.mf_premix.argtypes = [_P, _I32, _P, _I64, _P, _P]
_lib.mf_leaf.argtypes = [_P, _P, _I64, _P, _I64, _P, _P, _P, _P]
_lib.mf_postmix.argtypes = [_P, _D, _P, _P, _I64, _P]
_lib.mf_profile_read.argtypes = [_P, _P, ctypes.POINTER(_I32), _I32]
_lib.mf_nccl_unique_id.argtypes = [_P]
_lib.mf_nccl_comm_create.argtypes = [ctypes.POINTER(_P), _P, _I32, _I32]
_lib.mf_nccl_comm_destroy.argtypes = [_P]
_lib.mf_loop_comm_create.argtypes = [_I32, ctypes.POINTER(_P)]
_lib.mf_comm_info.argtypes = [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32)]
_lib.mf_comm_destroy.argtypes = [_P]
_lib.mf_triple_kron.argtypes = [_I32, _I32, _P, _P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P]
_lib.mf_jit_compile_check.argtypes = [_P, _I32, _I32, _I32, _I32, ctypes.c_char_p,
                                      ctypes.POINTER(_I32), ctypes.POINTER(_I64)]
for _f in EXPORTS:
    if _f not in ("mf_last_error", "mf_version"):
        getattr(_lib, _f).restype = ctypes.c_int


class MfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(status: int):
    if status != MF_OK:
        raise MfError(status, _lib.mf_last_error().decode())


def triple_kron(outer, inner):
    """mf_triple_kron: the composed triple outer (x) inner (U, V, W arrays of
    ((po*pi)^2, Ro*Ri)), as a C caller plans a mixed chain."""
    po, pi = int(outer.p), int(inner.p)
    Ro, Ri = int(outer.U.shape[1]), int(inner.U.shape[1])
    src = [np.ascontiguousarray(x, dtype=np.float64) for x in
           (outer.U, outer.V, outer.W, inner.U, inner.V, inner.W)]
    out = [np.empty(((po * pi) ** 2, Ro * Ri)) for _ in range(3)]
    _check(_lib.mf_triple_kron(po, Ro, *[x.ctypes.data for x in src[:3]], pi, Ri,
                               *[x.ctypes.data for x in src[3:]], *[x.ctypes.data for x in out]))
    return tuple(out)


def version() -> str:
    return _lib.mf_version().decode()


def jit_compile_check(coef, in_P: int, out_P: int, arch: str = "sm_100a"):
    """mf_jit_compile_check: generate + compile (no GPU) the fused-addition
    kernel of a coefficient table coef[nout][nin]; returns (vw, cubin_bytes)."""
    import numpy as np
    c = np.ascontiguousarray(coef, dtype=np.float64)
    vw, nb = _I32(0), _I64(0)
    _check(_lib.mf_jit_compile_check(c.ctypes.data, c.shape[0], c.shape[1], in_P, out_P,
                                     arch.encode(), ctypes.byref(vw), ctypes.byref(nb)))
    return vw.value, nb.value


def _mat(X, n, name, rows=None):
    """(pointer, leading dimension) of a row-major n x n (or rows x n) float64
    CUDA tensor view."""
    import torch
    rows = n if rows is None else rows
    if not isinstance(X, torch.Tensor) or not X.is_cuda or X.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if X.dim() != 2 or tuple(X.shape) != (rows, n) or X.stride(1) != 1:
        raise ValueError(f"{name} must be a {rows} x {n} row-major view, got "
                         f"shape {tuple(X.shape)} strides {X.stride()}")
    return X.data_ptr(), X.stride(0)


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class Plan:
    """mf_plan / mf_dgemm / mf_destroy for one (triple, levels, n, options)."""

    def __init__(self, triple: triples.Triple | None, levels: int, n: int, *, leaf: str = "dmma",
                 device: int | None = None, shard_rank: int = 0, shard_count: int = 1,
                 comm=None, nccl_comm=None, input_mode: int = IN_REPLICATED,
                 output_mode: int = OUT_ROOT,
                 profile: bool = False, host_only: bool = False, level_by_level: bool = False,
                 max_workspace: int = 0, fuse_postadd: int = 0, recurse_levels: int = 0,
                 graph: bool = False, comm_regions: int = 0):
        self.triple, self.levels, self.n = triple, int(levels), int(n)
        opt = mf_options()
        opt.struct_size = ctypes.sizeof(mf_options)
        opt.device = -1 if device is None else int(device)
        opt.leaf = {"dmma": LEAF_DMMA, "simple": LEAF_SIMPLE, "cublas": LEAF_CUBLAS}[leaf]
        opt.shard_rank, opt.shard_count = int(shard_rank), int(shard_count)
        comm = comm if comm is not None else nccl_comm  # (nccl_comm: the round-1 keyword)
        opt.comm = comm.value if isinstance(comm, ctypes.c_void_p) else comm
        opt.input_mode, opt.output_mode = int(input_mode), int(output_mode)
        opt.profile = int(bool(profile))
        opt.host_only = int(bool(host_only))
        opt.level_by_level = int(bool(level_by_level))
        opt.max_workspace = int(max_workspace)
        opt.fuse_postadd = int(fuse_postadd)  # True / 1: ordered fold; 2: bulk reductions
        opt.recurse_levels = int(recurse_levels)
        opt.graph = int(bool(graph))
        opt.comm_regions = int(comm_regions)
        self._opt = opt
        h = ctypes.c_void_p()
        if triple is None:
            _check(_lib.mf_plan(ctypes.byref(h), 1, 1, None, None, None, self.levels, self.n,
                                ctypes.byref(opt)))
        else:
            U = np.ascontiguousarray(triple.U, dtype=np.float64)
            V = np.ascontiguousarray(triple.V, dtype=np.float64)
            W = np.ascontiguousarray(triple.W, dtype=np.float64)
            self._keep = (U, V, W)
            _check(_lib.mf_plan(ctypes.byref(h), int(triple.p), int(U.shape[1]),
                                U.ctypes.data, V.ctypes.data, W.ctypes.data, self.levels, self.n,
                                ctypes.byref(opt)))
        self._h = h

    # -- queries --------------------------------------------------------------
    def info(self) -> dict:
        ws, m, nprod, na, nb = ctypes.c_size_t(), _I64(), _I64(), _I32(), _I32()
        _check(_lib.mf_plan_info(self._h, ctypes.byref(ws), ctypes.byref(m), ctypes.byref(nprod),
                                 ctypes.byref(na), ctypes.byref(nb)))
        return {"workspace_bytes": ws.value, "leaf_n": m.value, "n_products": nprod.value,
                "n_mat_a": na.value, "n_mat_b": nb.value}

    def products(self) -> dict:
        nprod = self.info()["n_products"]
        arrs = {k: np.zeros(nprod, dtype=np.int32)
                for k in ("a_src", "a_idx", "b_src", "b_idx", "sign", "shard")}
        _check(_lib.mf_plan_products(self._h, *[arrs[k].ctypes.data for k in
                                                ("a_src", "a_idx", "b_src", "b_idx", "sign", "shard")]))
        return arrs

    PHASES = ("premix_a", "premix_b", "leaf", "postmix", "comm")

    def profile_read(self, reset: bool = True) -> dict:
        """Summed device ms per phase over the profiled mf_dgemm calls (mf_profile_read)."""
        ms = (ctypes.c_double * 5)()
        calls = _I32()
        _check(_lib.mf_profile_read(self._h, ms, ctypes.byref(calls), int(reset)))
        out = dict(zip(self.PHASES, list(ms)))
        out["calls"] = calls.value
        return out

    KERNEL_KINDS = ("table", "fixed", "kron", "jit")

    def kernels(self) -> dict:
        """mf_plan_kernels: generated-kernel tables requested / built, and K4/K6
        launches so far by kind (table-driven, compiled-in, Kronecker, generated)."""
        jt, jb = _I32(), _I32()
        launches = (ctypes.c_int64 * 4)()
        _check(_lib.mf_plan_kernels(self._h, ctypes.byref(jt), ctypes.byref(jb), launches))
        return {"jit_tables": jt.value, "jit_built": jb.value,
                "launches": dict(zip(self.KERNEL_KINDS, list(launches)))}

    def exchange(self) -> list:
        """mf_plan_exchange: the collectives one mf_dgemm call of this rank issues, in
        order -- dicts with kind, buf, off, count, root, recv_buf, recv_off, group, phase."""
        n = _I64()
        _check(_lib.mf_plan_exchange(self._h, *([None] * 9), 0, ctypes.byref(n)))
        cols = {k: np.zeros(n.value, dtype=np.int64 if k in ("off", "count", "recv_off") else np.int32)
                for k in ("kind", "buf", "off", "count", "root", "recv_buf", "recv_off", "group", "phase")}
        _check(_lib.mf_plan_exchange(self._h, *[cols[k].ctypes.data for k in
                                                ("kind", "buf", "off", "count", "root", "recv_buf",
                                                 "recv_off", "group", "phase")], n.value, ctypes.byref(n)))
        return [{k: int(v[i]) for k, v in cols.items()} for i in range(n.value)]

    def shard_rows(self) -> tuple:
        """Row slab [r0, r1) this rank computes of each split product (0, 0 if none)."""
        r0, r1 = _I64(), _I64()
        _check(_lib.mf_plan_shard_rows(self._h, ctypes.byref(r0), ctypes.byref(r1)))
        return r0.value, r1.value

    # -- the hot path ------------------------------------------------------------
    def dgemm(self, A, B, C=None, alpha: float = 1.0, stream=None):
        """C <- alpha*A*B on the device (stream-ordered, no host sync)."""
        import torch
        n = self.n
        pa, lda = _mat(A, n, "A") if A is not None else (None, n)
        pb, ldb = _mat(B, n, "B") if B is not None else (None, n)
        rows = self.c_rows()
        if C is None:
            dev = A.device if A is not None else torch.device("cuda")
            C = torch.empty((rows, n), dtype=torch.float64, device=dev)
        pc, ldc = _mat(C, n, "C", rows)
        _check(_lib.mf_dgemm(self._h, float(alpha), pa, lda, pb, ldb, pc, ldc,
                             _stream_ptr(stream)))
        return C

    def c_rows(self) -> int:
        """Rows of this rank's C: n, or n / shard_count with MF_OUT_ROWSLAB."""
        o = self._opt
        if o.output_mode == OUT_ROWSLAB and o.comm and o.shard_count > 1:
            return self.n // o.shard_count
        return self.n

    def dgemm_host(self, A: np.ndarray | None, B: np.ndarray | None, C: np.ndarray | None = None,
                   alpha: float = 1.0, stream=None) -> np.ndarray:
        """The same product on HOST float64 row-major arrays (copies inside the call).
        With IN_ROOT, ranks other than 0 may pass None for A and B."""
        def host(X, name, rows=self.n):
            if X is None:
                return None, self.n
            if X.dtype != np.float64 or X.ndim != 2 or X.shape != (rows, self.n) or \
                    X.strides[1] != 8:
                raise ValueError(f"{name} must be a row-major {rows}x{self.n} float64 array")
            return X.ctypes.data, X.strides[0] // 8
        if C is None:
            C = np.empty((self.c_rows(), self.n))
        pa, lda = host(A, "A"); pb, ldb = host(B, "B"); pc, ldc = host(C, "C", self.c_rows())
        _check(_lib.mf_dgemm_host(self._h, float(alpha), pa, lda, pb, ldb, pc, ldc,
                                  _stream_ptr(stream)))
        return C

    def dgemm_host_ptr(self, pa: int, lda: int, pb: int, ldb: int, pc: int, ldc: int,
                       alpha: float = 1.0, stream=None):
        """mf_dgemm_host on raw host pointers (e.g. pinned torch CPU tensors)."""
        _check(_lib.mf_dgemm_host(self._h, float(alpha), pa, lda, pb, ldb, pc, ldc,
                                  _stream_ptr(stream)))

    def dgemm_host_async_ptr(self, pa: int, lda: int, pb: int, ldb: int, pc: int, ldc: int,
                             alpha: float = 1.0, stream=None):
        """mf_dgemm_host_async on raw host pointers: enqueue, return at once; the
        host buffers must stay untouched (A, B) / unread (C) until host_sync()."""
        _check(_lib.mf_dgemm_host_async(self._h, float(alpha), pa, lda, pb, ldb, pc, ldc,
                                        _stream_ptr(stream)))

    def host_sync(self):
        """mf_host_sync: wait for every enqueued dgemm_host_async call."""
        _check(_lib.mf_host_sync(self._h))

    # -- the steps, for step-by-step parity tests -------------------------------
    def premix(self, side: str, X, out, stream=None):
        import torch
        px, ldx = _mat(X, self.n, side)
        if not out.is_contiguous() or out.dtype != torch.float64:
            raise ValueError("out must be contiguous float64")
        _check(_lib.mf_premix(self._h, 0 if side == "A" else 1, px, ldx, out.data_ptr(),
                              _stream_ptr(stream)))
        return out

    def leaf(self, A, B, T, S, P, stream=None):
        pa, lda = _mat(A, self.n, "A")
        pb, ldb = _mat(B, self.n, "B")
        _check(_lib.mf_leaf(self._h, pa, lda, pb, ldb,
                            T.data_ptr() if T is not None and T.numel() else None,
                            S.data_ptr() if S is not None and S.numel() else None,
                            P.data_ptr(), _stream_ptr(stream)))
        return P

    def postmix(self, P, C, alpha: float = 1.0, stream=None):
        pc, ldc = _mat(C, self.n, "C")
        _check(_lib.mf_postmix(self._h, float(alpha), P.data_ptr(), pc, ldc, _stream_ptr(stream)))
        return C

    # -- lifetime ------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(_lib.mf_destroy(self._h))
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def dgemm(A, B, triple: triples.Triple | str | None = "strassen-winograd", levels: int = 1,
          alpha: float = 1.0, leaf: str = "dmma"):
    """One-shot C = alpha*A*B (plans, runs, destroys; the plan owns scratch memory)."""
    if isinstance(triple, str):
        triple = triples.get(triple)
    with Plan(triple, levels if triple is not None else 0, A.shape[0], leaf=leaf) as p:
        C = p.dgemm(A, B, alpha=alpha)
        import torch
        torch.cuda.current_stream().synchronize()
    return C


# -- NCCL bootstrap (mf_nccl_*) --------------------------------------------------
def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.mf_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_create(uid: bytes, rank: int, nranks: int) -> ctypes.c_void_p:
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    _check(_lib.mf_nccl_comm_create(ctypes.byref(comm), buf, rank, nranks))
    return comm


def nccl_comm_destroy(comm: ctypes.c_void_p):
    _check(_lib.mf_nccl_comm_destroy(comm))


def loop_comm_create(nranks: int) -> list:
    """mf_loop_comm_create: handles for `nranks` ranks run as threads of this
    process (each thread passes its handle as Plan(comm=...))."""
    arr = (_P * int(nranks))()
    _check(_lib.mf_loop_comm_create(int(nranks), arr))
    return [ctypes.c_void_p(arr[i]) for i in range(int(nranks))]


def comm_info(comm) -> dict:
    r, n, k = _I32(), _I32(), _I32()
    _check(_lib.mf_comm_info(comm, ctypes.byref(r), ctypes.byref(n), ctypes.byref(k)))
    return {"rank": r.value, "nranks": n.value,
            "kind": {COMM_NCCL: "nccl", COMM_LOOPBACK: "loopback"}[k.value]}


def comm_destroy(comm):
    _check(_lib.mf_comm_destroy(comm))


__all__ = ["Plan", "dgemm", "MfError", "triples", "version", "nccl_unique_id", "nccl_comm_create",
           "nccl_comm_destroy", "loop_comm_create", "comm_info", "comm_destroy", "EXPORTS",
           "LIB_PATH"]
