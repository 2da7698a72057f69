"""TEST INFRASTRUCTURE — ctypes front-ends for the two CPU checkers.

* ``Oracle``    wraps ``oracle/liboracle.so`` (our plain-C restatement,
  ``oracle/blockoa_oracle.c``), built from committed source — available on the
  GPU box too (built there with gcc if the prebuilt .so is missing).
* ``Reference`` wraps ``oracle/_ref/libblockoa_ref.so`` — the UNMODIFIED reference
  core (/root/reference/proj/core) compiled by ``oracle/Makefile`` plus
  ``oracle/ref_shim.cpp``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module. Both classes expose the same methods, so tests can run one case through
either checker. Face kinds follow include/blockoa_b200.h: 0 Dirichlet(a=u0),
1 Robin(a=h, b=u_inf), 2 adiabatic.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libblockoa_ref.so")

_dp = C.POINTER(C.c_double)
_lock = threading.Lock()


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def build_oracle(force: bool = False) -> str:
    """Compile liboracle.so from the committed C source (gcc only)."""
    with _lock:
        if force or not os.path.exists(ORACLE_SO) or (
            os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "blockoa_oracle.c"))
        ):
            subprocess.run(["make", "-C", HERE, "liboracle.so"], check=True,
                           stdout=subprocess.DEVNULL)
    return ORACLE_SO


def build_reference() -> str | None:
    """Compile oracle/_ref from /root/reference when the sources are present."""
    if os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run(["make", "-C", HERE, "ref"], check=True, stdout=subprocess.DEVNULL)
    return REF_SO if os.path.exists(REF_SO) else None


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def _bc_arrays(bc):
    kind = np.array([f[0] for f in bc], dtype=np.int32)
    a = np.array([f[1] for f in bc], dtype=np.float64)
    b = np.array([f[2] for f in bc], dtype=np.float64)
    return kind, a, b


class CheckerError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"status {code}: {msg}")
        self.code = code


class _Op:
    def __init__(self, lib, handle, n, free):
        self.lib, self.handle, self.n, self._free = lib, handle, n, free

    def __del__(self):
        try:
            self._free(self.handle)
        except Exception:
            pass


class _Base:
    prefix = ""

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    # ---- operator -------------------------------------------------------
    def csr(self, op):
        nnz = int(self._f("op_nnz")(op.handle))
        row_ptr = np.empty(op.n + 1, np.int64)
        col = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        g = np.empty(op.n, np.float64)
        vol = np.empty(op.n, np.float64)
        self._f("op_export")(op.handle, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(g), _ptr(vol))
        return row_ptr, col, val, g, vol

    def apply_block(self, op, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = 1 if x.ndim == 1 else x.shape[1]
        y = np.empty_like(x)
        self._f("apply_block")(op.handle, _ptr(x), C.c_int(s), _ptr(y))
        return y

    def _colwise(self, name, op, a):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim == 1:
            a = np.ascontiguousarray(a)
            out = np.empty_like(a)
            self._f(name)(op.handle, _ptr(a), _ptr(out))
            return out
        out = np.empty_like(a)
        for j in range(a.shape[1]):
            col = np.ascontiguousarray(a[:, j])
            res = np.empty_like(col)
            self._f(name)(op.handle, _ptr(col), _ptr(res))
            out[:, j] = res
        return out

    def rhs_from_power(self, op, q):
        """b = V q + g, column by column for an n x s block."""
        return self._colwise("rhs_from_power", op, q)

    def power_from_rhs(self, op, b):
        return self._colwise("power_from_rhs", op, b)

    def relative_residual(self, op, u, q):
        u = np.ascontiguousarray(u, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        f = self._f("relative_residual")
        f.restype = C.c_double
        return float(f(op.handle, _ptr(u), _ptr(q)))

    def field_digest(self, dims, values):
        f = self._f("field_digest")
        f.restype = C.c_uint64
        v = np.ascontiguousarray(values, dtype=np.float64)
        return int(f(C.c_int(dims[0]), C.c_int(dims[1]), C.c_int(dims[2]), _ptr(v)))

    def cg_error_bound(self, kappa, m, e0):
        f = self._f("cg_error_bound")
        f.restype = C.c_double
        st = C.c_int(0)
        v = f(C.c_double(kappa), C.c_int(m), C.c_double(e0), C.byref(st))
        if st.value:
            raise CheckerError(st.value, "cg_error_bound")
        return float(v)


class Oracle(_Base):
    """Plain-C restatement (oracle/blockoa_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path: str | None = None):
        path = path or build_oracle()
        self.lib = C.CDLL(path)
        self.lib.orc_derive_seed.restype = C.c_uint64
        self.lib.orc_op_nnz.restype = C.c_int64

    def assemble(self, grid, k, bc, dz=None):
        nx, ny, nz, lx, ly, lz = grid
        kind, a, b = _bc_arrays(bc)
        k = np.ascontiguousarray(k, dtype=np.float64)
        dzs = None if dz is None else np.ascontiguousarray(dz, dtype=np.float64)
        h = C.c_void_p()
        st = self.lib.orc_assemble(C.c_int(nx), C.c_int(ny), C.c_int(nz), C.c_double(lx),
                                   C.c_double(ly), C.c_double(lz), _ptr(dzs), _ptr(k),
                                   _ptr(kind), _ptr(a), _ptr(b), C.byref(h))
        if st:
            raise CheckerError(st, "orc_assemble")
        return _Op(self.lib, h, nx * ny * nz, self.lib.orc_op_free)

    def op_from_csr(self, row_ptr, col, val):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        n = row_ptr.size - 1
        h = C.c_void_p()
        self.lib.orc_op_from_csr(C.c_int64(n), _ptr(row_ptr), _ptr(col), _ptr(val), C.byref(h))
        return _Op(self.lib, h, n, self.lib.orc_op_free)

    def block_cg(self, op, B, tol=1e-12, max_iter=100000, precond=1):
        B = np.ascontiguousarray(B, dtype=np.float64)
        s = B.shape[1]
        X = np.empty_like(B)
        it = C.c_int(0)
        mv = C.c_int64(0)
        res = np.zeros(s, np.float64)
        conv = np.zeros(s, np.int8)
        st = self.lib.orc_block_cg(op.handle, _ptr(B), C.c_int(s), C.c_double(tol),
                                   C.c_int(max_iter), C.c_int(precond), _ptr(X), C.byref(it),
                                   C.byref(mv), _ptr(res), _ptr(conv))
        if st:
            raise CheckerError(st, "orc_block_cg")
        return X, dict(iterations=it.value, matvec_count=mv.value, final_rel_residual=res,
                       converged=conv.astype(bool))

    def cg(self, op, b, tol=1e-12, max_iter=100000, precond=1):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        it, mv, res, conv = C.c_int(0), C.c_int64(0), C.c_double(0), C.c_char(0)
        st = self.lib.orc_cg(op.handle, _ptr(b), C.c_double(tol), C.c_int(max_iter),
                             C.c_int(precond), _ptr(x), C.byref(it), C.byref(mv),
                             C.byref(res), C.byref(conv))
        if st:
            raise CheckerError(st, "orc_cg")
        return x, dict(iterations=it.value, matvec_count=mv.value,
                       final_rel_residual=res.value, converged=conv.value != b"\x00")

    def combine_action(self, op, X, Cm, j0=0, j1=None, resid=True):
        X = np.ascontiguousarray(X, dtype=np.float64)
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        s, N = Cm.shape
        j1 = N if j1 is None else j1
        m = j1 - j0
        T = np.empty((m, op.n), np.float64)
        Q = np.empty((m, op.n), np.float64)
        R = np.empty(m, np.float64) if resid else None
        st = self.lib.orc_combine_action(op.handle, _ptr(X), C.c_int(s), _ptr(Cm),
                                         C.c_int64(N), C.c_int64(j0), C.c_int64(j1),
                                         _ptr(T), _ptr(Q), _ptr(R))
        if st:
            raise CheckerError(st, "orc_combine_action")
        return T, Q, R

    def derive_seed(self, seed, tag, index=0):
        return int(self.lib.orc_derive_seed(C.c_uint64(seed), tag.encode(), C.c_uint64(index)))

    def rng_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.orc_rng_u64(C.c_uint64(seed), C.c_int64(n), _ptr(out))
        return out

    def rng_uniform(self, seed, lo, hi, n):
        out = np.empty(n, np.float64)
        self.lib.orc_rng_uniform(C.c_uint64(seed), C.c_double(lo), C.c_double(hi),
                                 C.c_int64(n), _ptr(out))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.orc_rng_normal(C.c_uint64(seed), C.c_int64(n), _ptr(out))
        return out

    def rng_below(self, seed, bound, n):
        out = np.empty(n, np.uint64)
        self.lib.orc_rng_below(C.c_uint64(seed), C.c_uint64(bound), C.c_int64(n), _ptr(out))
        return out

    def synth_chip(self, config, nx, ny, nz, s, N, master_seed=1, chip_id=0, fields=True):
        """Seeded BASELINE-config inputs (orc_synth_chip; DESIGN.md §3 pins),
        bitwise the product's host generator (tests/test_oracle.py). Returns a
        ChipCase: grid tuple (nx, ny, nz, lx, ly, lz), dz (or None), bc as
        (kind, a, b) tuples, k [n], q_basis [n, s], coef [s, N]. fields=False
        skips k and q_basis (coefficients and metadata only)."""
        meta = _ChipMeta()
        n = nx * ny * nz
        dz = np.zeros(max(nz, 1), np.float64)
        k = np.empty(n, np.float64) if fields else None
        q = np.empty((n, s), np.float64) if fields else None
        c = np.empty((s, N), np.float64)
        st = self.lib.orc_synth_chip(C.c_int(config), C.c_int(nx), C.c_int(ny), C.c_int(nz),
                                     C.c_int(s), C.c_int64(N), C.c_uint64(master_seed),
                                     C.c_uint64(chip_id), C.byref(meta), _ptr(dz), _ptr(k),
                                     _ptr(q), _ptr(c))
        if st:
            raise CheckerError(st, "orc_synth_chip")
        bc = tuple((int(meta.bc_kind[f]), float(meta.bc_a[f]), float(meta.bc_b[f]))
                   for f in range(6))
        return ChipCase((meta.nx, meta.ny, meta.nz, meta.lx, meta.ly, meta.lz),
                        dz.copy() if meta.has_dz else None, bc, k, q, c)


class _ChipMeta(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("lx", C.c_double),
                ("ly", C.c_double), ("lz", C.c_double), ("has_dz", C.c_int),
                ("bc_kind", C.c_int * 6), ("bc_a", C.c_double * 6), ("bc_b", C.c_double * 6)]


@dataclass
class ChipCase:
    grid: tuple
    dz: object
    bc: tuple
    k: object
    q_basis: object
    coef: object


class Reference(_Base):
    """The unmodified reference core via oracle/ref_shim.cpp."""

    prefix = "ref_"

    def __init__(self, path: str | None = None):
        path = path or REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.lib.ref_derive_seed.restype = C.c_uint64
        self.lib.ref_op_nnz.restype = C.c_longlong
        self.lib.ref_last_error.restype = C.c_char_p

    def _err(self, st, what):
        raise CheckerError(st, f"{what}: {self.lib.ref_last_error().decode()}")

    def assemble(self, grid, k, bc, dz=None):
        if dz is not None:
            raise NotImplementedError("reference GridSpec is uniform (grid.hpp:25-28)")
        nx, ny, nz, lx, ly, lz = grid
        kind, a, b = _bc_arrays(bc)
        k = np.ascontiguousarray(k, dtype=np.float64)
        h = C.c_void_p()
        st = self.lib.ref_op_create(C.c_int(nx), C.c_int(ny), C.c_int(nz), C.c_double(lx),
                                    C.c_double(ly), C.c_double(lz), _ptr(k), _ptr(kind),
                                    _ptr(a), _ptr(b), C.byref(h))
        if st:
            self._err(st, "assemble")
        return _Op(self.lib, h, nx * ny * nz, self.lib.ref_op_free)

    def block_cg(self, op, B, tol=1e-12, max_iter=100000, precond=1):
        B = np.ascontiguousarray(B, dtype=np.float64)
        s = B.shape[1]
        X = np.empty_like(B)
        it, mv, wall = C.c_int(0), C.c_longlong(0), C.c_double(0)
        res = np.zeros(s, np.float64)
        conv = np.zeros(s, np.int8)
        st = self.lib.ref_block_cg(op.handle, _ptr(B), C.c_int(s), C.c_double(tol),
                                   C.c_int(max_iter), C.c_int(precond), _ptr(X), C.byref(it),
                                   C.byref(mv), _ptr(res), _ptr(conv), C.byref(wall))
        if st:
            self._err(st, "block_cg")
        return X, dict(iterations=it.value, matvec_count=mv.value, final_rel_residual=res,
                       converged=conv.astype(bool), wall_time=wall.value)

    def block_cg_csr(self, row_ptr, col, val, B, tol=1e-10, max_iter=100000, precond=0):
        B = np.ascontiguousarray(B, dtype=np.float64)
        n, s = B.shape
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        X = np.empty_like(B)
        it, mv = C.c_int(0), C.c_longlong(0)
        res = np.zeros(s, np.float64)
        conv = np.zeros(s, np.int8)
        st = self.lib.ref_block_cg_csr(C.c_longlong(n), _ptr(row_ptr), _ptr(col), _ptr(val),
                                       _ptr(B), C.c_int(s), C.c_double(tol), C.c_int(max_iter),
                                       C.c_int(precond), _ptr(X), C.byref(it), C.byref(mv),
                                       _ptr(res), _ptr(conv))
        if st:
            self._err(st, "block_cg_csr")
        return X, dict(iterations=it.value, matvec_count=mv.value, final_rel_residual=res,
                       converged=conv.astype(bool))

    def cg(self, op, b, tol=1e-12, max_iter=100000, precond=1):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b)
        it, mv, res, conv = C.c_int(0), C.c_longlong(0), C.c_double(0), C.c_char(0)
        st = self.lib.ref_cg(op.handle, _ptr(b), C.c_double(tol), C.c_int(max_iter),
                             C.c_int(precond), _ptr(x), C.byref(it), C.byref(mv),
                             C.byref(res), C.byref(conv))
        if st:
            self._err(st, "cg")
        return x, dict(iterations=it.value, matvec_count=mv.value,
                       final_rel_residual=res.value, converged=conv.value != b"\x00")

    def cg_csr(self, row_ptr, col, val, b, tol=1e-12, max_iter=100000, precond=0):
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = b.size
        x = np.empty_like(b)
        it, mv, res, conv = C.c_int(0), C.c_longlong(0), C.c_double(0), C.c_char(0)
        st = self.lib.ref_cg_csr(C.c_longlong(n), _ptr(np.ascontiguousarray(row_ptr, np.int64)),
                                 _ptr(np.ascontiguousarray(col, np.int32)),
                                 _ptr(np.ascontiguousarray(val, np.float64)), _ptr(b),
                                 C.c_double(tol), C.c_int(max_iter), C.c_int(precond), _ptr(x),
                                 C.byref(it), C.byref(mv), C.byref(res), C.byref(conv))
        if st:
            self._err(st, "cg_csr")
        return x, dict(iterations=it.value, matvec_count=mv.value,
                       final_rel_residual=res.value, converged=conv.value != b"\x00")

    def combine_action(self, op, X, Cm, threads=1, resid=True):
        X = np.ascontiguousarray(X, dtype=np.float64)
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        s, N = Cm.shape
        T = np.empty((N, op.n), np.float64)
        Q = np.empty((N, op.n), np.float64)
        R = np.empty(N, np.float64) if resid else None
        st = self.lib.ref_combine_action(op.handle, _ptr(X), C.c_int(s), _ptr(Cm),
                                         C.c_longlong(N), _ptr(T), _ptr(Q), _ptr(R),
                                         C.c_int(threads))
        if st:
            self._err(st, "combine_action")
        return T, Q, R

    def basis(self, op, X):
        """A one-group BasisSet holding op and the solved basis X (the state
        generate_blockoa has after generate_basis), for timed per-sample
        combine + operator action calls (RefBasis.combine_action)."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        self.lib.ref_basis_create.restype = C.c_void_p
        h = self.lib.ref_basis_create(op.handle, _ptr(X), C.c_int(X.shape[1]))
        if not h:
            self._err(21, "basis_create")
        return RefBasis(self.lib, C.c_void_p(h), op.n)

    def derive_seed(self, seed, tag, index=0):
        return int(self.lib.ref_derive_seed(C.c_uint64(seed), tag.encode(), C.c_uint64(index)))

    def rng_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_rng_u64(C.c_uint64(seed), C.c_longlong(n), _ptr(out))
        return out

    def rng_uniform(self, seed, lo, hi, n):
        out = np.empty(n, np.float64)
        self.lib.ref_rng_uniform(C.c_uint64(seed), C.c_double(lo), C.c_double(hi),
                                 C.c_longlong(n), _ptr(out))
        return out

    def rng_normal(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.ref_rng_normal(C.c_uint64(seed), C.c_longlong(n), _ptr(out))
        return out

    def rng_below(self, seed, bound, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_rng_below(C.c_uint64(seed), C.c_uint64(bound), C.c_longlong(n), _ptr(out))
        return out

    # ---- dataset I/O (dataset_io.hpp) ----------------------------------------
    # ---- chip model + generate_blockoa on ChipSpec::default_chip() -------------
    def chip_fields(self, grid, n_k, eta, seed):
        """(k [n_k, n], q [n_k * eta, n]) of build_floorplans / rasterize_* as
        generate_basis draws them (chip.cpp:180-306, pipeline.cpp:92-134)."""
        nx, ny, nz = grid
        n = nx * ny * nz
        k = np.empty((n_k, n), np.float64)
        q = np.empty((n_k * eta, n), np.float64)
        st = self.lib.ref_chip_fields(C.c_int(nx), C.c_int(ny), C.c_int(nz), C.c_int(n_k),
                                      C.c_int(eta), C.c_ulonglong(seed), _ptr(k), _ptr(q))
        if st:
            self._err(st, "chip_fields")
        return k, q

    def draw_weights(self, n_basis, seed, n_data):
        w = np.empty((n_data, n_basis), np.float64)
        st = self.lib.ref_draw_weights(C.c_int(n_basis), C.c_ulonglong(seed),
                                       C.c_longlong(n_data), _ptr(w))
        if st:
            self._err(st, "draw_weights")
        return w

    def generate_blockoa(self, grid, n_data, n_basis, n_k, seed, bc, noise=("uniform", -0.01, 0.01),
                         tol=1e-9, max_iter=50000, threads=1):
        """generate_blockoa (pipeline.cpp:365-597) on the default chip: dict of
        k [n_k, n], u / q [n_data, n], residual, floorplan_id, iterations and
        the reference's own basis / total wall seconds."""
        nx, ny, nz = grid
        n = nx * ny * nz
        kind, a, b = _bc_arrays(bc)
        nkind = {"none": 0, "uniform": 1, "gaussian": 2}[noise[0]]
        lo, hi = (noise[1], noise[2]) if nkind == 1 else (0.0, 0.0)
        sigma = noise[1] if nkind == 2 else 0.0
        k = np.empty((n_k, n), np.float64)
        u = np.empty((n_data, n), np.float64)
        q = np.empty((n_data, n), np.float64)
        r = np.empty(n_data, np.float64)
        fp = np.empty(n_data, np.int64)
        it = np.zeros(1, np.int32)
        sec = np.zeros(4, np.float64)
        st = self.lib.ref_generate_blockoa(
            C.c_int(nx), C.c_int(ny), C.c_int(nz), C.c_longlong(n_data), C.c_int(n_basis),
            C.c_int(n_k), C.c_ulonglong(seed), C.c_int(nkind), C.c_double(lo), C.c_double(hi),
            C.c_double(sigma), C.c_double(tol), C.c_int(max_iter), C.c_int(threads), _ptr(kind),
            _ptr(a), _ptr(b), _ptr(k), _ptr(u), _ptr(q), _ptr(r), _ptr(fp), _ptr(it), _ptr(sec))
        if st:
            self._err(st, "generate_blockoa")
        return dict(k=k, u=u, q=q, residual=r, floorplan_id=fp, iterations=int(it[0]),
                    basis_s=float(sec[0]), total_s=float(sec[1]), combine_s=float(sec[2]),
                    action_s=float(sec[3]))

    def write_dataset(self, dir, grid, bc, k, q, u, ids, method="blockoa", master_seed=0,
                      tol_claimed=1e-12, tool_version="blockoa-0.1.0", digests=(),
                      timings=(0.0, 0.0, 0.0, 0.0, 0.0), counters=(0, 0), requested=None,
                      dropped=0, overwrite=False):
        """Reference write_dataset (dataset_io.cpp:160-225) of n_data samples
        given as n_data x n arrays; returns the status code (0 = ok)."""
        nx, ny, nz, lx, ly, lz = grid
        kind, a, b = _bc_arrays(bc)
        k, q, u = (np.ascontiguousarray(x, dtype=np.float64) for x in (k, q, u))
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        did = np.ascontiguousarray([d[0] for d in digests], dtype=np.uint64)
        dig = np.ascontiguousarray([d[1] for d in digests], dtype=np.uint64)
        tim = np.ascontiguousarray(timings, dtype=np.float64)
        cnt = np.ascontiguousarray(counters, dtype=np.int64)
        n_data = ids.size
        return int(self.lib.ref_write_dataset(
            str(dir).encode(), C.c_int(int(overwrite)), C.c_int(nx), C.c_int(ny), C.c_int(nz),
            C.c_double(lx), C.c_double(ly), C.c_double(lz), _ptr(kind), _ptr(a), _ptr(b),
            C.c_longlong(n_data), _ptr(k), _ptr(q), _ptr(u), _ptr(ids), method.encode(),
            C.c_ulonglong(master_seed), C.c_double(tol_claimed), tool_version.encode(),
            C.c_int(did.size), _ptr(did), _ptr(dig), _ptr(tim), _ptr(cnt),
            C.c_longlong(n_data if requested is None else requested), C.c_longlong(dropped)))

    def read_dataset(self, dir):
        """Reference read_dataset: (status, dims, extent, k, q, u, ids)."""
        nd = C.c_longlong(0)
        dims = np.zeros(3, np.int32)
        ext = np.zeros(3, np.float64)
        st = int(self.lib.ref_read_dataset(str(dir).encode(), C.byref(nd), _ptr(dims), _ptr(ext),
                                           None, None, None, None))
        if st:
            return st, None, None, None, None, None, None
        n = int(dims.prod())
        k = np.empty((nd.value, n)); q = np.empty((nd.value, n)); u = np.empty((nd.value, n))
        ids = np.empty(nd.value, np.uint64)
        st = int(self.lib.ref_read_dataset(str(dir).encode(), C.byref(nd), _ptr(dims), _ptr(ext),
                                           _ptr(k), _ptr(q), _ptr(u), _ptr(ids)))
        return st, tuple(int(d) for d in dims), tuple(float(e) for e in ext), k, q, u, ids

    def validate_dataset(self, dir, tol, cap=1 << 20):
        """Reference validate_dataset: (status, pass, fail, max_residual, residuals)."""
        res = np.empty(cap, np.float64)
        n, p, f = C.c_longlong(0), C.c_longlong(0), C.c_longlong(0)
        mx = C.c_double(0)
        st = int(self.lib.ref_validate_dataset(str(dir).encode(), C.c_double(tol), _ptr(res),
                                               C.c_longlong(cap), C.byref(n), C.byref(p),
                                               C.byref(f), C.byref(mx)))
        return st, p.value, f.value, mx.value, res[:n.value].copy()


class RefBasis:
    """Handle of a reference BasisSet (oracle/ref_shim.cpp ref_basis_*)."""

    def __init__(self, lib, handle, n):
        self.lib, self.handle, self.n = lib, handle, n

    def __del__(self):
        try:
            self.lib.ref_basis_free(self.handle)
        except Exception:
            pass

    def combine_action(self, Cm, j0=0, j1=None, threads=1, outputs=True):
        """combine_from_weights + operator_action + relative_residual
        (pipeline.cpp:187-251, discretize.cpp:275-286) for samples [j0, j1) of
        Cm (s x N), parallel_for over `threads` workers as generate_blockoa
        does (pipeline.cpp:410, 511)."""
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        N = Cm.shape[1]
        j1 = N if j1 is None else j1
        m = j1 - j0
        T = np.empty((m, self.n), np.float64) if outputs else None
        Q = np.empty((m, self.n), np.float64) if outputs else None
        R = np.empty(m, np.float64)
        st = self.lib.ref_basis_combine_action(self.handle, _ptr(Cm), C.c_longlong(N),
                                               C.c_longlong(j0), C.c_longlong(j1), _ptr(T),
                                               _ptr(Q), _ptr(R), C.c_int(threads))
        if st:
            raise CheckerError(st, "ref_basis_combine_action")
        return T, Q, R
