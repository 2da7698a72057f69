"""B200-native BlocKOA data-generation hot path (arxiv 2510.23221).

Python mirror of the reference's C++ operator API for the hot path
(/root/reference/proj/core/include/blockoa/*.hpp), bound through ctypes to the
C ABI of ``libblockoa_b200.so`` (include/blockoa_b200.h). Names, argument
meaning and error behaviour follow the reference:

==========================  ==================================================
this module                 reference
==========================  ==================================================
``GridSpec``                ``GridSpec`` grid.hpp:14-53 (+ optional layer dz)
``Dirichlet/Robin/...``     ``FaceCondition`` discretize.hpp:14-24
``BoundarySpec``            ``BoundarySpec`` discretize.hpp:28-38
``assemble``                ``assemble`` discretize.cpp:114-237
``DiscreteOperator.apply_block``  ``CsrMatrix::apply_block`` :75-95
``rhs_from_power``          ``rhs_from_power`` discretize.cpp:246-256
``power_from_rhs``          ``power_from_rhs`` discretize.cpp:258-267
``SolverConfig``            ``SolverConfig`` solvers.hpp:13-21
``block_cg``                ``block_cg`` solvers.cpp:452-665
``combine_action``          ``combine_from_weights`` + ``operator_action``
                            pipeline.cpp:187-251 (+ sample residual :548-571)
``generate_chip``           ``generate_blockoa`` for one basis group
                            pipeline.cpp:365-597
``cg_error_bound``          ``cg_error_bound`` solvers.cpp:672-680
``write_dataset`` ...       dataset_io.hpp (see paper_2510_23221_b200/dataset.py)
exceptions                  errors.hpp:9-71
==========================  ==================================================

Arrays may be numpy (host) or CUDA torch tensors (device, used in place). All
compute runs in the sm_100a kernels of libblockoa_b200.so; there is no CPU
fallback — without the built library or a GPU every call raises.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "GridSpec", "Dirichlet", "Robin", "Adiabatic", "BoundarySpec", "SolverConfig",
    "SolveReport", "BlockCgResult", "PhaseTimings", "DiscreteOperator", "Context",
    "assemble", "operator_from_csr", "block_cg", "combine_action", "generate_chip", "generate_batch", "rhs_from_power",
    "power_from_rhs", "cg_error_bound", "derive_seed", "synth_chip", "synth_chip_device",
    "library_path",
    "Dataset", "DatasetManifest", "DatasetWriter", "ManifestTimings", "ValidationReport",
    "WriteSummary", "field_digest", "read_dataset", "relative_residual", "validate_dataset",
    "write_dataset",
    "Error", "InvalidSpecError", "InvalidConfigError", "DimensionMismatchError",
    "NonPositiveConductivityError", "NonPositiveHtcError", "EmptyBasisError",
    "NotConvergedError", "InvalidKappaError", "IoError", "ExistsError",
    "CorruptManifestError", "SizeMismatchError", "DeviceError",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# BK_LIBRARY: an alternative in-tree build of the same library (A/B timing of
# kernel variants); default the package's own libblockoa_b200.so
LIB_PATH = os.environ.get("BK_LIBRARY") or os.path.join(HERE, "libblockoa_b200.so")


def library_path() -> str:
    return LIB_PATH


# ---------------------------------------------------------------- exceptions
class Error(RuntimeError):
    """Base of everything raised on purpose (blockoa::Error, errors.hpp:9)."""


class InvalidSpecError(Error): ...
class InvalidConfigError(Error): ...
class DimensionMismatchError(Error): ...
class NonPositiveConductivityError(Error): ...
class NonPositiveHtcError(Error): ...
class EmptyBasisError(Error): ...
class NotConvergedError(Error): ...
class InvalidKappaError(Error): ...
class IoError(Error): ...
class ExistsError(IoError): ...
class CorruptManifestError(IoError): ...
class SizeMismatchError(IoError): ...
class DeviceError(Error):
    """CUDA failure, out of device memory, or no usable sm_100 device."""


_STATUS = {
    1: InvalidSpecError, 2: InvalidConfigError, 3: DimensionMismatchError,
    4: NonPositiveConductivityError, 5: NonPositiveHtcError, 6: EmptyBasisError,
    7: NotConvergedError, 8: InvalidKappaError, 9: IoError, 10: ExistsError,
    11: CorruptManifestError, 12: SizeMismatchError, 20: DeviceError, 21: DeviceError,
    22: DeviceError, 99: Error,
}


# ---------------------------------------------------------------- C types
class _Face(C.Structure):
    _fields_ = [("kind", C.c_int), ("a", C.c_double), ("b", C.c_double)]


class _Grid(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("lx", C.c_double),
                ("ly", C.c_double), ("lz", C.c_double), ("dz", C.c_void_p)]


class _Cfg(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int), ("precond", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("matvec_count", C.c_int64), ("wall_time", C.c_double),
                ("final_rel_residual", C.c_void_p), ("converged", C.c_void_p)]


class _Timings(C.Structure):
    _fields_ = [("assemble_s", C.c_double), ("basis_solve_s", C.c_double),
                ("combine_action_s", C.c_double), ("h2d_s", C.c_double), ("d2h_s", C.c_double),
                ("total_s", C.c_double), ("iterations_total", C.c_int64),
                ("matvecs_total", C.c_int64)]


class _Synth(C.Structure):
    _fields_ = [("config", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
                ("s", C.c_int), ("N", C.c_int64), ("master_seed", C.c_uint64),
                ("chip_id", C.c_uint64)]


class _Layer(C.Structure):
    _fields_ = [("z_lo", C.c_double), ("z_hi", C.c_double), ("k", C.c_double), ("role", C.c_int)]


class _Chip(C.Structure):
    _fields_ = [("extent", C.c_double * 3), ("n_layers", C.c_int), ("layers", _Layer * 16),
                ("core_blocks", C.c_int), ("high_power", C.c_int), ("caches_per_layer", C.c_int),
                ("p_high", C.c_double * 2), ("p_normal", C.c_double * 2),
                ("p_cache", C.c_double * 2), ("tsv_count", C.c_int), ("tsv_width", C.c_double),
                ("tsv_k", C.c_double)]


class _GenCfg(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("bc", _Face * 6),
                ("n_data", C.c_int64), ("n_basis", C.c_int), ("n_k", C.c_int),
                ("master_seed", C.c_uint64), ("noise_kind", C.c_int), ("noise_lo", C.c_double),
                ("noise_hi", C.c_double), ("noise_sigma", C.c_double), ("solver", _Cfg),
                ("chip", _Chip)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH)
        vp, dp = C.c_void_p, C.c_void_p
        lib.bk_create.argtypes = [C.c_int, C.POINTER(vp)]
        lib.bk_destroy.argtypes = [vp]
        lib.bk_destroy.restype = None
        lib.bk_last_error.argtypes = [vp]
        lib.bk_last_error.restype = C.c_char_p
        lib.bk_set_stream.argtypes = [vp, vp]
        lib.bk_use_own_stream.argtypes = [vp]
        lib.bk_synchronize.argtypes = [vp]
        lib.bk_launch_count.argtypes = [vp]
        lib.bk_launch_count.restype = C.c_int64
        lib.bk_set_option.argtypes = [vp, C.c_char_p, C.c_int]
        lib.bk_last_solver_variant.argtypes = [vp]
        lib.bk_last_solver_variant.restype = C.c_char_p
        lib.bk_last_solve_phases.argtypes = [vp, vp, vp]
        lib.bk_measure_fp64_peak.argtypes = [vp, C.c_double, C.POINTER(C.c_double),
                                             C.POINTER(C.c_double)]
        lib.bk_assemble.argtypes = [vp, C.POINTER(_Grid), dp, C.POINTER(_Face), C.POINTER(vp)]
        lib.bk_operator_free.argtypes = [vp]
        lib.bk_assemble_into.argtypes = [vp, C.POINTER(_Grid), dp, C.POINTER(_Face), vp]
        lib.bk_operator_free.restype = None
        lib.bk_operator_n.argtypes = [vp]
        lib.bk_operator_n.restype = C.c_int64
        lib.bk_operator_export_csr.argtypes = [vp, vp, dp, dp, dp, C.POINTER(C.c_int64), dp, dp]
        lib.bk_operator_from_csr.argtypes = [vp, C.POINTER(_Grid), dp, dp, dp, dp, dp, C.POINTER(vp)]
        lib.bk_apply_block.argtypes = [vp, vp, dp, C.c_int, dp]
        lib.bk_rhs_from_power.argtypes = [vp, vp, dp, C.c_int, dp]
        lib.bk_power_from_rhs.argtypes = [vp, vp, dp, C.c_int, dp]
        lib.bk_block_cg.argtypes = [vp, vp, dp, C.c_int, C.POINTER(_Cfg), dp, C.POINTER(_Report)]
        lib.bk_combine_action.argtypes = [vp, vp, dp, C.c_int, dp, C.c_int64, dp, dp, dp]
        lib.bk_generate_chip.argtypes = [vp, C.POINTER(_Grid), dp, C.POINTER(_Face), dp, C.c_int,
                                         dp, C.c_int64, C.POINTER(_Cfg), dp, dp, dp,
                                         C.POINTER(_Report), C.POINTER(_Timings)]
        lib.bk_generate_batch.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int, vp, C.c_int64,
                                          C.POINTER(_Cfg), vp, vp, vp, vp, C.c_int,
                                          C.POINTER(_Timings)]
        lib.bk_set_cg_sm_budget.argtypes = [vp, C.c_int]
        lib.bk_generate_stream.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int, vp, C.c_int64,
                                           C.POINTER(_Cfg), C.c_int64, vp, vp, vp,
                                           C.POINTER(_Timings)]
        lib.bk_dd_sizes.argtypes = [vp, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp]
        lib.bk_dd_step.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int,
                                   vp, vp, vp]
        lib.bk_dd_pack.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, C.c_int]
        lib.bk_dd_deferred_x.argtypes = [vp, C.c_int]
        lib.bk_dd_deferred_x.restype = C.c_int
        lib.bk_dd_combine_action.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, vp,
                                             C.c_int64, vp, vp, vp]
        lib.bk_dd_resid_from_nd.argtypes = [vp, vp, C.c_int64, vp]
        lib.bk_cg_error_bound.argtypes = [C.c_double, C.c_int, C.c_double, C.POINTER(C.c_double)]
        lib.bk_derive_seed.argtypes = [C.c_uint64, C.c_char_p, C.c_uint64]
        lib.bk_derive_seed.restype = C.c_uint64
        lib.bk_rng_u64.argtypes = [C.c_uint64, C.c_int64, dp]
        lib.bk_rng_u64.restype = None
        lib.bk_rng_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int64, dp]
        lib.bk_rng_uniform.restype = None
        lib.bk_rng_normal.argtypes = [C.c_uint64, C.c_int64, dp]
        lib.bk_rng_normal.restype = None
        lib.bk_synth_chip.argtypes = [C.POINTER(_Synth), C.POINTER(_Grid), dp, C.POINTER(C.c_int),
                                      C.POINTER(_Face), dp, dp, dp]
        lib.bk_synth_chip_device.argtypes = [vp, C.POINTER(_Synth), C.POINTER(_Grid), dp,
                                             C.POINTER(C.c_int), C.POINTER(_Face), dp, dp, dp]
        lib.bk_field_digest.argtypes = [C.c_int, C.c_int, C.c_int, vp]
        lib.bk_field_digest.restype = C.c_uint64
        lib.bk_dataset_open.argtypes = [C.c_char_p, C.c_int, C.c_int64, vp]
        lib.bk_dataset_append.argtypes = [vp, vp, vp, C.c_int64, vp, vp]
        lib.bk_dataset_commit.argtypes = [vp, C.c_char_p]
        lib.bk_dataset_close.argtypes = [vp]
        lib.bk_dataset_close.restype = None
        lib.bk_dataset_error.argtypes = [vp]
        lib.bk_dataset_error.restype = C.c_char_p
        lib.bk_dataset_count.argtypes = [vp]
        lib.bk_dataset_count.restype = C.c_int64
        lib.bk_dataset_write_seconds.argtypes = [vp]
        lib.bk_dataset_write_seconds.restype = C.c_double
        lib.bk_residuals.argtypes = [vp, vp, vp, vp, C.c_int64, vp]
        lib.bk_validate_samples.argtypes = [vp, C.POINTER(_Grid), C.POINTER(_Face), vp, vp, vp,
                                            C.c_int64, vp, C.c_int, vp, vp, C.c_double, vp, vp]
        lib.bk_abi_version.restype = C.c_int
        lib.bk_default_chip.argtypes = [C.POINTER(_Chip)]
        lib.bk_default_chip.restype = None
        lib.bk_chip_fields.argtypes = [C.POINTER(_Chip), C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_uint64, vp, vp]
        lib.bk_draw_weights.argtypes = [C.c_int, C.c_uint64, C.c_int64, vp]
        lib.bk_generate_blockoa.argtypes = [vp, C.POINTER(_GenCfg), vp, vp, vp, vp, vp, vp, vp]
        _lib = lib
    return _lib


def _raise(st: int, ctx=None, what: str = ""):
    if st == 0:
        return
    msg = what
    if ctx is not None:
        msg = f"{what}: {_load().bk_last_error(ctx).decode()}"
    raise _STATUS.get(st, Error)(msg)


# ---------------------------------------------------------------- arrays
def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _ptr(a):
    """(pointer, keepalive) for a numpy array or a torch tensor (host or CUDA)."""
    if a is None:
        return None, None
    if _is_torch(a):
        if not a.is_contiguous() or str(a.dtype) != "torch.float64":
            raise DimensionMismatchError("tensors must be contiguous float64")
        return C.c_void_p(a.data_ptr()), a
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return arr.ctypes.data_as(C.c_void_p), arr


def _numel(a) -> int:
    return int(a.numel()) if _is_torch(a) else int(np.asarray(a).size)


# ---------------------------------------------------------------- reference types
@dataclass
class GridSpec:
    """Uniform cell-centred grid (grid.hpp:14-53); ``dz`` optionally gives the
    nz layer thicknesses of a non-uniform stack (BASELINE config 4)."""
    nx: int = 1
    ny: int = 1
    nz: int = 1
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0
    dz: Optional[Sequence[float]] = None

    def cell_count(self) -> int:
        return self.nx * self.ny * self.nz

    def flat(self, ix: int, iy: int, iz: int) -> int:
        return ix + self.nx * (iy + self.ny * iz)

    def _c(self):
        g = _Grid(self.nx, self.ny, self.nz, self.lx, self.ly, self.lz, None)
        keep = None
        if self.dz is not None:
            keep = np.ascontiguousarray(self.dz, dtype=np.float64)
            if keep.size != self.nz:
                raise DimensionMismatchError("grid: dz must have nz entries")
            g.dz = keep.ctypes.data_as(C.c_void_p)
        return g, keep


@dataclass(frozen=True)
class Dirichlet:
    u0: float = 0.0


@dataclass(frozen=True)
class Robin:
    h: float = 0.0
    u_inf: float = 0.0


@dataclass(frozen=True)
class Adiabatic:
    """Zero-flux face (the reference expresses it as Robin{1e-300, 0})."""


@dataclass
class BoundarySpec:
    """Face order x-, x+, y-, y+, z-, z+ (discretize.hpp:26)."""
    faces: list = field(default_factory=lambda: [Dirichlet()] * 6)

    @staticmethod
    def uniform_dirichlet(u0: float) -> "BoundarySpec":
        return BoundarySpec([Dirichlet(u0)] * 6)

    @staticmethod
    def uniform_robin(h: float, u_inf: float) -> "BoundarySpec":
        return BoundarySpec([Robin(h, u_inf)] * 6)

    @staticmethod
    def mixed(h: float, u_inf: float, side_u0: float) -> "BoundarySpec":
        return BoundarySpec([Dirichlet(side_u0)] * 4 + [Robin(h, u_inf)] * 2)

    def _c(self):
        arr = (_Face * 6)()
        for i, f in enumerate(self.faces):
            if isinstance(f, Dirichlet):
                arr[i] = _Face(0, f.u0, 0.0)
            elif isinstance(f, Robin):
                arr[i] = _Face(1, f.h, f.u_inf)
            elif isinstance(f, Adiabatic):
                arr[i] = _Face(2, 0.0, 0.0)
            else:
                raise InvalidSpecError(f"unknown face condition {f!r}")
        return arr

    def as_tuples(self):
        """(kind, a, b) per face — the form the CPU checkers take."""
        out = []
        for f in self.faces:
            if isinstance(f, Dirichlet):
                out.append((0, f.u0, 0.0))
            elif isinstance(f, Robin):
                out.append((1, f.h, f.u_inf))
            else:
                out.append((2, 0.0, 0.0))
        return out


@dataclass
class SolverConfig:
    rel_tol: float = 1e-9
    max_iter: int = 10000
    preconditioner: str = "none"  # "none" | "jacobi"

    def _c(self):
        if self.preconditioner not in ("none", "jacobi"):
            raise InvalidConfigError("solver: preconditioner must be none|jacobi")
        return _Cfg(self.rel_tol, self.max_iter, 1 if self.preconditioner == "jacobi" else 0)


@dataclass
class SolveReport:
    iterations: int
    final_rel_residual: np.ndarray
    converged: np.ndarray
    wall_time: float
    matvec_count: int

    def all_converged(self) -> bool:
        return bool(np.all(self.converged))


@dataclass
class BlockCgResult:
    x: object
    report: SolveReport


@dataclass
class PhaseTimings:
    assemble_s: float
    basis_solve_s: float
    combine_action_s: float
    h2d_s: float
    d2h_s: float
    total_s: float
    iterations_total: int
    matvecs_total: int


# ---------------------------------------------------------------- context
class Context:
    """One per (thread, GPU): stream + device workspace (bk_ctx)."""

    def __init__(self, device: int = 0):
        lib = _load()
        h = C.c_void_p()
        st = lib.bk_create(device, C.byref(h))
        if st:
            _raise(st, None, f"bk_create(device={device}): no usable sm_100 GPU")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            _load().bk_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: Optional[int]):
        """Launch on a cudaStream_t handle (0 = legacy default stream, e.g.
        torch.cuda.current_stream().cuda_stream); None = the context's own stream."""
        if stream_ptr is None:
            _raise(_load().bk_use_own_stream(self.h), self.h, "use_own_stream")
        else:
            _raise(_load().bk_set_stream(self.h, C.c_void_p(stream_ptr)), self.h, "set_stream")

    def synchronize(self):
        _raise(_load().bk_synchronize(self.h), self.h, "synchronize")

    @property
    def launch_count(self) -> int:
        return int(_load().bk_launch_count(self.h))

    @property
    def last_solver_variant(self) -> str:
        """Kernel instantiation of the last block-CG solve on this context."""
        return _load().bk_last_solver_variant(self.h).decode()

    def last_solve_phases(self) -> dict:
        """Per-sweep-kind device ms and launch counts of the last multi-kernel
        solve (needs option phase_timing = 1)."""
        ms = np.zeros(4, np.float64)
        cnt = np.zeros(4, np.int64)
        _raise(_load().bk_last_solve_phases(self.h, ms.ctypes.data_as(C.c_void_p),
                                            cnt.ctypes.data_as(C.c_void_p)), self.h, "phases")
        names = ("spmm", "update", "pupdate", "other")
        return {nm: {"ms": float(ms[i]), "launches": int(cnt[i])} for i, nm in enumerate(names)}

    def measure_fp64_peak(self, seconds: float = 4.0) -> tuple:
        """(burst, sustained) FP64 tensor-core TFLOP/s of this GPU
        (bk_measure_fp64_peak): best of 10 short launches, and launches back
        to back for `seconds` (the rate at the board's power limit)."""
        b, s = C.c_double(0.0), C.c_double(0.0)
        _raise(_load().bk_measure_fp64_peak(self.h, float(seconds), C.byref(b), C.byref(s)),
               self.h, "measure_fp64_peak")
        return float(b.value), float(s.value)

    def set_option(self, name: str, value: int) -> None:
        """Per-context kernel-variant switch (bk_set_option): "ring" (-1 auto,
        0, 1), "no_resident", "force_large", "cg_profile", "no_tma_spmm",
        "comb_profile", "batch_trace", "phase_timing", "no_ws_update",
        "no_ws_spmm", "no_defer_x", "no_w_prefetch", "comb_one_role",
        "graph_loop", "spmm_band", "spmm_teams" (A/B and test pins; see
        include/blockoa_b200.h)."""
        _raise(_load().bk_set_option(self.h, name.encode(), int(value)), self.h, "set_option")

    @contextlib.contextmanager
    def options(self, **kv):
        """Temporarily set kernel-variant switches (restored to 0 / auto)."""
        for k, v in kv.items():
            self.set_option(k, v)
        try:
            yield self
        finally:
            for k in kv:
                self.set_option(k, -1 if k == "ring" else 0)


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# ---------------------------------------------------------------- operator
class DiscreteOperator:
    """Device-resident matrix-free stencil (DiscreteOperator, discretize.hpp:62-69)."""

    def __init__(self, handle, ctx: Context, grid: GridSpec, boundary: BoundarySpec):
        self.h = handle
        self.ctx = ctx
        self.grid = grid
        self.boundary = boundary
        self.n = grid.cell_count()

    def __del__(self):
        try:
            if self.h:
                _load().bk_operator_free(self.h)
        except Exception:
            pass

    def csr(self):
        """(row_ptr int64[n+1], col int32[nnz], val, g, volumes) in the reference CSR order."""
        lib = _load()
        nnz = C.c_int64(0)
        row_ptr = np.empty(self.n + 1, np.int64)
        _raise(lib.bk_operator_export_csr(self.ctx.h, self.h, row_ptr.ctypes.data_as(C.c_void_p),
                                          None, None, C.byref(nnz), None, None), self.ctx.h, "csr")
        col = np.empty(nnz.value, np.int32)
        val = np.empty(nnz.value, np.float64)
        g = np.empty(self.n, np.float64)
        vol = np.empty(self.n, np.float64)
        _raise(lib.bk_operator_export_csr(
            self.ctx.h, self.h, row_ptr.ctypes.data_as(C.c_void_p), col.ctypes.data_as(C.c_void_p),
            val.ctypes.data_as(C.c_void_p), C.byref(nnz), g.ctypes.data_as(C.c_void_p),
            vol.ctypes.data_as(C.c_void_p)), self.ctx.h, "csr")
        return row_ptr, col, val, g, vol

    def apply_block(self, x, out=None):
        """Y = A X for an n x s block (or a length-n vector)."""
        s = 1 if len(x.shape) == 1 else int(x.shape[1])
        if int(x.shape[0]) != self.n:
            raise DimensionMismatchError("apply_block: rows != n")
        px, kx = _ptr(x)
        if out is None:
            out = np.empty(tuple(x.shape), np.float64)
        py, ky = _ptr(out)
        _raise(_load().bk_apply_block(self.ctx.h, self.h, px, s, py), self.ctx.h, "apply_block")
        return out


def assemble(k, grid: GridSpec, bc: BoundarySpec, ctx: Optional[Context] = None,
             out: Optional[DiscreteOperator] = None) -> DiscreteOperator:
    """assemble(k, grid, bc) (discretize.cpp:114-237) -> device stencil. With
    `out` (an operator of this context), re-assembles into its device buffers
    (reused when the cell count matches) and returns it."""
    ctx = _ctx(ctx)
    if _numel(k) != grid.cell_count():
        raise DimensionMismatchError("assemble: conductivity grid mismatch")
    g, keep = grid._c()
    faces = bc._c()
    pk, kk = _ptr(k)
    if out is not None:
        if out.ctx is not ctx:
            raise InvalidConfigError("assemble: out belongs to another context")
        _raise(_load().bk_assemble_into(ctx.h, C.byref(g), pk, faces, out.h), ctx.h, "assemble")
        out.grid, out.boundary, out.n = grid, bc, grid.cell_count()
        return out
    h = C.c_void_p()
    _raise(_load().bk_assemble(ctx.h, C.byref(g), pk, faces, C.byref(h)), ctx.h, "assemble")
    return DiscreteOperator(h, ctx, grid, bc)


def operator_from_csr(grid: GridSpec, row_ptr, col, val, g=None, volumes=None,
                      ctx: Optional[Context] = None,
                      boundary: Optional["BoundarySpec"] = None) -> DiscreteOperator:
    """Device stencil from the reference's assembled CSR (DiscreteOperator{A, g,
    volumes}, discretize.hpp:62-69): the drop-in for block_cg(const CsrMatrix&).
    Raises InvalidSpecError unless A is a symmetric 7-point stencil on `grid`
    with volumes uniform per z-layer."""
    ctx = _ctx(ctx)
    n = grid.cell_count()
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float64)
    if row_ptr.shape != (n + 1,) or col.shape != val.shape or int(row_ptr[-1]) != col.size:
        raise DimensionMismatchError("operator_from_csr: CSR shape does not match the grid")
    gg = None if g is None else np.ascontiguousarray(g, dtype=np.float64)
    vv = None if volumes is None else np.ascontiguousarray(volumes, dtype=np.float64)
    for a in (gg, vv):
        if a is not None and a.shape != (n,):
            raise DimensionMismatchError("operator_from_csr: g / volumes must have n entries")
    gr, keep = grid._c()
    h = C.c_void_p()
    ptr = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _raise(_load().bk_operator_from_csr(ctx.h, C.byref(gr), ptr(row_ptr), ptr(col), ptr(val),
                                        ptr(gg), ptr(vv), C.byref(h)), ctx.h, "operator_from_csr")
    return DiscreteOperator(h, ctx, grid, boundary)


def _cols(a) -> int:
    return 1 if len(a.shape) == 1 else int(a.shape[1])


def rhs_from_power(op: DiscreteOperator, q, out=None):
    """b = V q + g (column-wise for an n x s block)."""
    if int(q.shape[0]) != op.n:
        raise DimensionMismatchError("rhs_from_power: power grid mismatch")
    pq, kq = _ptr(q)
    out = np.empty(tuple(q.shape), np.float64) if out is None else out
    pb, kb = _ptr(out)
    _raise(_load().bk_rhs_from_power(op.ctx.h, op.h, pq, _cols(q), pb), op.ctx.h, "rhs_from_power")
    return out


def power_from_rhs(op: DiscreteOperator, b, out=None):
    """q = (b - g) / V."""
    if int(b.shape[0]) != op.n:
        raise DimensionMismatchError("power_from_rhs: vector length != n")
    pb, kb = _ptr(b)
    out = np.empty(tuple(b.shape), np.float64) if out is None else out
    pq, kq = _ptr(out)
    _raise(_load().bk_power_from_rhs(op.ctx.h, op.h, pb, _cols(b), pq), op.ctx.h, "power_from_rhs")
    return out


def _report(s, rep_c, res, conv) -> SolveReport:
    return SolveReport(iterations=rep_c.iterations, final_rel_residual=res,
                       converged=conv.astype(bool), wall_time=rep_c.wall_time,
                       matvec_count=rep_c.matvec_count)


def block_cg(op: DiscreteOperator, b, cfg: SolverConfig, out=None) -> BlockCgResult:
    """block_cg(op, B, cfg) (solvers.cpp:452-665) on the device."""
    cfg_c = cfg._c()
    if len(b.shape) != 2:
        raise DimensionMismatchError("block_cg: B must be n x s")
    if int(b.shape[0]) != op.n:
        raise DimensionMismatchError("block_cg: rhs rows != n")
    s = int(b.shape[1])
    pb, kb = _ptr(b)
    out = np.empty((op.n, s), np.float64) if out is None else out
    px, kx = _ptr(out)
    res = np.zeros(max(s, 1), np.float64)
    conv = np.zeros(max(s, 1), np.int8)
    rep = _Report(0, 0, 0.0, res.ctypes.data_as(C.c_void_p), conv.ctypes.data_as(C.c_void_p))
    _raise(_load().bk_block_cg(op.ctx.h, op.h, pb, s, C.byref(cfg_c), px, C.byref(rep)),
           op.ctx.h, "block_cg")
    return BlockCgResult(out, _report(s, rep, res[:s], conv[:s]))


def combine_action(op: DiscreteOperator, x, coef, t_out=None, q_out=None, resid_out=None,
                   want=("T", "Q", "resid")):
    """Fused combine_from_weights + operator_action for N samples.

    x: n x s basis solutions; coef: s x N weights (column j = sample j).
    Returns (T [N x n], Q [N x n], resid [N]).
    """
    s = _cols(x)
    if int(x.shape[0]) != op.n:
        raise DimensionMismatchError("operator_action: vector length != n")
    if int(coef.shape[0]) != s:
        raise DimensionMismatchError("combine: weight count != basis size")
    N = int(coef.shape[1])
    if t_out is None and "T" in want:
        t_out = np.empty((N, op.n), np.float64)
    if q_out is None and "Q" in want:
        q_out = np.empty((N, op.n), np.float64)
    if resid_out is None and "resid" in want:
        resid_out = np.empty(N, np.float64)
    px, kx = _ptr(x)
    pc, kc = _ptr(coef)
    pt, kt = _ptr(t_out)
    pq, kq = _ptr(q_out)
    pr, kr = _ptr(resid_out)
    _raise(_load().bk_combine_action(op.ctx.h, op.h, px, s, pc, N, pt, pq, pr), op.ctx.h,
           "combine_action")
    return t_out, q_out, resid_out


def generate_chip(grid: GridSpec, k, bc: BoundarySpec, q_basis, coef, cfg: SolverConfig,
                  t_out=None, q_out=None, resid_out=None, ctx: Optional[Context] = None,
                  check_converged: bool = True):
    """Whole per-chip pipeline: assemble -> B = V q + g -> block CG -> fused
    combine + operator action. Returns (T, Q, resid, SolveReport, PhaseTimings)."""
    ctx = _ctx(ctx)
    n = grid.cell_count()
    s = _cols(q_basis)
    N = int(coef.shape[1])
    if int(coef.shape[0]) != s:
        raise DimensionMismatchError("combine: weight count != basis size")
    if _numel(k) != n or int(q_basis.shape[0]) != n:
        raise DimensionMismatchError("generate: field length does not match grid")
    g, keep = grid._c()
    faces = bc._c()
    cfg_c = cfg._c()
    t_out = np.empty((N, n), np.float64) if t_out is None else t_out
    q_out = np.empty((N, n), np.float64) if q_out is None else q_out
    resid_out = np.empty(N, np.float64) if resid_out is None else resid_out
    ptrs = [_ptr(a) for a in (k, q_basis, coef, t_out, q_out, resid_out)]
    res = np.zeros(s, np.float64)
    conv = np.zeros(s, np.int8)
    rep = _Report(0, 0, 0.0, res.ctypes.data_as(C.c_void_p), conv.ctypes.data_as(C.c_void_p))
    tim = _Timings()
    st = _load().bk_generate_chip(ctx.h, C.byref(g), ptrs[0][0], faces, ptrs[1][0], s, ptrs[2][0],
                                  N, C.byref(cfg_c), ptrs[3][0], ptrs[4][0], ptrs[5][0],
                                  C.byref(rep), C.byref(tim))
    if st == 7 and not check_converged:
        st = 0
    _raise(st, ctx.h, "generate_chip")
    timings = PhaseTimings(tim.assemble_s, tim.basis_solve_s, tim.combine_action_s, tim.h2d_s,
                           tim.d2h_s, tim.total_s, tim.iterations_total, tim.matvecs_total)
    return t_out, q_out, resid_out, _report(s, rep, res, conv), timings


def generate_batch(chips, cfg: SolverConfig, t_out=None, q_out=None, resid_out=None,
                   streams: int = 8, ctx: Optional[Context] = None, check_converged: bool = True):
    """Batched per-chip pipeline (bk_generate_batch): `chips` is a list of
    ChipInputs (or objects with grid, bc, k, q_basis, coef) sharing s and N.
    streams = K > 1 with identical dims and device outputs: groups of K chips
    are solved by one cooperative launch (chip k on 1/K of the SMs); otherwise
    chips run one after another. Returns (T list, Q list, resid list,
    [SolveReport], PhaseTimings)."""
    ctx = _ctx(ctx)
    n = len(chips)
    if n == 0:
        return [], [], [], [], None
    s = _cols(chips[0].q_basis)
    N = int(chips[0].coef.shape[1])
    grids = (_Grid * n)()
    faces = (_Face * (6 * n))()
    keep = []
    for c, ch in enumerate(chips):
        g, kd = ch.grid._c()
        keep.append(kd)
        grids[c] = g
        fc = ch.bc._c()
        for f in range(6):
            faces[6 * c + f] = fc[f]
        if _cols(ch.q_basis) != s or int(ch.coef.shape[1]) != N:
            raise DimensionMismatchError("generate_batch: chips must share s and N")
    def ptr_array(arrs):
        out = (C.c_void_p * n)()
        for i, a in enumerate(arrs):
            p, kk = _ptr(a)
            keep.append(kk)
            out[i] = p.value if p is not None else None
        return out
    if t_out is None:
        t_out = [np.empty((N, ch.grid.cell_count())) for ch in chips]
    if q_out is None:
        q_out = [np.empty((N, ch.grid.cell_count())) for ch in chips]
    if resid_out is None:
        resid_out = [np.empty(N) for _ in chips]
    kp = ptr_array([ch.k for ch in chips])
    qp = ptr_array([ch.q_basis for ch in chips])
    cp = ptr_array([ch.coef for ch in chips])
    tp = ptr_array(t_out)
    qo = ptr_array(q_out)
    rp = ptr_array(resid_out)
    res = [np.zeros(s) for _ in chips]
    conv = [np.zeros(s, np.int8) for _ in chips]
    reps = (_Report * n)()
    for c in range(n):
        reps[c] = _Report(0, 0, 0.0, res[c].ctypes.data_as(C.c_void_p),
                          conv[c].ctypes.data_as(C.c_void_p))
    cfg_c = cfg._c()
    tim = _Timings()
    st = _load().bk_generate_batch(ctx.h, n, C.cast(grids, C.c_void_p), C.cast(kp, C.c_void_p),
                                   C.cast(faces, C.c_void_p), C.cast(qp, C.c_void_p), s,
                                   C.cast(cp, C.c_void_p), N, C.byref(cfg_c),
                                   C.cast(tp, C.c_void_p), C.cast(qo, C.c_void_p),
                                   C.cast(rp, C.c_void_p), C.cast(reps, C.c_void_p), streams,
                                   C.byref(tim))
    if st == 7 and not check_converged:
        st = 0
    _raise(st, ctx.h, "generate_batch")
    reports = [_report(s, reps[c], res[c], conv[c]) for c in range(n)]
    timings = PhaseTimings(tim.assemble_s, tim.basis_solve_s, tim.combine_action_s, tim.h2d_s,
                           tim.d2h_s, tim.total_s, tim.iterations_total, tim.matvecs_total)
    return t_out, q_out, resid_out, reports, timings


_SINK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                    C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double))


def generate_stream(chips, cfg: SolverConfig, sink=None, chunk: int = 0,
                    ctx: Optional[Context] = None, check_converged: bool = True):
    """Streaming per-chip pipeline (bk_generate_stream) for jobs whose outputs
    do not fit in memory: chips solved one after another, each chip's samples
    combined in chunks, copied to pinned host memory and handed to
    sink(chip, j0, T, Q, resid) (numpy views of m x n / m values, valid only
    during the call; return True to abort) from a library thread while the
    next chip solves. sink=None still copies every sample to host memory.
    Returns ([SolveReport], PhaseTimings)."""
    ctx = _ctx(ctx)
    n = len(chips)
    if n == 0:
        return [], None
    s = _cols(chips[0].q_basis)
    N = int(chips[0].coef.shape[1])
    grids = (_Grid * n)()
    faces = (_Face * (6 * n))()
    keep = []
    for c, ch in enumerate(chips):
        g, kd = ch.grid._c()
        keep.append(kd)
        grids[c] = g
        fc = ch.bc._c()
        for f in range(6):
            faces[6 * c + f] = fc[f]
        if _cols(ch.q_basis) != s or int(ch.coef.shape[1]) != N:
            raise DimensionMismatchError("generate_stream: chips must share s and N")

    def ptr_array(arrs):
        out = (C.c_void_p * n)()
        for i, a in enumerate(arrs):
            p, kk = _ptr(a)
            keep.append(kk)
            out[i] = p.value if p is not None else None
        return out

    kp = ptr_array([ch.k for ch in chips])
    qp = ptr_array([ch.q_basis for ch in chips])
    cp = ptr_array([ch.coef for ch in chips])
    res = [np.zeros(s) for _ in chips]
    conv = [np.zeros(s, np.int8) for _ in chips]
    reps = (_Report * n)()
    for c in range(n):
        reps[c] = _Report(0, 0, 0.0, res[c].ctypes.data_as(C.c_void_p),
                          conv[c].ctypes.data_as(C.c_void_p))
    errors = []

    def _cb(user, chip, j0, m, ncell, T, Q, R):
        try:
            tv = np.ctypeslib.as_array(T, shape=(int(m), int(ncell)))
            qv = np.ctypeslib.as_array(Q, shape=(int(m), int(ncell)))
            rv = np.ctypeslib.as_array(R, shape=(int(m),))
            return 1 if sink(int(chip), int(j0), tv, qv, rv) else 0
        except Exception as e:  # surfaced after the call
            errors.append(e)
            return 1

    cb = _SINK(_cb) if sink is not None else C.cast(None, _SINK)
    cfg_c = cfg._c()
    tim = _Timings()
    st = _load().bk_generate_stream(ctx.h, n, C.cast(grids, C.c_void_p), C.cast(kp, C.c_void_p),
                                    C.cast(faces, C.c_void_p), C.cast(qp, C.c_void_p), s,
                                    C.cast(cp, C.c_void_p), N, C.byref(cfg_c), int(chunk),
                                    C.cast(cb, C.c_void_p), None, C.cast(reps, C.c_void_p),
                                    C.byref(tim))
    if errors:
        raise errors[0]
    if st == 7 and not check_converged:
        st = 0
    _raise(st, ctx.h, "generate_stream")
    reports = [_report(s, reps[c], res[c], conv[c]) for c in range(n)]
    timings = PhaseTimings(tim.assemble_s, tim.basis_solve_s, tim.combine_action_s, tim.h2d_s,
                           tim.d2h_s, tim.total_s, tim.iterations_total, tim.matvecs_total)
    return reports, timings


def set_cg_sm_budget(ctx: Context, max_ctas: int) -> None:
    _raise(_load().bk_set_cg_sm_budget(ctx.h, max_ctas), ctx.h, "set_cg_sm_budget")


def cg_error_bound(kappa: float, m: int, e0: float) -> float:
    out = C.c_double(0)
    _raise(_load().bk_cg_error_bound(kappa, m, e0, C.byref(out)), None, "cg_error_bound")
    return out.value


def derive_seed(seed: int, tag: str, index: int = 0) -> int:
    return int(_load().bk_derive_seed(seed, tag.encode(), index))


def rng_u64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    _load().bk_rng_u64(seed, n, out.ctypes.data_as(C.c_void_p))
    return out


def rng_uniform(seed: int, lo: float, hi: float, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _load().bk_rng_uniform(seed, lo, hi, n, out.ctypes.data_as(C.c_void_p))
    return out


def rng_normal(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _load().bk_rng_normal(seed, n, out.ctypes.data_as(C.c_void_p))
    return out


@dataclass
class ChipInputs:
    grid: GridSpec
    bc: BoundarySpec
    k: np.ndarray        # n
    q_basis: np.ndarray  # n x s
    coef: np.ndarray     # s x N


def synth_chip(config: int, nx: int, ny: int, nz: int, s: int, N: int, master_seed: int = 1,
               chip_id: int = 0) -> ChipInputs:
    """Seeded synthetic inputs of BASELINE config 1..5."""
    lib = _load()
    sp = _Synth(config, nx, ny, nz, s, N, master_seed, chip_id)
    g = _Grid()
    dz = np.zeros(nz, np.float64)
    has_dz = C.c_int(0)
    faces = (_Face * 6)()
    n = nx * ny * nz
    k = np.empty(n, np.float64)
    q = np.empty((n, s), np.float64)
    c = np.empty((s, N), np.float64)
    st = lib.bk_synth_chip(C.byref(sp), C.byref(g), dz.ctypes.data_as(C.c_void_p),
                           C.byref(has_dz), faces, k.ctypes.data_as(C.c_void_p),
                           q.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p))
    _raise(st, None, "synth_chip")
    grid = GridSpec(g.nx, g.ny, g.nz, g.lx, g.ly, g.lz, dz.copy() if has_dz.value else None)
    fl = []
    for f in faces:
        fl.append(Dirichlet(f.a) if f.kind == 0 else Robin(f.a, f.b) if f.kind == 1 else Adiabatic())
    return ChipInputs(grid, BoundarySpec(fl), k, q, c)


def synth_chip_device(config: int, nx: int, ny: int, nz: int, s: int, N: int,
                      master_seed: int = 1, chip_id: int = 0,
                      ctx: Optional[Context] = None) -> ChipInputs:
    """synth_chip with the fields evaluated on the GPU: the same
    random draws (host), k and q_basis as CUDA torch tensors written by device
    kernels, coef as a CUDA tensor. k of configs 1, 2, 4 and coef are bitwise
    synth_chip's; the maps agree to a few ulp (CUDA exp vs host libm)."""
    import torch

    ctx = _ctx(ctx)
    lib = _load()
    sp = _Synth(config, nx, ny, nz, s, N, master_seed, chip_id)
    g = _Grid()
    dz = np.zeros(nz, np.float64)
    has_dz = C.c_int(0)
    faces = (_Face * 6)()
    dev = torch.device("cuda", ctx.device)
    n = nx * ny * nz
    k = torch.empty(n, dtype=torch.float64, device=dev)
    q = torch.empty((n, s), dtype=torch.float64, device=dev)
    c = torch.empty((s, N), dtype=torch.float64, device=dev)
    st = lib.bk_synth_chip_device(ctx.h, C.byref(sp), C.byref(g), dz.ctypes.data_as(C.c_void_p),
                                  C.byref(has_dz), faces, C.c_void_p(k.data_ptr()),
                                  C.c_void_p(q.data_ptr()), C.c_void_p(c.data_ptr()))
    _raise(st, ctx.h, "synth_chip_device")
    grid = GridSpec(g.nx, g.ny, g.nz, g.lx, g.ly, g.lz, dz.copy() if has_dz.value else None)
    fl = [Dirichlet(f.a) if f.kind == 0 else Robin(f.a, f.b) if f.kind == 1 else Adiabatic()
          for f in faces]
    return ChipInputs(grid, BoundarySpec(fl), k, q, c)


# BASELINE.json configs (shapes): (config id, nx, ny, nz, s, N)
CONFIGS = {
    1: (1, 64, 64, 1, 8, 256),
    2: (2, 256, 256, 1, 16, 2048),
    3: (3, 128, 128, 8, 32, 5000),
    4: (4, 128, 128, 4, 16, 8),      # per chip; 5000 chips
    5: (5, 512, 512, 16, 64, 5000),
}
C4_CHIPS = 5000


# dataset sink / validation (dataset_io.hpp) — imported last: it builds on the above
from .dataset import (Dataset, DatasetManifest, DatasetWriter, ManifestTimings,  # noqa: E402
                      ValidationReport, WriteSummary, field_digest, read_dataset,
                      relative_residual, validate_dataset, write_dataset)


# ---------------------------------------------------------------- reference-semantics generation
@dataclass
class ChipSpec:
    """ChipSpec (chip.hpp:55-80) with materials resolved to conductivities:
    layers are (z_lo, z_hi, k, role) bottom to top, role in {"core", "cache",
    "tim"}; lengths in meters, power ranges in W/mm^2."""
    extent: tuple = (10e-3, 10e-3, 0.51e-3)
    layers: list = field(default_factory=list)
    core_blocks: int = 0
    high_power: int = 0
    caches_per_layer: int = 0
    p_high: tuple = (0.0, 0.0)
    p_normal: tuple = (0.0, 0.0)
    p_cache: tuple = (0.0, 0.0)
    tsv_count: int = 0
    tsv_width: float = 0.0
    tsv_k: float = 0.0

    _ROLES = {"core": 0, "cache": 1, "tim": 2}

    @staticmethod
    def default_chip() -> "ChipSpec":
        """ChipSpec::default_chip() (chip.cpp:74-100), from the library."""
        c = _Chip()
        _load().bk_default_chip(C.byref(c))
        names = {v: k for k, v in ChipSpec._ROLES.items()}
        return ChipSpec(tuple(c.extent), [(c.layers[i].z_lo, c.layers[i].z_hi, c.layers[i].k,
                                           names[c.layers[i].role]) for i in range(c.n_layers)],
                        c.core_blocks, c.high_power, c.caches_per_layer, tuple(c.p_high),
                        tuple(c.p_normal), tuple(c.p_cache), c.tsv_count, c.tsv_width, c.tsv_k)

    def _c(self):
        c = _Chip()
        c.extent[:] = list(self.extent)
        if len(self.layers) > 16:
            raise InvalidSpecError("chip: at most 16 layers")
        c.n_layers = len(self.layers)
        for i, (lo, hi, k, role) in enumerate(self.layers):
            c.layers[i] = _Layer(lo, hi, k, self._ROLES[role])
        c.core_blocks, c.high_power, c.caches_per_layer = (self.core_blocks, self.high_power,
                                                           self.caches_per_layer)
        c.p_high[:], c.p_normal[:], c.p_cache[:] = (list(self.p_high), list(self.p_normal),
                                                    list(self.p_cache))
        c.tsv_count, c.tsv_width, c.tsv_k = self.tsv_count, self.tsv_width, self.tsv_k
        return c


@dataclass
class NoiseConfig:
    """NoiseConfig (pipeline.hpp:17-26): kind "none" | "uniform" | "gaussian"."""
    kind: str = "none"
    lo: float = 0.0
    hi: float = 0.0
    sigma: float = 0.0


@dataclass
class GenerationConfig:
    """GenerationConfig (pipeline.hpp:28-43); the grid spans the chip extent."""
    n_data: int = 0
    n_basis: int = 1
    n_k: int = 1
    solver: SolverConfig = field(default_factory=SolverConfig)
    noise: NoiseConfig = field(default_factory=NoiseConfig)
    master_seed: int = 0
    grid: tuple = (24, 24, 12)
    bc: BoundarySpec = field(default_factory=BoundarySpec)
    chip: ChipSpec = field(default_factory=ChipSpec.default_chip)

    def eta(self) -> int:
        return self.n_basis // self.n_k

    @staticmethod
    def default_run_config() -> "GenerationConfig":
        """configs/default.json (run_config.cpp:273-291): 24 x 24 x 12 over the
        default chip, Dirichlet 50 degC sides, Robin h = 3e4 / 50 degC top and
        bottom, 500 samples from 5 floorplans x 10 basis maps, uniform noise
        +-0.01 degC, Jacobi block CG to 1e-9."""
        bc = BoundarySpec([Dirichlet(50.0)] * 4 + [Robin(3e4, 50.0)] * 2)
        return GenerationConfig(500, 50, 5, SolverConfig(1e-9, 50000, "jacobi"),
                                NoiseConfig("uniform", -0.01, 0.01), 1, (24, 24, 12), bc)

    def _c(self):
        c = _GenCfg()
        c.nx, c.ny, c.nz = self.grid
        fc = self.bc._c()
        for f in range(6):
            c.bc[f] = fc[f]
        c.n_data, c.n_basis, c.n_k, c.master_seed = self.n_data, self.n_basis, self.n_k, \
            self.master_seed
        kinds = {"none": 0, "uniform": 1, "gaussian": 2}
        if self.noise.kind not in kinds:
            raise InvalidConfigError(f"noise: unknown kind {self.noise.kind!r}")
        c.noise_kind = kinds[self.noise.kind]
        c.noise_lo, c.noise_hi, c.noise_sigma = self.noise.lo, self.noise.hi, self.noise.sigma
        c.solver = self.solver._c()
        c.chip = self.chip._c()
        return c


def chip_fields(chip: ChipSpec, grid, n_k: int, eta: int, seed: int):
    """(k [n_k, n], q [n_k * eta, n]): the floorplan groups' conductivity and
    basis power maps (build_floorplans / rasterize_*, chip.cpp:180-306; draw
    seeds as generate_basis, pipeline.cpp:92-134). Host, bit-exact."""
    nx, ny, nz = grid
    n = nx * ny * nz
    k = np.empty((n_k, n), np.float64)
    q = np.empty((n_k * eta, n), np.float64)
    c = chip._c()
    _raise(_load().bk_chip_fields(C.byref(c), nx, ny, nz, n_k, eta, seed,
                                  k.ctypes.data_as(C.c_void_p), q.ctypes.data_as(C.c_void_p)),
           None, "chip_fields")
    return k, q


def draw_weights(n_basis: int, seed: int, n_data: int):
    """[n_data, n_basis]: draw_weights(n_basis, sample_seed_for(seed, l + 1))
    (pipeline.cpp:136-152) per sample l. Host, bit-exact."""
    w = np.empty((n_data, n_basis), np.float64)
    _raise(_load().bk_draw_weights(n_basis, seed, n_data, w.ctypes.data_as(C.c_void_p)), None,
           "draw_weights")
    return w


@dataclass
class GenerationResult:
    """generate_blockoa's result (pipeline.hpp:99-103) as arrays: k per
    floorplan group, per-sample u (= T) and q, residual and floorplan id."""
    k: object
    u: object
    q: object
    residual: object
    floorplan_id: np.ndarray
    reports: list
    timings: PhaseTimings


def generate_blockoa(cfg: GenerationConfig, u_out=None, q_out=None, resid_out=None,
                     ctx: Optional[Context] = None, check_converged: bool = True):
    """generate_blockoa(cfg) (pipeline.cpp:365-597) on the GPU: one batched
    block-CG launch for the n_k floorplan groups, then per group the fused
    combine + action kernel over all groups' basis columns (normalised Gaussian
    weights), per-sample interior noise, q = A_g (T) in apply_block order.
    Sample l belongs to group l mod n_k. Outputs may be numpy (host) or CUDA
    torch tensors."""
    ctx = _ctx(ctx)
    nx, ny, nz = cfg.grid
    n, N, nk = nx * ny * nz, int(cfg.n_data), int(cfg.n_k)
    eta = cfg.eta() if nk > 0 else 0
    k = np.empty((nk, n), np.float64)
    u_out = np.empty((N, n), np.float64) if u_out is None else u_out
    q_out = np.empty((N, n), np.float64) if q_out is None else q_out
    resid_out = np.empty(N, np.float64) if resid_out is None else resid_out
    fp = np.empty(N, np.int64)
    ptrs = [_ptr(a) for a in (u_out, q_out, resid_out)]
    res = [np.zeros(max(eta, 1), np.float64) for _ in range(max(nk, 1))]
    conv = [np.zeros(max(eta, 1), np.int8) for _ in range(max(nk, 1))]
    reps = (_Report * max(nk, 1))()
    for j in range(max(nk, 1)):
        reps[j] = _Report(0, 0, 0.0, res[j].ctypes.data_as(C.c_void_p),
                          conv[j].ctypes.data_as(C.c_void_p))
    tim = _Timings()
    c = cfg._c()
    st = _load().bk_generate_blockoa(ctx.h, C.byref(c), k.ctypes.data_as(C.c_void_p), ptrs[0][0],
                                     ptrs[1][0], ptrs[2][0], fp.ctypes.data_as(C.c_void_p), reps,
                                     C.byref(tim))
    if st == 7 and not check_converged:
        st = 0
    _raise(st, ctx.h, "generate_blockoa")
    timings = PhaseTimings(tim.assemble_s, tim.basis_solve_s, tim.combine_action_s, tim.h2d_s,
                           tim.d2h_s, tim.total_s, tim.iterations_total, tim.matvecs_total)
    return GenerationResult(k, u_out, q_out, resid_out, fp,
                            [_report(eta, reps[j], res[j], conv[j]) for j in range(nk)], timings)

