"""Dataset sink and validation — the reference's dataset_io.hpp on top of the
C ABI.

==========================  ==================================================
this module                 reference
==========================  ==================================================
``DatasetManifest``         ``DatasetManifest`` dataset.hpp:43-57
``ManifestTimings``         ``PhaseTimings`` dataset.hpp:17-25
``Dataset``                 ``Dataset`` dataset.hpp:59-64 (sample fields as
                            n_data x n arrays instead of a vector<Sample>)
``write_dataset``           ``write_dataset`` dataset_io.cpp:160-225
``DatasetWriter``           the same, streaming chip by chip (device outputs
                            drained through pinned buffers by the library)
``read_dataset``            ``read_dataset`` dataset_io.cpp:227-320
``validate_dataset``        ``validate_dataset`` dataset_io.cpp:322-361
``field_digest``            ``field_digest`` discretize.cpp:302-319
``relative_residual``       ``relative_residual`` discretize.cpp:275-286
==========================  ==================================================

On-disk format (identical to the reference): ``manifest.json`` plus
``k.bin`` / ``q.bin`` / ``u.bin``, each the stacked samples as little-endian
float64 in flat cell order. The manifest text follows nlohmann::json 3.11.3's
``dump(2)`` layout (sorted keys, two-space indent, one element per line,
shortest round-trip numbers), so a dataset written here is byte-identical to
one the reference writes for the same samples. (oracle/_ref is built against
the copy bundled with cudnn_frontend, patched to print integer arrays on one
line; tests/test_dataset.py compares modulo that.) The payload I/O, digest and residual sweeps run in
libblockoa_b200.so (residuals on the GPU); only the JSON is handled here.

Extension: a non-uniform stack (``GridSpec.dz``, BASELINE config 4) is recorded
under an extra ``dz_m`` key, which the reference's reader ignores.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import (Adiabatic, BoundarySpec, Context, CorruptManifestError, Dirichlet,
               DimensionMismatchError, DiscreteOperator, GridSpec, Robin, SizeMismatchError,
               _ctx, _is_torch, _load, _ptr, _raise)

TOOL_VERSION = "blockoa-b200-0.1.0"
MANIFEST = "manifest.json"
FIELD_FILES = ("k.bin", "q.bin", "u.bin")
_FACE_KEYS = ("xlo", "xhi", "ylo", "yhi", "zlo", "zhi")


# ---------------------------------------------------------------- types
@dataclass
class ManifestTimings:
    """PhaseTimings (dataset.hpp:17-25). The GPU pipeline fuses combine and
    operator action into one kernel; its time is recorded as combine_s."""
    basis_solve_s: float = 0.0
    combine_s: float = 0.0
    operator_action_s: float = 0.0
    solve_s: float = 0.0
    total_s: float = 0.0
    iterations_total: int = 0
    matvecs_total: int = 0


@dataclass
class DatasetManifest:
    format_version: int = 1
    method: str = "blockoa"
    n_data: int = 0
    master_seed: int = 0
    floorplan_ids: List[int] = field(default_factory=list)
    floorplan_digests: List[Tuple[int, int]] = field(default_factory=list)
    timings: ManifestTimings = field(default_factory=ManifestTimings)
    residual_tol_claimed: float = 0.0
    tool_version: str = TOOL_VERSION
    config_echo: str = ""
    requested_n_data: int = 0
    dropped_count: int = 0


@dataclass
class Dataset:
    """grid + bc + the samples' k, q, u as n_data x n arrays (read_dataset
    returns read-only memory maps) + manifest."""
    grid: GridSpec
    bc: BoundarySpec
    k: np.ndarray
    q: np.ndarray
    u: np.ndarray
    manifest: DatasetManifest


@dataclass
class WriteSummary:
    dir: str
    n_data: int
    payload_bytes_per_file: int


@dataclass
class ValidationReport:
    pass_count: int
    fail_count: int
    max_residual: float
    residuals: np.ndarray


# ---------------------------------------------------------------- JSON
def _fmt_float(x: float) -> str:
    """nlohmann::json's number format: shortest round-trip digits, fixed
    notation when the decimal point falls in (-4, 15], else d.ddde+XX."""
    if not math.isfinite(x):
        return "null"
    r = repr(float(x))
    neg = r.startswith("-")
    if neg:
        r = r[1:]
    mant, _, exp = r.partition("e")
    e = int(exp) if exp else 0
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    if not digits:  # zero
        return ("-" if neg else "") + "0.0"
    lead = len(ip + fp) - len((ip + fp).lstrip("0"))
    decpt = len(ip) - lead + e  # value = 0.digits x 10^decpt
    digits = digits.rstrip("0")
    n = decpt
    k = len(digits)
    if k <= n <= 15:
        s = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        s = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        s = "0." + "0" * (-n) + digits
    else:
        s = digits[0] + ("." + digits[1:] if k > 1 else "")
        ee = n - 1
        s += "e" + ("-" if ee < 0 else "+") + f"{abs(ee):02d}"
    return ("-" if neg else "") + s


def _dump(v, indent: int = 0) -> str:
    """nlohmann::json::dump(2) of a JSON value (objects with sorted keys)."""
    pad, inner = " " * indent, " " * (indent + 2)
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f"{inner}{json.dumps(k)}: {_dump(v[k], indent + 2)}" for k in sorted(v)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, (list, tuple)):
        if not v:
            return "[]"
        items = [inner + _dump(x, indent + 2) for x in v]
        return "[\n" + ",\n".join(items) + "\n" + pad + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if v is None:
        return "null"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return _fmt_float(float(v))
    return json.dumps(str(v))


def _face_json(f) -> dict:
    if isinstance(f, Dirichlet):
        return {"type": "dirichlet", "u0_c": float(f.u0)}
    if isinstance(f, Robin):
        return {"type": "robin", "h_w_m2k": float(f.h), "u_inf_c": float(f.u_inf)}
    if isinstance(f, Adiabatic):  # the reference's zero-flux face
        return {"type": "robin", "h_w_m2k": 1e-300, "u_inf_c": 0.0}
    raise CorruptManifestError(f"manifest: unknown face condition {f!r}")


def _face_from_json(j) -> object:
    t = j["type"]
    if t == "dirichlet":
        return Dirichlet(float(j["u0_c"]))
    if t == "robin":
        return Robin(float(j["h_w_m2k"]), float(j["u_inf_c"]))
    raise CorruptManifestError(f"manifest: unknown boundary type '{t}'")


def manifest_json(grid: GridSpec, bc: BoundarySpec, m: DatasetManifest) -> str:
    """manifest_to_json (dataset_io.cpp:120-142) + dump(2) + newline."""
    t = m.timings
    j = {
        "format_version": int(m.format_version),
        "method": m.method,
        "n_data": int(m.n_data),
        "grid": [grid.nx, grid.ny, grid.nz],
        "extent_m": [float(grid.lx), float(grid.ly), float(grid.lz)],
        "bc": {k: _face_json(f) for k, f in zip(_FACE_KEYS, bc.faces)},
        "master_seed": int(m.master_seed),
        "floorplan_ids": [int(i) for i in m.floorplan_ids],
        "timings": {"basis_solve_s": float(t.basis_solve_s), "combine_s": float(t.combine_s),
                    "operator_action_s": float(t.operator_action_s),
                    "solve_s": float(t.solve_s), "total_s": float(t.total_s),
                    "iterations_total": int(t.iterations_total),
                    "matvecs_total": int(t.matvecs_total)},
        "residual_tol_claimed": float(m.residual_tol_claimed),
        "tool_version": m.tool_version,
        "floorplan_digests": [{"id": int(i), "k_digest": int(d)} for i, d in m.floorplan_digests],
        "requested_n_data": int(m.requested_n_data),
        "dropped_count": int(m.dropped_count),
    }
    if m.config_echo:
        j["config"] = json.loads(m.config_echo)
    if grid.dz is not None:
        j["dz_m"] = [float(d) for d in grid.dz]
    return _dump(j) + "\n"


# ---------------------------------------------------------------- digests, residuals
def field_digest(k, grid: GridSpec) -> int:
    """field_digest (discretize.cpp:302-319): FNV-1a over (nx, ny, nz) and the
    value bytes. Host or CUDA input (a CUDA tensor is copied to the host)."""
    if _is_torch(k):
        k = k.detach().cpu().numpy()
    k = np.ascontiguousarray(k, dtype=np.float64).reshape(-1)
    if k.size != grid.cell_count():
        raise DimensionMismatchError("field_digest: field length does not match grid")
    return int(_load().bk_field_digest(grid.nx, grid.ny, grid.nz, k.ctypes.data_as(C.c_void_p)))


def relative_residual(op: DiscreteOperator, u, q, out=None):
    """relative_residual (discretize.cpp:275-286) for one sample (u, q of
    length n) or a batch (N x n each): ||V q + g - A u|| / ||V q + g||."""
    single = (u.ndim if hasattr(u, "ndim") else np.asarray(u).ndim) == 1
    n = op.grid.cell_count()
    N = 1 if single else int(u.shape[0])
    if (u.numel() if _is_torch(u) else np.asarray(u).size) != N * n:
        raise DimensionMismatchError("relative_residual: u length != n")
    if (q.numel() if _is_torch(q) else np.asarray(q).size) != N * n:
        raise DimensionMismatchError("relative_residual: q length != n")
    res = np.empty(N, np.float64) if out is None else out
    pu, pq, pr = _ptr(u), _ptr(q), _ptr(res)
    _raise(_load().bk_residuals(op.ctx.h, op.h, pu[0], pq[0], N, pr[0]), op.ctx.h,
           "relative_residual")
    return float(res[0]) if single and out is None else res


# ---------------------------------------------------------------- writer
class DatasetWriter:
    """Streaming write_dataset: ``append`` chip outputs as they are produced
    (numpy arrays or CUDA tensors), ``commit`` the manifest, which makes the
    dataset appear atomically at ``dir``. Leaving the ``with`` block without
    committing discards the staged files."""

    def __init__(self, dir: str, grid: GridSpec, bc: BoundarySpec, method: str = "blockoa",
                 master_seed: int = 0, residual_tol_claimed: float = 1e-12,
                 overwrite: bool = False, ctx: Optional[Context] = None):
        self.dir, self.grid, self.bc = str(dir), grid, bc
        self.ctx = ctx
        self.manifest = DatasetManifest(method=method, master_seed=master_seed,
                                        residual_tol_claimed=residual_tol_claimed)
        self._digests = {}
        lib = _load()
        h = C.c_void_p()
        st = lib.bk_dataset_open(self.dir.encode(), int(bool(overwrite)), grid.cell_count(),
                                 C.byref(h))
        self.h = h
        if st:
            msg = lib.bk_dataset_error(h).decode() if h else "write_dataset"
            self.close()
            _raise(st, None, msg)

    def _check(self, st, what):
        if st:
            raise _err_type(st)(f"{what}: {_load().bk_dataset_error(self.h).decode()}")

    def append(self, k, q, u, floorplan_id: int, k_digest: Optional[int] = None):
        """Add samples: k is the chip's field (n), q / u are m x n. On the GPU
        path pass CUDA tensors (drained by the library, PCIe overlapped with
        the file write)."""
        n = self.grid.cell_count()
        m = int(q.shape[0])
        for a, what in ((q, "q"), (u, "u")):
            if tuple(a.shape) != (m, n):
                raise DimensionMismatchError(f"write_dataset: {what} must be {m} x {n}")
        if (k.numel() if _is_torch(k) else np.asarray(k).size) != n:
            raise DimensionMismatchError("write_dataset: sample grid mismatch")
        if k_digest is None:
            k_digest = field_digest(k, self.grid)
        dev = any(_is_torch(a) and a.is_cuda for a in (k, q, u))
        ctx = _ctx(self.ctx) if dev else self.ctx
        pk, pq, pu = _ptr(k), _ptr(q), _ptr(u)
        st = _load().bk_dataset_append(self.h, ctx.h if ctx is not None else None, pk[0], m,
                                       pq[0], pu[0])
        self._check(st, "write_dataset")
        self.manifest.floorplan_ids.extend([int(floorplan_id)] * m)
        if int(floorplan_id) not in self._digests:
            self._digests[int(floorplan_id)] = int(k_digest)
            self.manifest.floorplan_digests.append((int(floorplan_id), int(k_digest)))

    @property
    def n_data(self) -> int:
        return int(_load().bk_dataset_count(self.h))

    @property
    def write_seconds(self) -> float:
        """Time spent inside write(2) so far."""
        return float(_load().bk_dataset_write_seconds(self.h))

    def commit(self, timings: Optional[ManifestTimings] = None,
               requested_n_data: Optional[int] = None, dropped_count: int = 0,
               config_echo: str = "") -> WriteSummary:
        m = self.manifest
        m.n_data = self.n_data
        if len(m.floorplan_ids) != m.n_data:
            raise DimensionMismatchError("write_dataset: floorplan_ids != samples")
        if timings is not None:
            m.timings = timings
        m.requested_n_data = m.n_data if requested_n_data is None else int(requested_n_data)
        m.dropped_count = int(dropped_count)
        m.config_echo = config_echo
        text = manifest_json(self.grid, self.bc, m)
        self._check(_load().bk_dataset_commit(self.h, text.encode()), "write_dataset")
        summary = WriteSummary(self.dir, m.n_data, m.n_data * self.grid.cell_count() * 8)
        self.close()
        return summary

    def close(self):
        if getattr(self, "h", None):
            _load().bk_dataset_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _err_type(st):
    from . import _STATUS, Error
    return _STATUS.get(st, Error)


def write_dataset(ds: Dataset, dir: str, overwrite: bool = False) -> WriteSummary:
    """write_dataset (dataset_io.cpp:160-225) for a dataset held in memory."""
    n = ds.grid.cell_count()
    n_data = int(ds.manifest.n_data)
    if int(ds.k.shape[0]) != n_data or int(ds.q.shape[0]) != n_data or int(ds.u.shape[0]) != n_data:
        raise DimensionMismatchError("write_dataset: manifest n_data != samples")
    if len(ds.manifest.floorplan_ids) != n_data:
        raise DimensionMismatchError("write_dataset: floorplan_ids != samples")
    for a in (ds.k, ds.q, ds.u):
        if a.ndim != 2 or int(a.shape[1]) != n:
            raise DimensionMismatchError("write_dataset: sample grid mismatch")
    m = ds.manifest
    w = DatasetWriter(dir, ds.grid, ds.bc, m.method, m.master_seed, m.residual_tol_claimed,
                      overwrite)
    with w:
        w.manifest.tool_version = m.tool_version
        w.manifest.format_version = m.format_version
        w.manifest.floorplan_digests = list(m.floorplan_digests)
        w._digests = {i: d for i, d in m.floorplan_digests}
        j = 0
        ids = m.floorplan_ids
        while j < n_data:  # runs of samples sharing k and id: one append each
            e = j + 1
            while e < n_data and ids[e] == ids[j] and np.array_equal(ds.k[e], ds.k[j]):
                e += 1
            dig = w._digests.get(int(ids[j]))
            w.append(ds.k[j], ds.q[j:e], ds.u[j:e], ids[j],
                     k_digest=dig if dig is not None else 0)
            j = e
        w.manifest.floorplan_digests = list(m.floorplan_digests)
        return w.commit(m.timings, m.requested_n_data, m.dropped_count, m.config_echo)


# ---------------------------------------------------------------- reader
def _required(j, key, typ):
    if key not in j:
        raise CorruptManifestError(f"manifest: missing key '{key}'")
    v = j[key]
    ok = {int: lambda x: isinstance(x, int) and not isinstance(x, bool),
          float: lambda x: isinstance(x, (int, float)) and not isinstance(x, bool),
          str: lambda x: isinstance(x, str),
          list: lambda x: isinstance(x, list)}[typ](v)
    if not ok:
        raise CorruptManifestError(f"manifest: bad value for '{key}'")
    return v


def read_dataset(dir: str) -> Dataset:
    """read_dataset (dataset_io.cpp:227-320): manifest checks, file sizes
    checked before any payload is touched; payloads are memory-mapped."""
    path = os.path.join(dir, MANIFEST)
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise CorruptManifestError(f"read_dataset: cannot open {path}")
    try:
        j = json.loads(text)
    except ValueError as e:
        raise CorruptManifestError(f"read_dataset: manifest parse: {e}")
    if not isinstance(j, dict):
        raise CorruptManifestError("read_dataset: manifest parse: not an object")
    m = DatasetManifest()
    m.format_version = _required(j, "format_version", int)
    if m.format_version != 1:
        raise CorruptManifestError("read_dataset: unsupported format_version")
    m.method = _required(j, "method", str)
    m.n_data = _required(j, "n_data", int)
    counts = _required(j, "grid", list)
    extent = _required(j, "extent_m", list)
    if len(counts) != 3 or len(extent) != 3:
        raise CorruptManifestError("read_dataset: grid/extent_m must have 3 entries")
    if "bc" not in j:
        raise CorruptManifestError("manifest: missing key 'bc'")
    try:
        bc = BoundarySpec([_face_from_json(j["bc"][k]) for k in _FACE_KEYS])
    except (KeyError, TypeError, ValueError) as e:
        raise CorruptManifestError(f"read_dataset: bad bc: {e}")
    m.master_seed = _required(j, "master_seed", int)
    m.floorplan_ids = [int(i) for i in _required(j, "floorplan_ids", list)]
    if "timings" not in j:
        raise CorruptManifestError("manifest: missing key 'timings'")
    try:
        t = j["timings"]
        m.timings = ManifestTimings(float(t["basis_solve_s"]), float(t["combine_s"]),
                                    float(t["operator_action_s"]), float(t["solve_s"]),
                                    float(t["total_s"]), int(t["iterations_total"]),
                                    int(t["matvecs_total"]))
    except (KeyError, TypeError, ValueError) as e:
        raise CorruptManifestError(f"read_dataset: bad timings: {e}")
    m.residual_tol_claimed = float(_required(j, "residual_tol_claimed", float))
    m.tool_version = _required(j, "tool_version", str)
    m.floorplan_digests = [(int(e["id"]), int(e["k_digest"])) for e in j.get("floorplan_digests", [])]
    m.requested_n_data = int(j.get("requested_n_data", 0))
    m.dropped_count = int(j.get("dropped_count", 0))
    if "config" in j:
        m.config_echo = json.dumps(j["config"])
    dz = j.get("dz_m")
    grid = GridSpec(int(counts[0]), int(counts[1]), int(counts[2]), float(extent[0]),
                    float(extent[1]), float(extent[2]), dz)
    if min(grid.nx, grid.ny, grid.nz) < 1 or min(grid.lx, grid.ly, grid.lz) <= 0:
        raise CorruptManifestError("read_dataset: invalid grid")
    if m.n_data < 0:
        raise CorruptManifestError("read_dataset: negative n_data")
    if len(m.floorplan_ids) != m.n_data:
        raise CorruptManifestError("read_dataset: floorplan_ids length != n_data")
    n = grid.cell_count()
    expect = m.n_data * n * 8
    for name in FIELD_FILES:
        p = os.path.join(dir, name)
        if not os.path.exists(p):
            raise SizeMismatchError(f"read_dataset: missing {name}")
        size = os.path.getsize(p)
        if size != expect:
            raise SizeMismatchError(f"read_dataset: {name} is {size} bytes, expected {expect}")
    fields = []
    for name in FIELD_FILES:
        if m.n_data == 0:
            fields.append(np.empty((0, n), np.float64))
        else:
            fields.append(np.memmap(os.path.join(dir, name), dtype="<f8", mode="r",
                                    shape=(m.n_data, n)))
    return Dataset(grid, bc, fields[0], fields[1], fields[2], m)


def validate_dataset(dir: str, tol: float, ctx: Optional[Context] = None) -> ValidationReport:
    """validate_dataset (dataset_io.cpp:322-361): per stored sample,
    ||A u - (M q + g)|| / ||M q + g|| against one GPU-assembled operator per
    distinct k; a k whose digest contradicts the manifest fails with +inf."""
    ds = read_dataset(dir)
    return validate_samples(ds, tol, ctx)


def validate_samples(ds: Dataset, tol: float, ctx: Optional[Context] = None) -> ValidationReport:
    ctx = _ctx(ctx)
    m = ds.manifest
    n_data = int(m.n_data)
    res = np.zeros(n_data, np.float64)
    ids = np.ascontiguousarray(m.floorplan_ids, dtype=np.uint64)
    dids = np.ascontiguousarray([d[0] for d in m.floorplan_digests], dtype=np.uint64)
    ddig = np.ascontiguousarray([d[1] for d in m.floorplan_digests], dtype=np.uint64)
    g, keep = ds.grid._c()
    faces = ds.bc._c()

    class _Val(C.Structure):
        _fields_ = [("pass_count", C.c_int64), ("fail_count", C.c_int64),
                    ("max_residual", C.c_double)]

    rep = _Val()
    pk, pu, pq = _ptr(ds.k), _ptr(ds.u), _ptr(ds.q)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    st = _load().bk_validate_samples(ctx.h, C.byref(g), faces, pk[0], pu[0], pq[0], n_data,
                                     vp(ids), len(dids), vp(dids), vp(ddig), float(tol),
                                     vp(res), C.byref(rep))
    _raise(st, ctx.h, "validate_dataset")
    return ValidationReport(int(rep.pass_count), int(rep.fail_count), float(rep.max_residual), res)
