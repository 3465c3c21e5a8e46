"""B200-native multigrid hierarchical data refactoring (arXiv 2007.04457).

Python mirror of the reference's public API (``hgr``, /root/reference/proj/
include/hgr), running on the sm_100a kernels of ``libhgr_b200.so`` through the
C ABI (include/hgr_cuda.h). Names, argument meaning and error behaviour follow
the reference:

=========================  ==================================================
reference (hgr::)           here
=========================  ==================================================
GridHierarchy              GridHierarchy (grid_hierarchy.hpp:47-194)
decompose(data, g)         decompose(data, g) -> RefactoredArray (refactor.hpp:32-57)
recompose(r, upto_class)   recompose(r, upto_class)            (refactor.hpp:63-90)
error_report               error_report                        (refactor.hpp:100-120)
extract_class/scatter_class extract_class / scatter_class      (refactor.hpp:149-170)
interpolate_to_fine, compute_coefficients, apply_coefficients (transforms.hpp:76-124)
compute_correction         compute_correction                  (correction.hpp:348-365)
masstrans_apply, thomas_solve, mass_apply, transfer_apply (correction.hpp:58-223)
hgr::error                 HgrError (error.hpp:9-11)
=========================  ==================================================

Arrays are torch CUDA tensors (device path, stream-ordered on torch's current
stream) or numpy arrays (host path: H2D, kernels, D2H). torch is plumbing for
device memory and streams only; all arithmetic runs in the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib

__all__ = [
    "HgrError", "GridHierarchy", "RefactoredArray", "Plan", "decompose", "recompose",
    "error_report", "ErrorReport", "extract_class", "scatter_class", "interpolate_to_fine",
    "compute_coefficients", "apply_coefficients", "compute_correction", "masstrans_apply",
    "thomas_solve", "mass_apply", "transfer_apply", "build_hierarchy",
]


class HgrError(RuntimeError):
    """hgr::error (error.hpp:9-11): all domain failures."""


def _check(rc: int) -> None:
    if rc != _lib.HGR_OK:
        raise HgrError(_lib.last_error())


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _dtype_tag(x) -> str:
    if _is_torch(x):
        import torch
        if x.dtype == torch.float64:
            return "f64"
        if x.dtype == torch.float32:
            return "f32"
    else:
        if x.dtype == np.float64:
            return "f64"
        if x.dtype == np.float32:
            return "f32"
    raise HgrError(f"unsupported dtype {x.dtype} (float32 / float64 only)")


def _ptr(x) -> int:
    return x.data_ptr() if _is_torch(x) else x.ctypes.data


def _stream_of(x) -> Optional[int]:
    if _is_torch(x):
        import torch
        return torch.cuda.current_stream(x.device).cuda_stream
    return None


class GridHierarchy:
    """Dyadic level structure over per-dimension coordinates
    (grid_hierarchy.hpp:47-194). Validation and messages match the reference;
    the hierarchy arithmetic (spacings, weights) is done in double as there."""

    def __init__(self, coords_per_dim: Sequence[Sequence[float]]):
        coords = [np.ascontiguousarray(np.asarray(c, dtype=np.float64)) for c in coords_per_dim]
        if not (1 <= len(coords) <= 3):
            raise HgrError("grid must have 1 to 3 dimensions")
        self._coords = coords
        self._desc = _lib.GridDesc()
        self._desc.rank = len(coords)
        for d, c in enumerate(coords):
            self._desc.extents[d] = c.size
            self._desc.coords[d] = c.ctypes.data
        L = _lib.load().hgr_levels(C.byref(self._desc))
        if L < 0:
            raise HgrError(_lib.last_error())
        self._levels = L

    @staticmethod
    def uniform(sizes: Sequence[int]) -> "GridHierarchy":
        """GridHierarchy::uniform (grid_hierarchy.hpp:73-80)."""
        return GridHierarchy([np.arange(n, dtype=np.float64) for n in sizes])

    # -- accessors (grid_hierarchy.hpp:82-150)
    def rank(self) -> int:
        return len(self._coords)

    def levels(self) -> int:
        return self._levels

    def class_count(self) -> int:
        return self._levels + 1

    def coords(self, d: int) -> np.ndarray:
        return self._coords[self._check_dim(d)]

    def finest_extent(self, d: int) -> int:
        return int(self._coords[self._check_dim(d)].size)

    def finest_extents(self) -> list:
        return [int(c.size) for c in self._coords]

    def level_stride(self, level: int) -> int:
        return 1 << (self._levels - self._check_level(level))

    def level_extent(self, level: int, d: int) -> int:
        return (self.finest_extent(d) - 1) // self.level_stride(level) + 1

    def level_extents(self, level: int) -> list:
        return [self.level_extent(level, d) for d in range(self.rank())]

    def level_node_count(self, level: int) -> int:
        return int(np.prod(self.level_extents(level)))

    def spacings(self, level: int, d: int) -> np.ndarray:
        s = self.level_stride(level)
        c = self.coords(d)
        return c[s::s] - c[:-1:s] if c.size > 1 else np.zeros(0)

    def refined_weights(self, level: int, d: int) -> np.ndarray:
        """(to_left, to_right) per refined node (grid_hierarchy.hpp:27-31)."""
        if not (1 <= level <= self._levels):
            raise HgrError("level out of range")
        h = self.spacings(level, d)
        span = h[0::2] + h[1::2]
        return np.stack([h[1::2] / span, h[0::2] / span], axis=1)

    def node_class(self, finest_index: Sequence[int]) -> int:
        cls = 0
        for i in finest_index[: self.rank()]:
            if i == 0:
                continue
            tz = (int(i) & -int(i)).bit_length() - 1
            cls = max(cls, self._levels - tz)
        return cls

    def class_node_count(self, cls: int) -> int:
        n = _lib.load().hgr_class_node_count(C.byref(self._desc), int(cls))
        if n == 0:
            raise HgrError(_lib.last_error() or "level out of range")
        return int(n)

    def _check_dim(self, d: int) -> int:
        if not (0 <= d < self.rank()):
            raise HgrError("dimension index out of range")
        return d

    def _check_level(self, level: int) -> int:
        if not (0 <= level <= self._levels):
            raise HgrError("level out of range")
        return level

    @property
    def desc(self):
        return self._desc


def build_hierarchy(coords_per_dim) -> GridHierarchy:
    return GridHierarchy(coords_per_dim)


@dataclass
class RefactoredArray:
    """In-place coefficient pyramid (refactor.hpp:20-26)."""
    data: object
    hierarchy: GridHierarchy


class Plan:
    """Reusable device plan (tables + workspace) for repeated calls on one grid
    and dtype -- hgr_cuda_plan_* in the C ABI."""

    def __init__(self, g: GridHierarchy, dtype: str = "f64"):
        if dtype not in ("f64", "f32"):
            raise HgrError("dtype must be 'f32' or 'f64'")
        self.hierarchy = g
        self.dtype = dtype
        self._h = C.c_void_p()
        _check(_lib.load().hgr_cuda_plan_create(C.byref(g.desc),
                                                 _lib.HGR_F64 if dtype == "f64" else _lib.HGR_F32,
                                                 C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().hgr_cuda_plan_destroy(h)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self._h = None

    @property
    def levels(self) -> int:
        return _lib.load().hgr_cuda_plan_levels(self._h)

    @property
    def workspace_bytes(self) -> int:
        return int(_lib.load().hgr_cuda_plan_workspace_bytes(self._h))

    def launches(self, direction: int, upto_class: int) -> int:
        return _lib.load().hgr_cuda_plan_launches(self._h, direction, upto_class)

    def _operand(self, x, what: str):
        """A plan operand must be a contiguous CUDA tensor of the plan's finest
        shape and dtype (the kernels trust these; a mismatch would read or
        write past the tensor)."""
        import torch
        if not _is_torch(x) or not x.is_cuda:
            raise HgrError(f"{what}: expected a CUDA tensor")
        if list(x.shape) != self.hierarchy.finest_extents():
            raise HgrError(f"{what}: array shape does not match grid")
        if x.dtype != (torch.float64 if self.dtype == "f64" else torch.float32):
            raise HgrError(f"{what}: dtype {x.dtype} does not match the plan ({self.dtype})")
        if not x.is_contiguous():
            raise HgrError(f"{what}: tensor must be contiguous")
        return x

    def _pair(self, src, out, what: str):
        self._operand(src, what)
        self._operand(out, what)
        if src.device != out.device:
            raise HgrError(f"{what}: input and output are on different devices")

    def decompose_(self, data, stream: Optional[int] = None) -> None:
        """In-place, stream-ordered decompose of a device tensor (no sync)."""
        self._operand(data, "decompose")
        _check(_lib.load().hgr_cuda_plan_decompose(self._h, _ptr(data),
                                                   stream if stream is not None else _stream_of(data)))

    def decompose_into(self, src, out, stream: Optional[int] = None) -> None:
        """Out-of-place, stream-ordered decompose (src untouched; no sync)."""
        self._pair(src, out, "decompose")
        _check(_lib.load().hgr_cuda_plan_decompose_to(self._h, _ptr(src), _ptr(out),
                                                      stream if stream is not None else _stream_of(src)))

    def recompose_into(self, src, out, upto_class: int, stream: Optional[int] = None) -> None:
        self._pair(src, out, "recompose")
        _check(_lib.load().hgr_cuda_plan_recompose(self._h, _ptr(src), _ptr(out), int(upto_class),
                                                   stream if stream is not None else _stream_of(src)))

    def sync_status(self, stream: Optional[int] = None) -> None:
        _check(_lib.load().hgr_cuda_plan_sync_status(self._h, stream))

    def autotune(self, src, out, stream: Optional[int] = None) -> dict:
        """Tile-segment autotuning: rank the segment lengths of the
        fused decompose / recompose / interpolation kernels per level with the
        sector model (perf_model.hpp:71-137), time the top three, keep the
        fastest. src is read, out is overwritten. Returns the JSON report."""
        self._pair(src, out, "autotune")
        lib = _lib.load()
        st = stream if stream is not None else _stream_of(src)
        n = C.c_size_t(0)
        buf = C.create_string_buffer(1 << 20)  # ~100 bytes per candidate
        _check(lib.hgr_cuda_plan_autotune(self._h, _ptr(src), _ptr(out), st, buf, len(buf),
                                          C.byref(n)))
        if n.value >= len(buf):
            raise HgrError("autotune report truncated")
        return json.loads(buf.value.decode())

    def reset_tuning(self) -> None:
        _check(_lib.load().hgr_cuda_plan_reset_tuning(self._h))

    KINDS = ("fused_decompose_level", "fused_recompose_level", "thomas", "recompose_interp",
             "assembly", "small_levels")

    def set_profiling(self, on: bool) -> None:
        """Bracket every launch with CUDA events (per kernel class); resets totals."""
        _check(_lib.load().hgr_cuda_plan_set_profiling(self._h, 1 if on else 0))

    def read_profile(self) -> dict:
        """{kind: (ms, algorithmic bytes, launches)} since set_profiling (synchronizes)."""
        n = len(self.KINDS)
        ms, by, la = (C.c_double * n)(), (C.c_double * n)(), (C.c_long * n)()
        _check(_lib.load().hgr_cuda_plan_read_profile(self._h, ms, by, la))
        return {k: (ms[i], by[i], la[i]) for i, k in enumerate(self.KINDS)}


def _check_shape(data, g: GridHierarchy, what: str) -> None:
    if list(data.shape) != g.finest_extents():
        raise HgrError(f"{what}: array shape does not match grid")


def decompose(data, g: GridHierarchy) -> RefactoredArray:
    """hgr::decompose (refactor.hpp:32-57). The input is taken by value (not modified)."""
    _check_shape(data, g, "decompose")
    t = _dtype_tag(data)
    lib = _lib.load()
    if _is_torch(data) and data.is_cuda:
        src = data.detach().contiguous()
        out = src.new_empty(src.shape)
        _check(getattr(lib, f"hgr_cuda_decompose_to_{t}")(C.byref(g.desc), _ptr(src), _ptr(out),
                                                           _stream_of(src)))
    elif _is_torch(data):  # host tensor (pinned ones move by direct DMA)
        import torch
        out = torch.empty(tuple(data.shape), dtype=data.dtype, pin_memory=data.is_pinned())
        out.copy_(data)
        _check(getattr(lib, f"hgr_decompose_host_{t}")(C.byref(g.desc), _ptr(out)))
    else:
        out = np.array(data, copy=True, order="C")
        _check(getattr(lib, f"hgr_decompose_host_{t}")(C.byref(g.desc), _ptr(out)))
    return RefactoredArray(out, g)


def recompose(r: RefactoredArray, upto_class: int):
    """hgr::recompose (refactor.hpp:63-90)."""
    g, src = r.hierarchy, r.data
    t = _dtype_tag(src)
    lib = _lib.load()
    if _is_torch(src) and src.is_cuda:
        src = src.contiguous()
        out = src.new_empty(src.shape)
        _check(getattr(lib, f"hgr_cuda_recompose_{t}")(C.byref(g.desc), _ptr(src), _ptr(out),
                                                        int(upto_class), _stream_of(src)))
    elif _is_torch(src):  # host tensor
        src = src.contiguous()
        out = src.new_empty(src.shape, pin_memory=src.is_pinned())
        _check(getattr(lib, f"hgr_recompose_host_{t}")(C.byref(g.desc), _ptr(src), _ptr(out),
                                                        int(upto_class)))
    else:
        src = np.ascontiguousarray(src)
        out = np.empty_like(src)
        _check(getattr(lib, f"hgr_recompose_host_{t}")(C.byref(g.desc), _ptr(src), _ptr(out),
                                                        int(upto_class)))
    return out


@dataclass
class ErrorReport:
    l2_abs: float = 0.0
    l2_rel: float = 0.0
    linf_abs: float = 0.0
    linf_rel: float = 0.0


def error_report(original, reconstruction) -> ErrorReport:
    """error_report (refactor.hpp:100-120), accumulated in double by the
    device reduction (hgr_cuda_error_report_*); host arrays are staged to the
    current CUDA device."""
    if tuple(original.shape) != tuple(reconstruction.shape):
        raise HgrError("error_report: shape mismatch")
    if (original.numel() if _is_torch(original) else np.size(original)) == 0:
        return ErrorReport()
    a, _ = _to_device(original)
    b, _ = _to_device(reconstruction)
    if a.dtype != b.dtype:
        b = b.to(a.dtype)
    b = b.to(a.device).contiguous()
    out = (C.c_double * 4)()
    _check(getattr(_lib.load(), f"hgr_cuda_error_report_{_dtype_tag(a)}")(
        a.numel(), _ptr(a), _ptr(b), out, _stream_of(a)))
    return ErrorReport(l2_abs=out[0], l2_rel=out[1], linf_abs=out[2], linf_rel=out[3])


def _to_device(x):
    if _is_torch(x):
        return (x.contiguous(), True) if x.is_cuda else (x.contiguous().cuda(), False)
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda(), False


def _back(x, was_torch):
    return x if was_torch else x.cpu().numpy()


def extract_class(r: RefactoredArray, cls: int):
    """extract_class (refactor.hpp:149-157): class values in row-major order."""
    import torch
    g = r.hierarchy
    if not (0 <= cls <= g.levels()):
        raise HgrError("level out of range")
    d, was = _to_device(r.data)
    out = torch.empty(g.class_node_count(cls), dtype=d.dtype, device=d.device)
    _check(getattr(_lib.load(), f"hgr_cuda_extract_class_{_dtype_tag(d)}")(
        C.byref(g.desc), _ptr(d), int(cls), _ptr(out), _stream_of(d)))
    return _back(out, was)


def scatter_class(r: RefactoredArray, cls: int, values) -> None:
    """scatter_class (refactor.hpp:159-170), in place on r.data."""
    g = r.hierarchy
    if not (0 <= cls <= g.levels()):
        raise HgrError("level out of range")
    if len(values) != g.class_node_count(cls):
        raise HgrError("scatter_class: value count does not match class size")
    d, was = _to_device(r.data)
    v, _ = _to_device(values if _is_torch(values) else np.asarray(values))
    v = v.to(d.dtype).contiguous()
    _check(getattr(_lib.load(), f"hgr_cuda_scatter_class_{_dtype_tag(d)}")(
        C.byref(g.desc), _ptr(d), int(cls), _ptr(v), _stream_of(d)))
    if not was:
        r.data[...] = d.cpu().numpy()


def _single(op: str, x, g: GridHierarchy, level: int, out_level: int):
    import torch
    d, was = _to_device(x)
    ext = g.level_extents(out_level) if 0 <= out_level <= g.levels() else list(d.shape)
    out = torch.empty(ext, dtype=d.dtype, device=d.device)
    _check(getattr(_lib.load(), f"hgr_cuda_{op}_{_dtype_tag(d)}")(
        C.byref(g.desc), int(level), _ptr(d), _ptr(out), _stream_of(d)))
    return _back(out, was)


def _require_level(g, level):
    if not (1 <= level <= g.levels()):
        raise HgrError("level out of range")


def interpolate_to_fine(coarse, g: GridHierarchy, level: int):
    """interpolate_to_fine (transforms.hpp:76-92)."""
    _require_level(g, level)
    if list(coarse.shape) != g.level_extents(level - 1):
        raise HgrError("interpolate_to_fine: shape mismatch")
    return _single("interpolate_to_fine", coarse, g, level, level)


def compute_coefficients(fine, g: GridHierarchy, level: int):
    """compute_coefficients (transforms.hpp:96-111)."""
    _require_level(g, level)
    if list(fine.shape) != g.level_extents(level):
        raise HgrError("compute_coefficients: shape mismatch")
    return _single("compute_coefficients", fine, g, level, level)


def apply_coefficients(coarse, coeffs, g: GridHierarchy, level: int):
    """apply_coefficients (transforms.hpp:115-124)."""
    _require_level(g, level)
    if list(coarse.shape) != g.level_extents(level - 1) or list(coeffs.shape) != g.level_extents(level):
        raise HgrError("apply_coefficients: shape mismatch")
    import torch
    c, was = _to_device(coarse)
    k, _ = _to_device(coeffs)
    k = k.to(device=c.device, dtype=c.dtype).contiguous()
    out = torch.empty(g.level_extents(level), dtype=c.dtype, device=c.device)
    _check(getattr(_lib.load(), f"hgr_cuda_apply_coefficients_{_dtype_tag(c)}")(
        C.byref(g.desc), int(level), _ptr(c), _ptr(k), _ptr(out), _stream_of(c)))
    return _back(out, was)


def compute_correction(coeffs, g: GridHierarchy, level: int):
    """compute_correction (correction.hpp:348-365)."""
    _require_level(g, level)
    if list(coeffs.shape) != g.level_extents(level):
        raise HgrError("compute_correction: shape mismatch")
    return _single("compute_correction", coeffs, g, level, level - 1)


def _fiber(op: str, v, h, nout_fn):
    import torch
    d, was = _to_device(v)
    n = d.shape[-1]
    hh = np.ascontiguousarray(np.asarray(h.cpu() if _is_torch(h) else h, dtype=d.cpu().numpy().dtype))
    if hh.size != n - 1:
        raise HgrError(f"{op}: |v| must equal |h|+1")
    count = d.numel() // n
    out = torch.empty(d.shape[:-1] + (nout_fn(n),), dtype=d.dtype, device=d.device)
    _check(getattr(_lib.load(), f"hgr_cuda_{op}_{_dtype_tag(d)}")(
        n, count, _ptr(d), hh.ctypes.data, _ptr(out), _stream_of(d)))
    return _back(out, was)


def synthetic_field(shape, dtype: str = "f64", seed: int = 12345, device=None):
    """Deterministic benchmark field on the device:
    sin(0.21 i) cos(0.13 j) + 0.5 sin(0.07 k) + 1e-3 eta(seed + flat), bitwise
    identical to tests/synthetic.smooth_field (factor tables built here with
    numpy, combined on the device with IEEE-exact mul/add)."""
    import torch
    e = list(shape) + [1] * (3 - len(shape))
    i, j, k = (np.arange(n, dtype=np.float64) for n in e)
    fa = np.ascontiguousarray(np.sin(0.21 * i))
    fb = np.ascontiguousarray(np.cos(0.13 * j))
    fc = np.ascontiguousarray(0.5 * np.sin(0.07 * k))
    out = torch.empty(tuple(shape), dtype=torch.float64 if dtype == "f64" else torch.float32,
                      device=device or "cuda")
    desc = _lib.GridDesc()
    desc.rank = len(shape)
    for d, n in enumerate(shape):
        desc.extents[d] = n
    _check(getattr(_lib.load(), f"hgr_cuda_synthetic_field_{dtype}")(
        C.byref(desc), _ptr(out), C.c_ulonglong(seed), fa.ctypes.data, fb.ctypes.data,
        fc.ctypes.data, _stream_of(out)))
    return out


def mass_apply(v, h):
    """mass_apply (correction.hpp:58-62)."""
    return _fiber("mass_apply", v, h, lambda n: n)


def transfer_apply(v, h):
    """transfer_apply (correction.hpp:67-88): R = P^T on one fiber (or a batch)."""
    n = v.shape[-1]
    if n < 3 or n % 2 == 0:
        raise HgrError("transfer_apply: fine fiber length must be odd")
    return _fiber("transfer_apply", v, h, lambda n: (n - 1) // 2 + 1)


def masstrans_apply(v, h):
    """masstrans_apply (correction.hpp:173-180)."""
    return _fiber("masstrans_apply", v, h, lambda n: (n - 1) // 2 + 1)


def thomas_solve(rhs, h):
    """thomas_solve (correction.hpp:217-223)."""
    return _fiber("thomas_solve", rhs, h, lambda n: n)


# ---- the progressive .hg container (storage.hpp:17-218) ------------------------

@dataclass
class HgFileHeader:
    """storage.hpp:36-55."""
    version: int
    precision_bytes: int
    rank: int
    extents: list
    coords: list
    class_offsets: list
    class_bytes: list
    header_bytes: int
    file_bytes: int

    def class_count(self) -> int:
        return len(self.class_bytes)

    def class_elements(self, cls: int) -> int:
        return self.class_bytes[cls] // self.precision_bytes

    def total_elements(self) -> int:
        n = 1
        for e in self.extents:
            n *= e
        return n


def write_file(r: RefactoredArray, path) -> int:
    """hgr::write_file (storage.hpp:86-126) of a pyramid held on the device (or
    host: it is staged to the current device). Classes are packed on the GPU;
    the file is byte-identical to the reference's. Returns the byte count."""
    import torch
    lib = _lib.load()
    data = r.data if _is_torch(r.data) else torch.from_numpy(np.ascontiguousarray(r.data)).cuda()
    data = data.contiguous()
    _check_shape(data, r.hierarchy, "write_file")
    n = C.c_uint64(0)
    _check(getattr(lib, f"hgr_cuda_write_hg_{_dtype_tag(data)}")(
        str(path).encode(), C.byref(r.hierarchy.desc), _ptr(data), C.byref(n), _stream_of(data)))
    return int(n.value)


def read_info(path) -> HgFileHeader:
    """hgr::read_info (storage.hpp:129-177): header and class table only."""
    lib = _lib.load()
    info = _lib.HgInfo()
    p = str(path).encode()
    _check(lib.hgr_hg_read_info(p, C.byref(info)))
    rank = info.rank
    extents = [int(info.extents[d]) for d in range(rank)]
    coords = []
    for d in range(rank):
        c = np.empty(extents[d], np.float64)
        _check(lib.hgr_hg_read_coords(p, d, c.ctypes.data))
        coords.append(c)
    nc = info.class_count
    offs, byts = np.zeros(nc, np.uint64), np.zeros(nc, np.uint64)
    _check(lib.hgr_hg_read_class_table(p, offs.ctypes.data, byts.ctypes.data, nc))
    return HgFileHeader(int(info.version), int(info.precision_bytes), rank, extents, coords,
                        [int(v) for v in offs], [int(v) for v in byts], int(info.header_bytes),
                        int(info.file_bytes))


@dataclass
class PrefixRead:
    array: RefactoredArray
    bytes_read: int


def read_prefix(path, upto_class: int, dtype: Optional[str] = None, device=None) -> PrefixRead:
    """hgr::read_prefix (storage.hpp:187-216): classes 0..upto_class into a
    zero-filled device pyramid (classes are scattered on the GPU)."""
    import torch
    h = read_info(path)
    dt = dtype or ("f64" if h.precision_bytes == 8 else "f32")
    g = GridHierarchy(h.coords)
    out = torch.empty(h.extents, dtype=torch.float64 if dt == "f64" else torch.float32,
                      device=device or "cuda")
    n = C.c_uint64(0)
    _check(getattr(_lib.load(), f"hgr_cuda_read_hg_prefix_{dt}")(
        str(path).encode(), int(upto_class), _ptr(out), C.byref(n), _stream_of(out)))
    return PrefixRead(RefactoredArray(out, g), int(n.value))
