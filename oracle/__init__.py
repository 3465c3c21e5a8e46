"""TEST INFRASTRUCTURE ONLY -- parity checkers for the B200 path.

Two CPU oracles behind one numpy-facing API:

* ``port``      -- ``oracle/lib/libhgr_oracle.so``, the plain-C restatement of
  the reference algorithm (``oracle/hgr_oracle.c``; every function cites the
  reference file:line it follows). Always buildable (``make -C oracle``).
* ``reference`` -- ``oracle/_ref/libhgr_ref.so``, the unmodified reference
  headers (/root/reference/proj/include) compiled behind a C ABI
  (``oracle/ref_capi.cpp``, ``make -C oracle ref``). Exists only where the
  reference tree was present at build time (it travels prebuilt to GPU boxes).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. The product library
(``paper_2007_04457_b200``) never imports it and has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "lib" / "libhgr_oracle.so"
REF_SO = HERE / "_ref" / "libhgr_ref.so"
REF_NATIVE_SO = HERE / "_ref" / "libhgr_ref_native.so"
REF_INCLUDE = Path("/root/reference/proj/include")


class OracleError(RuntimeError):
    pass


class _Grid(C.Structure):
    _fields_ = [("rank", C.c_int), ("n", C.c_size_t * 3), ("coords", C.c_void_p * 3)]


def build(force: bool = False) -> None:
    """Compile the C restatement, and the reference wrapper when the reference tree exists."""
    if force or not PORT_SO.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if REF_INCLUDE.exists() and (force or not REF_SO.exists()):
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def _dt(a):
    return "f64" if a.dtype == np.float64 else "f32"


class Oracle:
    """numpy wrapper over either CPU oracle (prefix ``hgro_`` or ``hgrref_``)."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            if not PORT_SO.exists():
                build()
            self.lib = C.CDLL(str(PORT_SO))
            self.pfx = "hgro_"
        elif kind == "reference-native":
            # the timing build (-O3 -march=native); only where this CPU has every
            # flag of the build machine
            if not native_usable():
                raise OracleError("reference-native build missing or not runnable on this CPU")
            self.lib = C.CDLL(str(REF_NATIVE_SO))
            self.pfx = "hgrref_"
        elif kind == "reference":
            if not REF_SO.exists():
                if REF_INCLUDE.exists():
                    build()
                else:
                    raise OracleError("reference oracle not built (oracle/_ref/libhgr_ref.so missing)")
            self.lib = C.CDLL(str(REF_SO))
            self.pfx = "hgrref_"
        else:
            raise ValueError(kind)
        getattr(self.lib, self.pfx + "last_error").restype = C.c_char_p

    # -- plumbing ---------------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self.pfx + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self._fn("last_error")().decode())

    def _grid(self, shape, coords=None):
        g = _Grid()
        g.rank = len(shape)
        keep = []
        for d, n in enumerate(shape):
            g.n[d] = int(n)
            if coords is not None and coords[d] is not None:
                c = np.ascontiguousarray(coords[d], dtype=np.float64)
                keep.append(c)
                g.coords[d] = c.ctypes.data
            else:
                g.coords[d] = None
        return g, keep

    @staticmethod
    def _p(a):
        return C.c_void_p(a.ctypes.data)

    # -- hierarchy --------------------------------------------------------------
    def levels(self, shape, coords=None):
        g, _k = self._grid(shape, coords)
        L = self._fn("levels")(C.byref(g))
        if L < 0:
            raise OracleError(self._fn("last_error")().decode())
        return L

    # -- refactor ---------------------------------------------------------------
    def decompose(self, data, coords=None):
        out = np.array(data, copy=True, order="C")
        g, _k = self._grid(out.shape, coords)
        self._check(self._fn("decompose_" + _dt(out))(C.byref(g), self._p(out)))
        return out

    def recompose(self, pyramid, upto_class=None, coords=None):
        src = np.ascontiguousarray(pyramid)
        g, _k = self._grid(src.shape, coords)
        if upto_class is None:
            upto_class = self.levels(src.shape, coords)
        out = np.empty_like(src)
        self._check(self._fn("recompose_" + _dt(src))(C.byref(g), self._p(src), self._p(out),
                                                      int(upto_class)))
        return out

    # -- single level -----------------------------------------------------------
    def _level_shape(self, shape, coords, level):
        L = self.levels(shape, coords)
        s = 1 << (L - level) if 0 <= level <= L else 1
        return tuple((n - 1) // s + 1 for n in shape)

    def interpolate_to_fine(self, coarse, shape, level, coords=None):
        coarse = np.ascontiguousarray(coarse)
        g, _k = self._grid(shape, coords)
        out = np.empty(self._level_shape(shape, coords, level), dtype=coarse.dtype)
        self._check(self._fn("interpolate_to_fine_" + _dt(coarse))(C.byref(g), int(level),
                                                                   self._p(coarse), self._p(out)))
        return out

    def compute_coefficients(self, fine, shape, level, coords=None):
        fine = np.ascontiguousarray(fine)
        g, _k = self._grid(shape, coords)
        out = np.empty_like(fine)
        self._check(self._fn("compute_coefficients_" + _dt(fine))(C.byref(g), int(level),
                                                                  self._p(fine), self._p(out)))
        return out

    def compute_correction(self, coeffs, shape, level, coords=None):
        coeffs = np.ascontiguousarray(coeffs)
        g, _k = self._grid(shape, coords)
        out = np.empty(self._level_shape(shape, coords, level - 1), dtype=coeffs.dtype)
        self._check(self._fn("compute_correction_" + _dt(coeffs))(C.byref(g), int(level),
                                                                  self._p(coeffs), self._p(out)))
        return out

    def _fiber(self, name, v, h, nout):
        v = np.ascontiguousarray(v)
        h = np.ascontiguousarray(h, dtype=v.dtype)
        out = np.empty(nout, dtype=v.dtype)
        self._check(self._fn(name + "_" + _dt(v))(C.c_size_t(v.size), self._p(v), self._p(h),
                                                  self._p(out)))
        return out

    def mass_apply(self, v, h):
        return self._fiber("mass_apply", v, h, len(v))

    def transfer_apply(self, v, h):
        return self._fiber("transfer_apply", v, h, (len(v) - 1) // 2 + 1)

    def masstrans_apply(self, v, h):
        return self._fiber("masstrans_apply", v, h, (len(v) - 1) // 2 + 1)

    def thomas_solve(self, rhs, h):
        return self._fiber("thomas_solve", rhs, h, len(rhs))

    def class_node_count(self, shape, cls, coords=None):
        L = self.levels(shape, coords)
        def cnt(l):
            s = 1 << (L - l)
            return int(np.prod([(n - 1) // s + 1 for n in shape]))
        return cnt(0) if cls == 0 else cnt(cls) - cnt(cls - 1)

    def extract_class(self, data, cls, coords=None):
        data = np.ascontiguousarray(data)
        g, _k = self._grid(data.shape, coords)
        out = np.empty(self.class_node_count(data.shape, cls, coords), dtype=data.dtype)
        self._check(self._fn("extract_class_" + _dt(data))(C.byref(g), self._p(data), int(cls),
                                                           self._p(out)))
        return out

    def scatter_class(self, data, cls, values, coords=None):
        data = np.array(data, copy=True, order="C")
        values = np.ascontiguousarray(values, dtype=data.dtype)
        g, _k = self._grid(data.shape, coords)
        self._check(self._fn("scatter_class_" + _dt(data))(C.byref(g), self._p(data), int(cls),
                                                           self._p(values)))
        return data

    # -- reference-only helpers (seeded fixtures, worker count) ------------------
    # storage.hpp (reference only): the .hg container
    def write_file(self, pyramid, path, coords=None):
        """hgr::write_file of a decomposed pyramid; returns the byte count."""
        assert self.kind.startswith("reference"), "the .hg container exists in the reference only"
        src = np.ascontiguousarray(pyramid)
        g, _k = self._grid(src.shape, coords)
        n = C.c_ulonglong(0)
        self._check(self._fn("write_file_" + _dt(src))(C.byref(g), self._p(src),
                                                       str(path).encode(), C.byref(n)))
        return int(n.value)

    def read_prefix(self, path, upto_class, shape, dtype):
        """hgr::read_prefix: (zero-filled pyramid, bytes_read)."""
        assert self.kind.startswith("reference"), "the .hg container exists in the reference only"
        out = np.zeros(shape, dtype=dtype)
        n = C.c_ulonglong(0)
        self._check(self._fn("read_prefix_" + _dt(out))(str(path).encode(), int(upto_class),
                                                        self._p(out), C.byref(n)))
        return out, int(n.value)

    def set_worker_count(self, n: int) -> None:
        if not self.kind.startswith("reference"):
            return
        self.lib.hgrref_set_worker_count(C.c_size_t(n))

    def worker_count(self) -> int:
        if not self.kind.startswith("reference"):
            return 1
        self.lib.hgrref_worker_count.restype = C.c_size_t
        return int(self.lib.hgrref_worker_count())


def native_usable() -> bool:
    """True if oracle/_ref/libhgr_ref_native.so exists and this CPU has every
    feature flag of the machine it was compiled on (-march=native)."""
    flags_file = HERE / "_ref" / "native_flags.txt"
    if not (REF_NATIVE_SO.exists() and flags_file.exists()):
        return False
    try:
        here = next(l for l in open("/proc/cpuinfo") if l.startswith("flags")).split(":", 1)[1].split()
    except (OSError, StopIteration):
        return False
    return set(flags_file.read_text().split()) <= set(here)


def available(kind: str) -> bool:
    if kind == "reference-native":
        return native_usable()
    return PORT_SO.exists() if kind == "port" else REF_SO.exists()


# -- libstdc++-compatible seeded fixtures (tests/oracle_helpers.hpp:230-246) ------
def _canonical(rng: np.random.RandomState, n: int) -> np.ndarray:
    # std::generate_canonical<double,53>(mt19937): two 32-bit draws, low word first,
    # summed in double then divided by 2^64 (libstdc++ bits/random.tcc).
    raw = rng._bit_generator.random_raw(2 * n).astype(np.float64)
    s = raw[0::2] + raw[1::2] * 4294967296.0
    r = s / 18446744073709551616.0
    r[r >= 1.0] = np.nextafter(1.0, 0.0)
    return r


def random_values(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """oracle::random_values (oracle_helpers.hpp:239-246), bit-exact vs libstdc++."""
    rng = np.random.RandomState(seed)
    return _canonical(rng, n) * (hi - lo) + lo


def random_coords(n: int, seed: int) -> np.ndarray:
    """oracle::random_coords (oracle_helpers.hpp:230-237), bit-exact vs libstdc++."""
    rng = np.random.RandomState(seed)
    gaps = _canonical(rng, n - 1) * (1.8 - 0.2) + 0.2
    c = np.zeros(n)
    for i in range(1, n):
        c[i] = c[i - 1] + gaps[i - 1]
    return c
